"""Build A/B variants of libut.so (same source, -D knobs) into build/variants/ (dev aid)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_07956_b200 import _build  # noqa: E402

VARIANTS = {
    "base": [],
    "l2_64": ["-DUT_LDHINT=4"], "l2_128": ["-DUT_LDHINT=1"], "l2_256": ["-DUT_LDHINT=2"],
    "ldplain": ["-DUT_LDHINT=3"],
    "ku1": ["-DUT_KU=1"], "ku2": ["-DUT_KU=2"], "ku8": ["-DUT_KU=8"], "kux1": ["-DUT_KUX=1"], "kux4": ["-DUT_KUX=4"],
    "minb6": ["-DUT_MINB=6"], "minb8": ["-DUT_MINB=8"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    out = os.path.join(_build.ROOT, "build", "variants")
    os.makedirs(out, exist_ok=True)
    for n in names:
        cmd = _build.command(os.path.join(out, f"libut_{n}.so"), VARIANTS[n])
        p = subprocess.run(cmd, capture_output=True, text=True)
        spill = [l for l in p.stderr.splitlines() if "spill" in l and " 0 bytes spill stores" not in l]
        print(n, "rc", p.returncode, "spills:", len(spill))
        if p.returncode:
            print(p.stderr[-2000:])
