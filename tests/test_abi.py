"""C-ABI library: loads, exports what include/ut.h declares, host-side logic (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2101_07956_b200 as ut

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ut.h")).read()
    return set(re.findall(r"^UT_API[^(]*?\b(ut_\w+)\s*\(", src, flags=re.M))


def test_header_and_binding_agree():
    assert _declared() == set(ut.ABI)


def test_library_exports_every_declared_symbol_and_nothing_else():
    out = subprocess.run(["nm", "-D", "--defined-only", ut.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert _declared() <= exported
    assert {s for s in exported if s.startswith("ut_")} == _declared()
    lib = ctypes.CDLL(ut.LIB_PATH)
    for s in _declared():
        assert getattr(lib, s)


def test_kernels_are_sm100a_sass():
    out = subprocess.run(["cuobjdump", "--list-elf", ut.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_null_and_empty_arguments():
    L = ut._lib
    assert L.ut_gather(None, None, 0, None, None) == ut.UT_EINVAL
    assert L.ut_release(None) == ut.UT_OK
    assert L.ut_register(None, 1, 1) is None
    assert ut.last_error()[0] == ut.UT_EINVAL
    assert L.ut_register(ctypes.c_void_p(4096), 0, 1) is None
    assert L.ut_register(ctypes.c_void_p(4096), 1 << 40, 1 << 40) is None   # overflow
    assert "overflow" in ut.last_error()[1]
    v = ctypes.c_int64()
    assert L.ut_error_pos(None, None, ctypes.byref(v)) == ut.UT_EINVAL
    assert ut.ut_plan_name(0) == "invalid"


def test_register_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    buf = ctypes.create_string_buffer(4096)
    with pytest.raises(ut.UTError) as e:
        ut.ut_register(ctypes.addressof(buf), 64, 64)
    assert e.value.code in (ut.UT_ECUDA, ut.UT_ENOTSUP)


# ---- plan selection (DESIGN.md §Plan selection; the paper's activation rule P:568) ------------
@pytest.mark.parametrize("rb,base,plan", [
    (2048, 0, "vec16.g32x"),     # 128-B multiple: no realignment
    (2052, 0, "realign.g32x"),   # 2052 B: realignment on
    (400, 0, "vec16.g32"),       # products rows
    (512, 0, "vec16.g32"),       # papers rows
    (2408, 0, "realign.g32x"),   # reddit rows
    (68, 0, "realign.g8"),       # tiny rows: 68 B from offsets 0/4/8/12 spans <= 5 chunks
    (4, 0, "narrow4"), (8, 8, "narrow8"), (1, 3, "narrow1"), (2, 2, "narrow2"),
    (4, 2, "realign.g2"),        # misaligned 4-B rows
    (16, 0, "vec16.g1"), (16, 8, "realign.g2"), (32, 0, "vec16.g2"),
    (400, 4, "realign.g32"), (520, 0, "realign.g32x"), (1024, 0, "vec16.g32x"),
])
def test_plan_examples(rb, base, plan):
    assert ut.ut_plan_probe(0x7F0000000000 + base, 1000, rb, 0x7E0000000000) == plan


def test_plan_admissible_for_every_width_and_base():
    for rb in range(1, 4097):
        for base in range(0, 128, 1 if rb < 64 else 7):
            p = ut.ut_plan_probe(0x10000 + base, 100, rb, 0x20000)
            if p.startswith("narrow"):
                assert rb in (1, 2, 4, 8) and base % rb == 0 and p == f"narrow{rb}"
            elif p.startswith("vec16"):
                assert rb % 16 == 0 and base % 16 == 0
                assert p == ("vec16.g32x" if rb > 512 else f"vec16.g{1 << max(0, (rb // 16 - 1).bit_length())}")
            else:
                assert p.startswith("realign")
                span = max((((base + k * rb) % 16) + rb + 15) // 16 for k in range(16))
                span = max(span, max(((k * rb) % 16 + rb + 15) // 16 for k in range(16)))
                if span <= 32:
                    g = int(p.split(".g")[1])
                    assert g >= span and g < 2 * span + 1
                else:
                    assert p == "realign.g32x"


def test_plan_depends_on_output_alignment():
    assert ut.ut_plan_probe(0x10000, 10, 400, 0x20000) == "vec16.g32"
    assert ut.ut_plan_probe(0x10000, 10, 400, 0x20004) == "realign.g32"
    assert ut.ut_plan_probe(0x10000, 10, 4, 0x20002) == "realign.g2"


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of ut_stats, ut_table_info and ut_coop_stats have the C structs' size
    and field offsets (compiled from include/ut.h by gcc)."""
    mirrors = {"ut_stats": ut._Stats, "ut_table_info": ut._Info, "ut_coop_stats": ut._CoopStats}
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "ut.h"', "int main(void) {"]
    for cname, py in mirrors.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    "-o", str(exe), str(src)], check=True)
    got = {}
    for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        c, f, v = l.split()
        got[(c, f)] = int(v)
    for cname, py in mirrors.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
