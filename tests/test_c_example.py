"""The C ABI from plain C (examples/c_gather.c): compiles here against include/ut.h and
libut.so; runs on a B200 (-m gpu) and checks bytes against a memcpy loop."""
import os
import subprocess

import pytest

import paper_2101_07956_b200 as ut

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "c_gather")
BOX = os.path.join(ROOT, "build", "c_box")
POOL = os.path.join(ROOT, "build", "c_pool")


def _compile(name="c_gather", exe=EXE):
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    libdir = os.path.dirname(ut.LIB_PATH)
    cmd = ["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", f"{name}.c"), "-L", libdir, "-lut",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_example_compiles():
    _compile()
    assert os.path.exists(EXE)
    _compile("c_box", BOX)
    assert os.path.exists(BOX)


@pytest.mark.gpu
def test_c_box_example_runs():
    """ut_create(MANAGED) + ut_gather_multi from plain C: three entries on this box's GPU(s)."""
    _compile("c_box", BOX)
    p = subprocess.run([BOX, "8", "3"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "C-BOX OK" in p.stdout


@pytest.mark.gpu
def test_c_example_runs():
    _compile()
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "C-ABI OK" in p.stdout


def test_c_pool_example_runs_on_the_malloc_backend():
    """ut_pool_* bookkeeping from plain C, no GPU (the SYSTEM kind)."""
    _compile("c_pool", POOL)
    p = subprocess.run([POOL, "system"], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "C-POOL OK (system)" in p.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["managed", "pinned"])
def test_c_pool_example_runs(kind):
    """Two tables over one recycled block, each gather checked against memcmp."""
    _compile("c_pool", POOL)
    p = subprocess.run([POOL, kind], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert f"C-POOL OK ({kind})" in p.stdout
