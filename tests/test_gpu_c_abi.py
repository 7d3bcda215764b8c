"""The C-ABI used from plain C (examples/c_solve.c): compiled with gcc against
include/spcg_b200.h and the in-tree library, run on the GPU; three solves of
a 2-D Poisson system (full CSR, symmetric half privatized / atomic) checked on
the host."""

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_c_program_solves_through_the_c_abi(tmp_path):
    from paper_1010_4639_b200 import _native as N

    lib = Path(N.LIB_PATH)
    exe = tmp_path / "c_solve"
    subprocess.run(["gcc", "-O2", "-I", str(ROOT / "include"), str(ROOT / "examples" / "c_solve.c"),
                    "-L", str(lib.parent), "-lspcg_b200", f"-Wl,-rpath,{lib.parent}", "-lm",
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "64"], capture_output=True, text=True, timeout=120)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
    assert out.stdout.count("converged 1") == 3
