"""The portable cos used by the normal draw: the single-kernel pcos the
kernels run equals the definition form pcos_ref bit for bit (CPU)."""
import os
import subprocess

from conftest import ROOT


def test_pcos_single_kernel_equals_definition(tmp_path):
    exe = tmp_path / "test_pmath"
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", os.path.join(ROOT, "tests", "cpp", "test_pmath.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "5000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    assert " 0 mismatches" in r.stdout
