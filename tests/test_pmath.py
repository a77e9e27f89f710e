"""The normal draw's log / cos (pmath.h, shared by the kernels and the
oracle): correctly rounded against libquadmath (113-bit) on the draw's input
sets, and how often they equal glibc's (the literal reference's libm), which
is itself not correctly rounded on ~0.1% of these inputs (CPU)."""
import os
import re
import subprocess

from conftest import ROOT


def test_plog_pcos_correctly_rounded_and_glibc_rates(tmp_path):
    exe = tmp_path / "test_pmath"
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", os.path.join(ROOT, "tests", "cpp", "test_pmath.cpp"),
                    "-o", str(exe), "-lquadmath"], check=True)
    r = subprocess.run([str(exe), "2000000"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    m = re.search(r"log not CR (\d+), cos not CR (\d+) \| equal to glibc: log ([\d.]+)% cos ([\d.]+)% normal ([\d.]+)% "
                  r"\| glibc CR: log ([\d.]+)% cos ([\d.]+)%", r.stdout)
    assert m, r.stdout
    log_bad, cos_bad = int(m.group(1)), int(m.group(2))
    normal_eq, glibc_log_cr, glibc_cos_cr = float(m.group(5)), float(m.group(6)), float(m.group(7))
    assert log_bad == 0 and cos_bad == 0
    # every mismatch with glibc is a draw where glibc itself is not correctly rounded
    assert normal_eq >= min(glibc_log_cr, glibc_cos_cr) - 0.1
    assert normal_eq > 99.5
