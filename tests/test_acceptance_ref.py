"""The reference's own acceptance suite (proj/tests/acceptance.cpp, all 9
criteria), compiled UNMODIFIED against the drop-in headers (include/pump)
and libpump_gpu.so by tools/Makefile, run on the B200 with the reference's
2-D scenarios (committed under tests/golden/scenarios).

Criterion 4 draws 100000 particles (cp_compare), criterion 9 observes every
explore round through the RoundHook, criterion 3 builds its Scenario in code
(build_models without the JSON loader)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "acceptance_ref")


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_on_the_gpu():
    if not os.path.exists(BIN):
        pytest.skip("tools/acceptance_ref not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "scenarios")], capture_output=True, text=True,
                       timeout=1500)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if re.match(r"^\[\d\]", ln)]
    assert len(lines) == 9, r.stdout + r.stderr
    failed = [ln for ln in lines if " PASS " not in ln]
    assert not failed, "\n".join(failed)
    assert r.returncode == 0
