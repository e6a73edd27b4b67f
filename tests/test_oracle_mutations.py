"""The oracle's pins must catch plausible mistakes in the oracle itself (VERDICT r01 item 1:
inflated magnitude scales passed every pin).  scripts/oracle_mutations.py applies each
mutation to a scratch copy of oracle/dcnv4_oracle.c and runs the CPU pin tests against it;
here a subset (the two scales the verdict named, a dropped m, a sign) runs in the suite."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import oracle_mutations  # noqa: E402

SUBSET = ["grad_dy magnitude scale x50", "softmax grad_mask magnitude scale x100",
          "grad_input drops m", "grad_dy sign"]


@pytest.mark.parametrize("name", SUBSET)
def test_mutation_is_caught(name):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "oracle_mutations.py"), "--only", name],
                       capture_output=True, text=True, timeout=600)
    assert "PATTERN NOT FOUND" not in r.stdout, r.stdout
    assert r.returncode == 0 and "caught" in r.stdout, r.stdout + r.stderr[-2000:]


def test_mutation_table_patterns_exist():
    src = open(os.path.join(ROOT, "oracle", "dcnv4_oracle.c")).read()
    for name, a, _ in oracle_mutations.MUTATIONS:
        assert a in src, name
