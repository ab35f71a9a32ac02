"""The numeric kernel's scheduling knobs must never change a bit of the result: pieces of any
length (accumulators handed between CTAs inside a super-tile), ring depth, CTAs per SM, programmatic
dependent launch on or off.  Each setting runs in its own process (the knobs are read once per process) and
repeats the product, so a hand-over race would show up as a mismatch with the oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = [
    {},                                                                  # defaults
    {"SPAMM_EX_CTAS": "1", "SPAMM_PIECE_RECORDS": "1"},                  # as many pieces as fit: most are 1-2 records inside one tile
    {"SPAMM_EX_CTAS": "1", "SPAMM_PIECE_RECORDS": "3", "SPAMM_REC_WEIGHT": "1"},
    {"SPAMM_EX_CTAS": "1", "SPAMM_EX_STAGES": "2", "SPAMM_PIECE_RECORDS": "2", "SPAMM_REC_WEIGHT": "64"},
    {"SPAMM_PIECE_RECORDS": "1000000"},                                  # one piece per team
    {"SPAMM_PDL": "0", "SPAMM_EX_CTAS": "1", "SPAMM_PIECE_RECORDS": "2"},
    # a grid larger than what is resident (3 CTAs per SM requested, 1 fits) with chained pieces: a team only
    # waits for the head of a piece that was drawn, and therefore begun, before its own
    {"SPAMM_EX_CTAS": "3", "SPAMM_PIECE_RECORDS": "1", "N": "4096"},
]


@pytest.mark.parametrize("env", SETTINGS, ids=lambda e: ",".join(f"{k[6:] if k.startswith('SPAMM_') else k}={v}" for k, v in e.items()) or "defaults")
def test_scheduling_knobs_do_not_change_results(env):
    full = dict(os.environ)
    full.update({k: v for k, v in env.items() if k != "N"})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "stress_child.py"), env.get("N", "2048"), "1e-8",
                          "6" if "N" not in env else "3"],
                         env=full, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout[-2000:] + out.stderr[-2000:]
    if env.get("SPAMM_EX_CTAS") == "1" or "N" in env:
        assert "chained=0 " not in out.stdout, "this setting is meant to exercise pieces chained inside super-tiles: " + out.stdout
