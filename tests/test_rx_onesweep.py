"""The one-sweep request-index sort (look-back digit offsets, OB_RX_ONESWEEP=1) against the oracle.

The build default is the hist + scan path; the environment switch makes the engine take the
one-sweep path, so the srpe / full parity and long-request tests are re-run under it in a
child process (the switch is read per sort, captured graphs keep their path).
"""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_onesweep_sort_parity():
    env = dict(os.environ, OB_RX_ONESWEEP="1")
    cmd = [sys.executable, "-m", "pytest", os.path.join(HERE, "test_gpu_parity.py"), "-x", "-q", "-m", "gpu",
           "-k", "srpe_strategy or long_request_segments or config1_against_reference or graph_replay"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
