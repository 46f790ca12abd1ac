"""BASELINE config 5 at full size (n = 5e7, 1.6e9 entries): two GPU solves and the SURVEY §8(c)
host certificate through the Tier S oracle (tests/tools/cfg5_certificate.py; ~20-30 min on one
B200 + its host).  Opt-in: SFAIRSC_CFG5_CERT=1 (the default GPU suite stays within minutes; the
committed record is profiles/r2x_cfg5_certificate.json).  SFAIRSC_CFG5_N overrides n."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(os.environ.get("SFAIRSC_CFG5_CERT") != "1", reason="opt-in: SFAIRSC_CFG5_CERT=1 (~25 min)")
def test_config5_certificate(tmp_path):
    out = tmp_path / "cert.json"
    cmd = [sys.executable, os.path.join(ROOT, "tests", "tools", "cfg5_certificate.py"), "--out", str(out)]
    if os.environ.get("SFAIRSC_CFG5_N"):
        cmd += ["--n", os.environ["SFAIRSC_CFG5_N"]]
    subprocess.run(cmd, check=True, cwd=ROOT)
    contract = json.loads(out.read_text())["contract"]
    assert all(contract.values()), contract
