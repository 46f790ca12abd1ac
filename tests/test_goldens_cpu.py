"""The stored oracle goldens (tests/golden/, scripts/make_goldens.py) still describe the
graphs the generator draws, and are internally consistent with the paper's facts:
lambda_1 = 0 (F^T 1 = 0), ascending, below sigma (Prop. 3.4), the
oracle's own residuals through P:803 at the contract's 1e-9."""
import json
import os

import numpy as np
from synth import baseline_config

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _check(c, name, k):
    with open(os.path.join(GOLDEN, name)) as f:
        gold = json.load(f)
    ev = np.array(gold["evals"])
    assert len(ev) == k + 1 and gold["k"] == k
    assert abs(ev[0]) <= 1e-12 * gold["sigma"]
    assert np.all(np.diff(ev) >= -1e-12 * gold["sigma"]) and ev[-1] < gold["sigma"]
    assert max(gold["resid_rel_via_P803"]) <= 1e-9
    g, _ = baseline_config(c)
    ci = g.col.astype(np.int64)
    chk = int((ci * (np.arange(len(ci), dtype=np.int64) % 1000003 + 1)).sum() % (1 << 61))
    assert (gold["graph"]["n"], gold["graph"]["nnz"], gold["graph"]["col_checksum"]) == (g.n, g.nnz, chk)


def test_cfg2_tier_d_golden():
    _check(2, "cfg2_tier_d.json", 10)
    X = np.load(os.path.join(GOLDEN, "cfg2_tier_d_X.npz"))["X"]
    assert X.shape == (20000, 10)
    assert np.abs(X.T @ X - np.eye(10)).max() <= 1e-12


def test_cfg3_tier_s_golden():
    _check(3, "cfg3_tier_s.json", 20)
