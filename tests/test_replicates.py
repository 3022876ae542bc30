"""Host logic of the replicate MLE study (tools/replicates.py; NEXT (f2), R29):
seeded subsets of the master field and the boxplot statistics per n."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import replicates  # noqa: E402


def test_subsets_seeded_distinct_and_sorted():
    a = replicates.subset(524288, 2000, 3)
    b = replicates.subset(524288, 2000, 3)
    c = replicates.subset(524288, 2000, 4)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert len(np.unique(a)) == 2000 and np.all(np.diff(a) > 0) and a.max() < 524288


def test_summary_statistics(tmp_path):
    p = tmp_path / "r.jsonl"
    rows = []
    for n, vals in ((2000, [0.4, 0.5, 0.6, 0.7]), (4000, [0.45, 0.5, 0.55])):
        for r, v in enumerate(vals):
            rows.append({"n": n, "rep": r, "seconds": 1.0,
                         "theta_hat": {"nu": v, "ell": 0.1, "sigma2": 1.0, "microergodic": 1.0 / 0.1 ** (2 * v)}})
    p.write_text("\n".join(json.dumps(x) for x in rows) + "\n")
    s = replicates.summary(str(p))
    d = s["per_n"]["2000"]["nu"]
    assert d["median"] == np.median([0.4, 0.5, 0.6, 0.7]) and d["min"] == 0.4 and d["max"] == 0.7
    assert abs(d["std"] - np.std([0.4, 0.5, 0.6, 0.7], ddof=1)) < 1e-15
    assert s["per_n"]["4000"]["replicates"] == 3
