"""Generate tests/golden/theory.json by running the REFERENCE's theory checks
(dbsim.checks.check_theorem1_bound, check_lemma1; sgdlab.estimate_gradient_noise,
verify_lemma1_variance).  Build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_theory_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from dbsim import checks, sgdlab  # noqa: E402


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=float).ravel()]


def main():
    q = sgdlab.ConvexProblem.quadratic(dimension=8, mu=1.0, sample_noise_scale=0.02, sample_count=4096, seed=0)
    out = {"problem": {"dimension": 8, "mu": 1.0, "sample_noise_scale": 0.02, "sample_count": 4096, "seed": 0}}
    r = checks.check_theorem1_bound(q, 0.5, np.ones(8), n_seeds=200, n_iterations=80, seed=0)
    out["theorem1"] = {"gamma": 0.5, "n_seeds": 200, "n_iterations": 80, "seed": 0, "means": hx(r.means),
                       "std_errors": hx(r.std_errors), "bounds": hx(r.bounds), "sigma_sq": float(r.sigma_sq).hex(),
                       "passed": bool(r.passed), "max_excess_se": float(r.max_excess_se).hex()}
    v = checks.check_lemma1(q, np.ones(8), (1, 4, 16), n_draws=20_000, seed=0)
    out["lemma1"] = {"m_values": [1, 4, 16], "n_draws": 20000, "seed": 0, "variances": hx(v.variances),
                     "std_errors": hx(v.std_errors), "passed": bool(v.passed)}
    lg = sgdlab.LogisticProblem.synthetic(dimension=6, mu=0.1, sample_count=2000, seed=3)
    pts = [np.zeros(6), lg.optimum, np.ones(6) * 0.3]
    out["noise_logistic"] = {"dimension": 6, "mu": 0.1, "sample_count": 2000, "seed": 3, "batch_size": 1,
                             "n_draws": 3000, "draw_seed": 7,
                             "value": float(sgdlab.estimate_gradient_noise(lg, pts, 1, 3000, seed=7)).hex()}
    est = sgdlab.verify_lemma1_variance(q, np.ones(8), [2, 8], 5000, seed=4, with_replacement=False)
    out["lemma1_without_replacement"] = {"m_values": [2, 8], "n_draws": 5000, "seed": 4,
                                         "variances": hx([e.variance for e in est]),
                                         "std_errors": hx([e.std_error for e in est])}
    (HERE / "theory.json").write_text(json.dumps(out, indent=1))
    print("theorem1 passed", r.passed, "sigma^2", r.sigma_sq, "lemma1", v.variances)


if __name__ == "__main__":
    main()
