"""Writes tests/golden/oracle_C1_trajectories.json by calling ONLY oracle/
and qfgen/ (never the CUDA path): the C1 workload (4 starts) run to verdict
by the plain C oracle, with the per-sweep cost of the first 30 sweeps.

It is a regression fixture for the oracle itself (an accidental change to its
arithmetic shows up as a diff); it is not a pin -- the pins are in
tests/test_oracle_pins.py.  Regenerate only with a commit message naming the
passage or DESIGN.md reading that justifies the change.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import qfgen  # noqa: E402


def main():
    w = qfgen.workload("C1")
    c = oracle.Circuit(w.n, w.locs, w.kinds, w.const_mats)
    r = oracle.instantiate(c, w.target_unitary(), w.initial(),
                           oracle.default_params(max_iters=w.max_iters), record_sweeps=30,
                           nthreads=1)
    out = {
        "citation": "Alg. 1 QFactor (PAPER.md P:579-638), hyperparameters P:532; "
                    "workload C1 of SURVEY.md 8d (qfgen)",
        "generator": "tests/golden/make_golden.py (oracle only)",
        "verdict": r.verdict.tolist(),
        "iters": r.iters.tolist(),
        "delta": [float(x) for x in r.delta],
        "cost_first30": [[None if np.isnan(x) else float(x) for x in row] for row in r.cost_hist],
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_C1_trajectories.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
