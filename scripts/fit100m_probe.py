"""The 100M-event Dalitz fit of tests/test_gpu_fit100m.py with timings and the
distance to the reference's minimum, as one JSON line.

    python scripts/fit100m_probe.py
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from tests.test_gpu_fit100m import run_fit

    with open(os.path.join(ROOT, "tests", "golden", "fit_c4_100m.json")) as fh:
        ref = json.load(fh)
    r, _, tm = run_fit(ref)
    dev = [abs(v - rv) / re for v, rv, re in zip(r.values, ref["values"], ref["errors"])]
    rel = [abs(v - rv) / abs(rv) for v, rv in zip(r.values, ref["values"])]
    print(json.dumps({
        "probe": "100M-event Dalitz fit (C4 model, 6 free) vs the reference's fit of the same events",
        "status": r.status, "calls": r.n_calls, "ref_calls": ref["n_calls"],
        "nll_min": r.nll_min, "ref_nll_min": ref["nll_min"],
        "nll_min_rel": abs(r.nll_min - ref["nll_min"]) / abs(ref["nll_min"]),
        "max_dev_sigma": max(dev), "max_dev_rel": max(rel),
        "device": tm, "fit_timing": r.timing, "reference_timing": ref["reference_timing"],
    }), flush=True)


if __name__ == "__main__":
    main()
