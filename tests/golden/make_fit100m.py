"""Golden fixture for the north-star target: a 100M-event Dalitz fit, run with
the REAL reference (parafit) in this container.

    python tests/golden/make_fit100m.py            # ~20 min on 8 cores, ~15 GB RAM

The reference draws 100M D0 -> pi+ pi- pi0 events with its own generator
(parafit/mcgen.py:157, GenSpec seed below) and fits the C3 model (six free
coherent-sum coefficients, 400 x 400 normalisation grid) from the same start
as fits.json's c3 entry, with its FitManager (parafit/fitting.py:410) over a
thread-pool backend.  The fixture keeps the generator spec, SHA-256 of the raw
columns, exact column sums and sample rows (so the GPU box, which regenerates the events on the device
from the spec, can prove it holds the same 100M events), the reference's fit
result and its wall-clock times.  tests/test_gpu_fit100m.py checks the device
fit against it.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (puts the reference on sys.path)

from parafit.core import UnbinnedDataSet, Variable, snapshot  # noqa: E402
from parafit.dalitz import dalitz_pdf  # noqa: E402
from parafit.engine import Backend, nll  # noqa: E402
from parafit.fitting import FitManager  # noqa: E402
from parafit.mcgen import GenSpec, generate_dalitz  # noqa: E402

N_EVENTS = 100_000_000
SEED = 4  # GenSpec(100_000_000, seed=4), grid 400 x 400
START = {"rhom_mag": 0.8, "rhom_ph": 0.05, "rho0_mag": 0.5, "rho0_ph": 0.2, "nr_mag": 18.0, "nr_ph": -0.4}
SAMPLE_ROWS = [0, 1, 2, 4095, 4096, 12_345_678, 50_000_000, 99_999_998, 99_999_999]


def main():
    workers = os.cpu_count() or 1
    terms = mg.c3_terms()  # generator truth
    t0 = time.perf_counter()
    ds = generate_dalitz(terms, mg.D_CHANNEL, GenSpec(n_events=N_EVENTS, seed=SEED))
    t_gen = time.perf_counter() - t0
    s12v, s13v = ds.column("s12"), ds.column("s13")
    print(f"generated {len(s12v)} in {t_gen:.1f} s", flush=True)

    terms = mg.c3_terms()
    for t in terms:
        for var in (t.magnitude, t.phase):
            if var.name in START:
                var.value = START[var.name]
    s12 = Variable.observable("s12", *mg.D_CHANNEL.s12_range)
    s13 = Variable.observable("s13", *mg.D_CHANNEL.s13_range)
    data = UnbinnedDataSet([s12, s13])
    data.extend([s12v, s13v])
    pdf = dalitz_pdf(terms, mg.D_CHANNEL, s12_obs=s12, s13_obs=s13, grid=(400, 400))
    backend = Backend("pool", workers=workers)
    t0 = time.perf_counter()
    nll_start = nll(pdf, data, snapshot(pdf.param_closure()), backend)
    t_nll = time.perf_counter() - t0
    print(f"nll at start {nll_start!r} in {t_nll:.2f} s", flush=True)
    t0 = time.perf_counter()
    r = FitManager(pdf, data, backend=backend).fit()
    t_fit = time.perf_counter() - t0
    print(f"fit {r.status} in {t_fit:.1f} s, {r.n_calls} calls", flush=True)

    out = {
        "spec": {"n_events": N_EVENTS, "seed": SEED},
        "columns": {
            "sha256_s12": hashlib.sha256(np.ascontiguousarray(s12v, dtype="<f8").tobytes()).hexdigest(),
            "sha256_s13": hashlib.sha256(np.ascontiguousarray(s13v, dtype="<f8").tobytes()).hexdigest(),
            "fsum_s12": math.fsum(s12v),
            "fsum_s13": math.fsum(s13v),
            "rows": SAMPLE_ROWS,
            "s12": [float(s12v[i]) for i in SAMPLE_ROWS],
            "s13": [float(s13v[i]) for i in SAMPLE_ROWS],
        },
        "start": START,
        "grid": [400, 400],
        "nll_start": nll_start,
        "names": list(r.names),
        "values": np.asarray(r.values).tolist(),
        "errors": np.asarray(r.errors).tolist(),
        "nll_min": r.nll_min,
        "n_calls": r.n_calls,
        "status": r.status,
        "reference_timing": {"generate_s": t_gen, "nll_s": t_nll, "fit_s": t_fit, "workers": workers,
                             "host": "builder container CPU (not the GPU box)"},
    }
    with open(os.path.join(mg.OUT, "fit_c4_100m.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
