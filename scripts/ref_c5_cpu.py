"""C5 on the REAL reference (parafit), CPU: 8 toys of the C1 model at 10M
events (seeds 1000..1007, fit start (4.95, 0.52, -0.29, 0.31)), FitManager
over a thread pool of every core; the 256-toy figure is extrapolated x32 as
SURVEY §8(d) prescribes.  Runs only where /root/reference exists (the
builder container, not the GPU box); the output is kept in profiles/.

    python scripts/ref_c5_cpu.py [--toys 8] > profiles/r1_c5_reference_cpu.json
"""

import argparse
import json
import os
import platform
import sys
import time

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--toys", type=int, default=8)
    ap.add_argument("--n", type=int, default=10_000_000)
    args = ap.parse_args()
    os.environ.pop("PARAFIT_WORKERS", None)
    from parafit.core import Variable
    from parafit.engine import Backend
    from parafit.fitting import FitManager
    from parafit.mcgen import GenSpec, generate_1d
    from parafit.pdf import add_pdf, exponential, gaussian

    x = Variable.observable("x", 0.0, 10.0)
    mu = Variable("mu", 5.0, 0.0, 10.0, step=0.01)
    sigma = Variable("sigma", 0.5, 0.01, 5.0, step=1e-3)
    alpha = Variable("alpha", -0.3, -5.0, 5.0, step=1e-3)
    f = Variable("f", 0.3, 0.0, 1.0, step=1e-3)
    pdf = add_pdf([gaussian(x, mu, sigma), exponential(x, alpha)], [f])
    params = (mu, sigma, alpha, f)
    truth, start = (5.0, 0.5, -0.3, 0.3), (4.95, 0.52, -0.29, 0.31)
    workers = os.cpu_count() or 1
    backend = Backend("pool", workers=workers)
    gen_s = fit_s = 0.0
    calls = 0
    for t in range(args.toys):
        for v, val in zip(params, truth):
            v.value = val
        t0 = time.perf_counter()
        ds = generate_1d(pdf, x, GenSpec(args.n, seed=1000 + t))
        gen_s += time.perf_counter() - t0
        for v, val in zip(params, start):
            v.value = val
        t0 = time.perf_counter()
        r = FitManager(pdf, ds, backend=backend).fit()
        fit_s += time.perf_counter() - t0
        calls += r.n_calls
        print(f"toy {t}: {r.n_calls} calls, {r.status}", file=sys.stderr, flush=True)
    print(json.dumps({
        "study": "C5 toy fits on the reference (parafit FitManager, pool backend), CPU",
        "toys_run": args.toys, "events_per_toy": args.n, "nll_calls": calls, "fit_wall_s": fit_s,
        "nll_calls_per_s": calls / fit_s, "generation_s_per_toy": gen_s / args.toys,
        "extrapolated_256_toys_s": (gen_s + fit_s) * 256 / args.toys,
        "workers": workers, "cpu": platform.processor() or platform.machine(),
        "host": "builder container (the GPU box has no /root/reference)",
    }), flush=True)


if __name__ == "__main__":
    main()
