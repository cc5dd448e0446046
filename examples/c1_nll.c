/* examples/c1_nll.c -- a native (C) host on the C ABI alone (include/pfb200.h):
 * the C1 SumPdf NLL, add_pdf([gaussian(x; mu, sigma), exponential(x; alpha)],
 * [f]) on x in [0, 10], over events read from a raw little-endian float64 file.
 *
 *   cc -O2 -I include examples/c1_nll.c -L paper_1710_08826_b200/_native -lpfb200 \
 *      -L /usr/local/cuda/lib64 -lcudart -lm -o examples/c1_nll
 *   LD_LIBRARY_PATH=paper_1710_08826_b200/_native examples/c1_nll events.f64 5.0 0.5 -0.3 0.3
 *
 * Prints the NLL with 17 significant digits, or the reference error class the
 * status maps to.  The norms are the reference's closed forms
 * (pdf.py:130-161: gaussian via erf, exponential via exp; add nodes have
 * norm 1) on the same libm the reference's math module uses, so the value is
 * bitwise the reference nll's through DeviceBackend (tests/test_gpu_c_host.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pfb200.h"

static const double kLo = 0.0, kHi = 10.0;

/* pdf.py:130-138: sigma * sqrt(pi / 2) * (erf((hi - mu) / (sigma sqrt 2)) - erf((lo - mu) / (sigma sqrt 2))) */
static double gaussian_norm(double mu, double sigma) {
    const double s2 = sqrt(2.0), shp = sqrt(0.5 * 3.141592653589793);  /* math.pi */
    const double hi = erf((kHi - mu) / (sigma * s2)), lo = erf((kLo - mu) / (sigma * s2));
    return sigma * shp * (hi - lo);
}

/* pdf.py:147-161 on a finite box: (e^{alpha hi} - e^{alpha lo}) / alpha, or hi - lo for alpha = 0 */
static double exponential_norm(double alpha) {
    if (alpha == 0.0) return kHi - kLo;
    return (exp(alpha * kHi) - exp(alpha * kLo)) / alpha;
}

static const char* status_name(int code) {
    switch (code) {
        case PFB_OK: return "ok";
        case PFB_E_NONPOSITIVE_DENSITY: return "NonPositiveDensity";
        case PFB_E_NONFINITE_DENSITY: return "NonFiniteDensity";
        case PFB_E_NEGATIVE_DENSITY: return "NegativeDensity";
        case PFB_E_FRACTION_OUT_OF_RANGE: return "FractionOutOfRange";
        default: return "error";
    }
}

int main(int argc, char** argv) {
    if (argc != 6) {
        fprintf(stderr, "usage: %s events.f64 mu sigma alpha f\n", argv[0]);
        return 2;
    }
    FILE* fh = fopen(argv[1], "rb");
    if (!fh) {
        perror(argv[1]);
        return 2;
    }
    fseek(fh, 0, SEEK_END);
    const int64_t n = (int64_t)(ftell(fh) / 8);
    fseek(fh, 0, SEEK_SET);
    double* xs = (double*)malloc((size_t)n * sizeof(double));
    if (!xs || fread(xs, sizeof(double), (size_t)n, fh) != (size_t)n) {
        fprintf(stderr, "short read\n");
        return 2;
    }
    fclose(fh);
    const double mu = atof(argv[2]), sigma = atof(argv[3]), alpha = atof(argv[4]), f = atof(argv[5]);

    pfb_ctx* ctx = NULL;
    int rc = pfb_ctx_create(0, &ctx);
    if (rc != PFB_OK) {
        fprintf(stderr, "pfb_ctx_create: %s\n", pfb_strerror(rc));
        return 1;
    }
    pfb_store* st = NULL;
    pfb_plan* plan = NULL;
    if ((rc = pfb_store_create(ctx, 1, n, &st)) == PFB_OK) rc = pfb_store_upload(st, 0, xs, 0, n);
    /* post-order tree (PdfNode.walk): the two leaves on column 0, then the add node */
    const pfb_node nodes[3] = {
        {PFB_GAUSSIAN, 0, 0, -1, 2, 0},
        {PFB_EXPONENTIAL, 0, 0, -1, 1, 0},
        {PFB_ADD, 2, -1, -1, 1, 0},
    };
    if (rc == PFB_OK) rc = pfb_plan_compile(ctx, nodes, 3, NULL, 0, &plan);
    double nll = 0.0;
    pfb_err err;
    if (rc == PFB_OK) {
        const double values[4] = {mu, sigma, alpha, f};
        const double norms[3] = {gaussian_norm(mu, sigma), exponential_norm(alpha), 1.0};
        rc = pfb_nll(ctx, plan, st, 0, n, 0, values, 4, norms, 3, &nll, &err);
    }
    if (rc == PFB_OK)
        printf("%.17g\n", nll);
    else if (rc <= PFB_E_FRACTION_OUT_OF_RANGE)
        printf("%s index %lld\n", status_name(rc), (long long)err.index);
    else
        printf("%s: %s\n", status_name(rc), pfb_strerror(rc));
    if (plan) pfb_plan_destroy(plan);
    if (st) pfb_store_destroy(st);
    pfb_ctx_destroy(ctx);
    free(xs);
    return rc == PFB_OK ? 0 : 1;
}
