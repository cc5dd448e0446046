// pfb_objective.cuh -- the minimiser's objective in C (included at the end of
// pfb_api.cu: it uses the plan / store / pack internals).
//
// The reference objective (FitManager.fcn, P/fitting.py:436-447) costs
// ~20-35 us of Python per call on top of the kernel (set_value, snapshot,
// resolve_norms with its fingerprints, _needed_columns, backend.map): more
// than the NLL itself at 1M events.  A pfb_objective binds a plan, a store
// and a range once; a call maps the free-parameter vector x straight to the
// plan's raw values, recomputes only the normalisations whose inputs changed
// (bit compare, the role of the reference's generation fingerprints), and
// runs the fused launch -- one C call per minimiser step.
//
// Norms in C are the reference's own formulas on the same doubles:
//   gaussian   sigma * sqrt(pi/2) * (erf((hi - mu)/(sigma sqrt 2)) - erf((lo - mu)/(sigma sqrt 2)))
//              (P/pdf.py:130-138; libm erf as CPython's math.erf -> the same bits)
//   exponential (exp(alpha hi) - exp(alpha lo)) / alpha, hi - lo at alpha = 0 (P/pdf.py:147-161)
//   add / prod 1 (P/pdf.py:238-239), or a constant supplied at creation
//   dalitz     Re(c I c^H), c_k = mag_k e^{i phase_k}, I the overlap matrix supplied at
//              creation (P/dalitz.py:332-349; shapes must be fixed)
// Any norm failure returns PFB_E_NONPOSITIVE_NORM / PFB_E_UNBOUNDED_OBSERVABLE
// with err->node set: the caller re-evaluates that point through the
// reference path, which raises the reference's exception.

struct pfb_objective {
    pfb_ctx* ctx = nullptr;
    pfb_plan* plan = nullptr;
    const pfb_store* store = nullptr;
    int64_t begin = 0, end = 0;
    int nfree = 0;
    std::vector<int> src;            // per raw value: index into x, or -1
    std::vector<double> cval;        // per raw value: the constant
    std::vector<pfb_obj_node> node;  // per plan node
    std::vector<double> mat;         // dalitz overlap matrix, K x K (re, im)
    std::vector<double> lower, upper;  // free-parameter bounds (empty: unchecked)
    // caches: last inputs and norms per node
    std::vector<double> values, norms;
    std::vector<std::vector<double>> last_in;
    std::vector<char> have;
};

static const double kSqrt2 = 1.4142135623730951;        // math.sqrt(2.0)
static const double kSqrtHalfPi = 1.2533141373155001;   // math.sqrt(0.5 * math.pi)

// One node's norm from the raw values; PFB_OK or the failing status.
static int obj_norm(const pfb_objective* o, int i, const double* raw, double* out) {
    const pfb_obj_node& nd = o->node[i];
    double v = nd.value;
    switch (nd.norm_kind) {
        case PFB_NORM_CONST:
            break;
        case PFB_NORM_GAUSSIAN: {
            const double mu = raw[0], sigma = raw[1];
            if (!(sigma > 0.0)) return PFB_E_NONPOSITIVE_NORM;
            const double h = std::isinf(nd.hi) ? 1.0 : erf((nd.hi - mu) / (sigma * kSqrt2));
            const double l = std::isinf(nd.lo) ? -1.0 : erf((nd.lo - mu) / (sigma * kSqrt2));
            v = sigma * kSqrtHalfPi * (h - l);
            break;
        }
        case PFB_NORM_EXPONENTIAL: {
            const double alpha = raw[0], lo = nd.lo, hi = nd.hi;
            if (alpha == 0.0) {
                if (std::isinf(lo) || std::isinf(hi)) return PFB_E_UNBOUNDED_OBSERVABLE;
                v = hi - lo;
                break;
            }
            const double up = !std::isinf(hi) ? exp(alpha * hi) : (alpha < 0 ? 0.0 : INFINITY);
            const double dn = !std::isinf(lo) ? exp(alpha * lo) : (alpha > 0 ? 0.0 : INFINITY);
            if (std::isinf(up) || std::isinf(dn)) return PFB_E_UNBOUNDED_OBSERVABLE;
            v = (up - dn) / alpha;
            break;
        }
        case PFB_NORM_DALITZ: {
            const int K = (int)nd.value;  // term count
            double cre[kMaxDal], cim[kMaxDal];
            for (int k = 0; k < K; ++k) {
                const double mag = raw[4 * k + 2], ph = raw[4 * k + 3];
                cre[k] = mag * cos(ph);
                cim[k] = mag * sin(ph);
            }
            // total = sum_i c_i sum_j I_ij conj(c_j)
            double tre = 0.0, tim = 0.0;
            for (int a = 0; a < K; ++a) {
                double sre = 0.0, sim = 0.0;
                for (int b = 0; b < K; ++b) {
                    const double ire = o->mat[2 * (a * K + b)], iim = o->mat[2 * (a * K + b) + 1];
                    // I_ab * conj(c_b)
                    sre += ire * cre[b] + iim * cim[b];
                    sim += iim * cre[b] - ire * cim[b];
                }
                tre += cre[a] * sre - cim[a] * sim;
                tim += cre[a] * sim + cim[a] * sre;
            }
            const double scale = fabs(tre) > 1e-300 ? fabs(tre) : 1e-300;
            if (fabs(tim) > 1e-10 * scale) return PFB_E_NONPOSITIVE_NORM;
            if (!(tre > 0.0)) return PFB_E_NONPOSITIVE_NORM;
            v = tre;
            break;
        }
        default:
            return PFB_E_INVALID_ARGUMENT;
    }
    if (!(std::isfinite(v) && v > 0.0)) return PFB_E_NONPOSITIVE_NORM;  // NormalizationValue (pdf.py:45-55)
    *out = v;
    return PFB_OK;
}

// x -> o->values, o->norms (cached per node on its raw inputs' bits).
static int obj_fill(pfb_objective* o, const double* x, pfb_err* err) {
    pfb_plan* p = o->plan;
    for (size_t k = 0; k < o->lower.size(); ++k)
        if (!(o->lower[k] <= x[k] && x[k] <= o->upper[k])) {  // NaN fails too
            if (err) {
                err->code = PFB_E_OUT_OF_BOUNDS;
                err->node = -1;
                err->index = (int64_t)k;
                err->value = x[k];
            }
            return PFB_E_OUT_OF_BOUNDS;
        }
    for (int r = 0; r < p->nraw; ++r) o->values[r] = o->src[r] >= 0 ? x[o->src[r]] : o->cval[r];
    const int nn = (int)p->nodes.size();
    for (int i = 0; i < nn; ++i) {
        const int off = p->raw_off[i], np = p->nodes[i].nparam;
        const double* raw = o->values.data() + off;
        std::vector<double>& last = o->last_in[i];
        if (o->have[i] && memcmp(last.data(), raw, sizeof(double) * np) == 0) continue;
        double v = 0.0;
        const int st = obj_norm(o, i, raw, &v);
        if (st) {
            if (err) {
                err->code = st;
                err->node = i;
                err->index = -1;
                err->value = NAN;
            }
            o->have[i] = 0;
            return st;
        }
        o->norms[i] = v;
        last.assign(raw, raw + np);
        o->have[i] = 1;
    }
    return PFB_OK;
}

extern "C" {

int pfb_objective_create(pfb_ctx* c, pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end, int32_t nfree,
                         const int32_t* value_src, const double* value_const, const pfb_obj_node* nodes,
                         const double* dalitz_matrix, pfb_objective** out) {
    if (!c || !p || !st || !out || p->ctx != c || st->ctx != c || nfree < 0 || !value_src || !value_const ||
        !nodes)
        return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end <= begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    *out = nullptr;
    auto o = std::make_unique<pfb_objective>();
    o->ctx = c;
    o->plan = p;
    o->store = st;
    o->begin = begin;
    o->end = end;
    o->nfree = nfree;
    o->src.assign(value_src, value_src + p->nraw);
    o->cval.assign(value_const, value_const + p->nraw);
    for (int r = 0; r < p->nraw; ++r)
        if (o->src[r] >= nfree) return PFB_E_INVALID_ARGUMENT;
    const int nn = (int)p->nodes.size();
    o->node.assign(nodes, nodes + nn);
    for (int i = 0; i < nn; ++i) {
        const int k = o->node[i].norm_kind;
        const int kind = p->nodes[i].kind;
        if (k == PFB_NORM_GAUSSIAN && kind != PFB_GAUSSIAN) return PFB_E_INVALID_ARGUMENT;
        if (k == PFB_NORM_EXPONENTIAL && kind != PFB_EXPONENTIAL) return PFB_E_INVALID_ARGUMENT;
        if (k == PFB_NORM_DALITZ) {
            if (kind != PFB_DALITZ || !dalitz_matrix) return PFB_E_INVALID_ARGUMENT;
            const int K = p->nodes[i].nparam / 4;
            o->node[i].value = K;
            o->mat.assign(dalitz_matrix, dalitz_matrix + 2 * K * K);
        }
        if (k < PFB_NORM_CONST || k > PFB_NORM_DALITZ) return PFB_E_INVALID_ARGUMENT;
    }
    o->values.assign(p->nraw, 0.0);
    o->norms.assign(nn, 1.0);
    o->last_in.resize(nn);
    o->have.assign(nn, 0);
    *out = o.release();
    return PFB_OK;
}

int pfb_objective_set_bounds(pfb_objective* o, const double* lower, const double* upper) {
    if (!o || (!lower && o->nfree) || (!upper && o->nfree)) return PFB_E_INVALID_ARGUMENT;
    o->lower.assign(lower, lower + o->nfree);
    o->upper.assign(upper, upper + o->nfree);
    return PFB_OK;
}

int pfb_objective_set_matrix(pfb_objective* o, const double* dalitz_matrix) {
    if (!o || !dalitz_matrix || o->mat.empty()) return PFB_E_INVALID_ARGUMENT;
    std::copy(dalitz_matrix, dalitz_matrix + o->mat.size(), o->mat.begin());
    for (auto& h : o->have) h = 0;
    return PFB_OK;
}

int pfb_objective_eval(pfb_objective* o, const double* x, int32_t nfree, double* out_nll, pfb_err* out_err) {
    if (!o || (!x && nfree) || nfree != o->nfree || !out_nll) return PFB_E_INVALID_ARGUMENT;
    clear_err(out_err);
    const int st = obj_fill(o, x, out_err);
    if (st) return st;
    return nll_common(o->ctx, o->plan, o->store, o->begin, o->end, 0, o->values.data(), o->plan->nraw,
                      o->norms.data(), (int32_t)o->norms.size(), nullptr, 0, out_nll, out_err);
}

int pfb_objective_eval_batch(pfb_objective* o, const double* xs, int32_t npts, int32_t nfree, double* out_nll,
                             pfb_err* out_err) {
    if (!o || !xs || nfree != o->nfree || !out_nll || !out_err || npts < 1 || npts > kMaxPts)
        return PFB_E_INVALID_ARGUMENT;
    const int nraw = o->plan->nraw, nn = (int)o->norms.size();
    std::vector<double> vals((size_t)npts * nraw), nv((size_t)npts * nn);
    int first_bad = npts;  // sequential semantics: nothing after the first host failure
    for (int m = 0; m < npts; ++m) {
        clear_err(out_err + m);
        const int st = obj_fill(o, xs + (size_t)m * nfree, out_err + m);
        if (st) {
            first_bad = m;
            break;
        }
        std::copy(o->values.begin(), o->values.end(), vals.begin() + (size_t)m * nraw);
        std::copy(o->norms.begin(), o->norms.end(), nv.begin() + (size_t)m * nn);
    }
    if (first_bad > 0) {
        const int code = pfb_nll_batch(o->ctx, o->plan, o->store, o->begin, o->end, 0, vals.data(), first_bad,
                                       nraw, nv.data(), nn, out_nll, out_err);
        if (code >= PFB_E_INVALID_ARGUMENT) return code;
    }
    return PFB_OK;
}

int pfb_objective_destroy(pfb_objective* o) {
    delete o;
    return PFB_OK;
}

}  // extern "C"
