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
//   polynomial the device Gauss-Legendre integral of the node alone (pfb_quadrature,
//              P/pdf.py:181-199), launched only when a coefficient moved
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
    int persistent = 0;              // pfb_objective_set_persistent
    NllArgs args;                    // the persistent path's packed arguments
    // caches: last inputs and norms per node
    std::vector<double> values, norms;
    std::vector<std::vector<double>> last_in;
    std::vector<char> have;
    std::vector<int> pend;  // per node: the unresolved quadrature slot its norm waits on, or -1
};

// The quadrature norms of one pfb_objective_eval_batch: each is launched into
// its own result slot as obj_fill meets it and the batch waits once for all
// of them (instead of a launch + wait per norm); a point's norm that is still
// in flight is recorded as a use (point, node, slot) and filled in at the wait.
struct QuadBatch {
    struct Req {
        int m, node, frac;
        std::unique_ptr<NllArgs> A;
    };
    std::vector<Req> req;
    std::vector<std::array<int, 3>> use;  // (point, node, slot)
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
        case PFB_NORM_QUADRATURE: {
            // the node's own plan (one node: its raw values, root norm 1) over the rule
            const double one = 1.0;
            pfb_err e;
            const int st = pfb_quadrature(o->ctx, nd.quad_plan, nd.quad_rule, nd.weight_col, raw,
                                          nd.quad_plan->nraw, &one, 1, &v, &e);
            if (st) return st;
            break;
        }
        default:
            return PFB_E_INVALID_ARGUMENT;
    }
    if (!(std::isfinite(v) && v > 0.0)) return PFB_E_NONPOSITIVE_NORM;  // NormalizationValue (pdf.py:45-55)
    *out = v;
    return PFB_OK;
}

// x -> o->values, o->norms (cached per node on its raw inputs' bits).  With
// `qb`, quadrature norms are enqueued for point m (o->pend) instead of waited for.
static int obj_fill(pfb_objective* o, const double* x, pfb_err* err, QuadBatch* qb = nullptr, int m = 0) {
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
        const pfb_obj_node& nd = o->node[i];
        if (qb && nd.norm_kind == PFB_NORM_QUADRATURE) {
            const int q = (int)qb->req.size();  // the caller keeps a slot per quadrature node free
            if (quad_check(o->ctx, nd.quad_plan, nd.quad_rule, nd.weight_col)) return PFB_E_INVALID_ARGUMENT;
            QuadBatch::Req r{m, i, -1, std::make_unique<NllArgs>()};
            const double one = 1.0;
            const int rc = quad_enqueue(o->ctx, nd.quad_plan, nd.quad_rule, nd.weight_col, raw, &one, q, r.A.get(),
                                        &r.frac);
            if (rc) return rc;
            qb->req.push_back(std::move(r));
            o->pend[i] = q;
            o->norms[i] = NAN;
            last.assign(raw, raw + np);
            o->have[i] = 1;
            continue;
        }
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
        if (!o->pend.empty()) o->pend[i] = -1;
        last.assign(raw, raw + np);
        o->have[i] = 1;
    }
    return PFB_OK;
}

// Wait for the batch's quadratures and fill their norms into the points that
// use them (nv: npts x nn) and into the node cache.  Returns PFB_OK, a fatal
// code, or -1 with the first failing norm in sequential order (lowest point,
// then lowest node) in *fail_m / *fail_err -- the cache is then dropped (the
// sequential objective stops at that norm; recomputing gives the same bits).
static int quad_flush(pfb_objective* o, QuadBatch* qb, double* nv, int* fail_m, pfb_err* fail_err) {
    if (qb->req.empty()) return PFB_OK;
    const int nn = (int)o->norms.size();
    int rc = quad_wait(o->ctx);
    if (rc) return rc;
    std::vector<double> v(qb->req.size());
    std::vector<int> code(qb->req.size());
    int worst = -1;
    for (size_t q = 0; q < qb->req.size(); ++q) {
        const QuadBatch::Req& r = qb->req[q];
        pfb_err e;
        code[q] = quad_collect(o->ctx, o->node[r.node].quad_plan, *r.A, (int)q, r.frac, &v[q], &e);
        if (code[q] >= PFB_E_INVALID_ARGUMENT) return code[q];
        if (!code[q] && !(std::isfinite(v[q]) && v[q] > 0.0)) code[q] = PFB_E_NONPOSITIVE_NORM;
        if (code[q] && (worst < 0 || r.m < qb->req[worst].m || (r.m == qb->req[worst].m && r.node < qb->req[worst].node)))
            worst = (int)q;
    }
    for (const auto& u : qb->use) nv[(size_t)u[0] * nn + u[1]] = v[u[2]];
    for (int i = 0; i < nn; ++i)
        if (o->pend[i] >= 0) {
            o->norms[i] = v[o->pend[i]];
            o->pend[i] = -1;
        }
    if (worst >= 0) {
        *fail_m = qb->req[worst].m;
        fail_err->code = code[worst];
        fail_err->node = qb->req[worst].node;
        fail_err->index = -1;
        fail_err->value = NAN;
        for (auto& h : o->have) h = 0;
    }
    qb->req.clear();
    qb->use.clear();
    return worst >= 0 ? -1 : PFB_OK;
}

// ---- the persistent kernel (pfb_nll_task.cuh nll_persist_kernel) -----------------

static constexpr unsigned long long kPersistIdleNs = 20ull * 1000 * 1000;  // 20 ms without a call: leave

// Make the resident kernel the one of `kind` (stop / start as needed).  The
// kernel's doorbell starts at c->persist_ctl[0], which the device release word
// go[0] is set to on the persistent stream before the launch.
static int persist_start(pfb_ctx* c, int kind) {
    if (c->persist_kind == kind) return PFB_OK;
    if (c->persist_kind) {
        const int r = persist_stop(c);
        if (r) return r;
    }
    if (!c->persist_stream) {
        CK(cudaStreamCreateWithFlags(&c->persist_stream, cudaStreamNonBlocking));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->persist_ctl), 64, cudaHostAllocMapped));
        memset(c->persist_ctl, 0, 64);
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->persist_ctl_dev), c->persist_ctl, 0));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->persist_box), sizeof(PersistBox), cudaHostAllocMapped));
        memset(c->persist_box, 0, sizeof(PersistBox));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->persist_box_dev), c->persist_box, 0));
        CK(cudaMalloc(&c->persist_args, (size_t)kMaxArgChunks * kArgChunk));
        CK(cudaMalloc(&c->persist_chunks, sizeof(unsigned int) * (1 + kMaxArgChunks)));
        CK(cudaMalloc(&c->persist_go, 4 * sizeof(unsigned long long)));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->persist_trace), 8 * sizeof(unsigned long long),
                         cudaHostAllocMapped));
        memset(c->persist_trace, 0, 8 * sizeof(unsigned long long));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->persist_trace_dev), c->persist_trace, 0));
        c->persist_shadow.reset(new unsigned char[(size_t)kMaxArgChunks * kArgChunk]());
    }
    // work queued on the context stream finishes before the kernel takes the SMs
    CK(cudaStreamSynchronize(c->stream));
    unsigned long long go[4] = {c->persist_ctl[0], 0ull, 0ull, 0ull};
    CK(cudaMemcpyAsync(c->persist_go, go, sizeof(go), cudaMemcpyHostToDevice, c->persist_stream));
    PersistCtl P;
    P.host_seq = c->persist_ctl_dev;
    P.host_args = c->persist_box_dev;
    P.dev_chunks = c->persist_chunks;
    P.dev_args = c->persist_args;
    P.go = c->persist_go;
    P.start_seq = c->persist_ctl[0];
    P.idle_ns = kPersistIdleNs;
    P.trace = getenv("PFB_PERSIST_TRACE") ? c->persist_trace_dev : nullptr;
    CK(launch_persist_kind(kind, P, c->persist_stream, c->sm_count));
    ++c->launches;
    c->persist_kind = kind;
    c->persist_shadow_valid = false;  // a new kernel holds no arguments yet
    return PFB_OK;
}

// Mailbox for `A`: the 128-byte chunks that differ from what the kernel holds.
static void persist_post_args(pfb_ctx* c, const NllArgs& A) {
    const unsigned char* a = reinterpret_cast<const unsigned char*>(&A);
    unsigned char* sh = c->persist_shadow.get();
    PersistBox* box = c->persist_box;
    constexpr int kChunks = (int)((sizeof(NllArgs) + kArgChunk - 1) / kArgChunk);
    unsigned int n = 0;
    for (int k = 0; k < kChunks; ++k) {
        const size_t off = (size_t)k * kArgChunk;
        const size_t len = std::min((size_t)kArgChunk, sizeof(NllArgs) - off);
        if (c->persist_shadow_valid && memcmp(sh + off, a + off, len) == 0) continue;
        memcpy(sh + off, a + off, len);
        memcpy(box->payload[n], a + off, len);
        box->idx[n] = (unsigned int)k;
        ++n;
    }
    box->nchunks = n;
    c->persist_shadow_valid = true;
}

// One call through the resident kernel.  Returns 1 (nothing done) when the
// call cannot take this path: the caller then runs the ordinary launch.
static int objective_eval_persistent(pfb_objective* o, double* out_nll, pfb_err* out_err) {
    pfb_ctx* c = o->ctx;
    pfb_plan* p = o->plan;
    const pfb_store* st = o->store;
    if (c->timing || !c->res_mapped || !range_aligned(p, st, o->begin)) return 1;
    const int64_t nb = (o->end - o->begin + kBlock - 1) / kBlock;
    if (c->fix_cap < nb || c->fold_cap < nb) {  // (re)allocation synchronises the device: not under the resident kernel
        int rc = persist_stop(c);
        if (rc) return rc;
        rc = ensure_fix(c, nb);
        if (rc) return rc;
    }
    NllArgs& A = o->args;
    const int frac = pack_args(p, st, o->begin, o->end, o->values.data(), o->norms.data(), &A);
    const int kind = persist_kind(A, sop_ncols(p));
    if (!kind) return 1;
    if (c->persist_kind != kind) {
        const int rc = persist_start(c, kind);
        if (rc) return rc;
    }
    const long long seq = ++c->call_seq;
    A.seq = seq;
    persist_post_args(c, A);
    c->persist_ctl[1] = 0;  // op: run
    std::atomic_thread_fence(std::memory_order_seq_cst);
    reinterpret_cast<volatile unsigned long long*>(c->persist_ctl)[0] = (unsigned long long)seq;
    // wait for the posted result (post_seq); a kernel that left (idle exit) is restarted
    volatile long long* flag = c->res_host + 4;
    for (unsigned spins = 1;; ++spins) {
        if (*flag == seq) break;
        if ((spins & 4095u) == 0u) {
            const cudaError_t e = cudaStreamQuery(c->persist_stream);
            if (e == cudaErrorNotReady) continue;
            if (e != cudaSuccess) return cuda_fail(e);
            if (*flag == seq) break;
            // the kernel is gone without this call's result: start again from
            // the previous doorbell value, so the pending one is served
            c->persist_kind = 0;
            c->persist_ctl[0] = (unsigned long long)(seq - 1);
            int rc = persist_start(c, kind);
            if (rc) return rc;
            persist_post_args(c, A);
            std::atomic_thread_fence(std::memory_order_seq_cst);
            reinterpret_cast<volatile unsigned long long*>(c->persist_ctl)[0] = (unsigned long long)seq;
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (c->res_host[0] > 0) {  // deferred blocks: stop, exact fix-up on the context stream
        int rc = persist_stop(c);
        if (rc) return rc;
        NllArgs F = A;
        F.seq = 0;
        rc = launch_fixup(c, F, c->res_dev + kResHead);
        if (rc) return rc;
        rc = wait_result(c, F.seq);
        if (rc) return rc;
    }
    const unsigned long long key = (unsigned long long)c->res_host[1];
    const int code = decode_error(c, p, A, key, frac, 0, out_err);
    if (code) return code;
    const int st_round = round_result(c, out_nll);
    if (st_round && out_err) out_err->code = st_round;
    return st_round;
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
        if (k == PFB_NORM_QUADRATURE) {
            const pfb_plan* qp = o->node[i].quad_plan;
            if (!qp || !o->node[i].quad_rule || qp->ctx != c || qp->nodes.size() != 1 ||
                qp->nraw != p->nodes[i].nparam)
                return PFB_E_INVALID_ARGUMENT;
        }
        if (k < PFB_NORM_CONST || k > PFB_NORM_QUADRATURE) return PFB_E_INVALID_ARGUMENT;
    }
    o->values.assign(p->nraw, 0.0);
    o->norms.assign(nn, 1.0);
    o->last_in.resize(nn);
    o->have.assign(nn, 0);
    o->pend.assign(nn, -1);
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
    if (o->persistent) {
        const int r = objective_eval_persistent(o, out_nll, out_err);
        if (r != 1) return r;
    }
    return nll_common(o->ctx, o->plan, o->store, o->begin, o->end, 0, o->values.data(), o->plan->nraw,
                      o->norms.data(), (int32_t)o->norms.size(), nullptr, 0, out_nll, out_err);
}

int pfb_objective_eval_batch(pfb_objective* o, const double* xs, int32_t npts, int32_t nfree, double* out_nll,
                             pfb_err* out_err) {
    if (!o || !xs || nfree != o->nfree || !out_nll || !out_err || npts < 1 || npts > kMaxPts)
        return PFB_E_INVALID_ARGUMENT;
    const int nraw = o->plan->nraw, nn = (int)o->norms.size();
    std::vector<double> vals((size_t)npts * nraw), nv((size_t)npts * nn);
    int nquad = 0;
    for (const auto& nd : o->node) nquad += nd.norm_kind == PFB_NORM_QUADRATURE;
    QuadBatch qb;
    QuadBatch* qbp = nquad && nquad <= kMaxPts && !o->persistent ? &qb : nullptr;
    if (qbp) {
        CK(cudaSetDevice(o->ctx->device));
        PFB_QUIESCE(o->ctx);
    }
    int first_bad = npts;  // sequential semantics: nothing after the first host failure
    int fail_m = npts;
    pfb_err fail_err;
    for (int m = 0; m < npts; ++m) {
        clear_err(out_err + m);
        if (qbp && (int)qb.req.size() + nquad > kMaxPts) {  // keep a slot per quadrature node free
            const int rc = quad_flush(o, qbp, nv.data(), &fail_m, &fail_err);
            if (rc > 0) return rc;
            if (rc < 0) break;
        }
        const int st = obj_fill(o, xs + (size_t)m * nfree, out_err + m, qbp, m);
        if (st >= PFB_E_INVALID_ARGUMENT) return st;
        if (st) {
            first_bad = m;
            break;
        }
        std::copy(o->values.begin(), o->values.end(), vals.begin() + (size_t)m * nraw);
        std::copy(o->norms.begin(), o->norms.end(), nv.begin() + (size_t)m * nn);
        if (qbp)
            for (int i = 0; i < nn; ++i)
                if (o->pend[i] >= 0) qb.use.push_back({m, i, o->pend[i]});
    }
    if (qbp && fail_m == npts) {
        const int rc = quad_flush(o, qbp, nv.data(), &fail_m, &fail_err);
        if (rc > 0) return rc;
    }
    if (fail_m < npts && fail_m <= first_bad) {  // a quadrature norm failed first (in sequential order)
        if (first_bad < npts) clear_err(out_err + first_bad);
        first_bad = fail_m;
        out_err[fail_m] = fail_err;
    }
    if (first_bad > 0) {
        const int code = pfb_nll_batch(o->ctx, o->plan, o->store, o->begin, o->end, 0, vals.data(), first_bad,
                                       nraw, nv.data(), nn, out_nll, out_err);
        if (code >= PFB_E_INVALID_ARGUMENT) return code;
    }
    return PFB_OK;
}

int pfb_objective_set_persistent(pfb_objective* o, int32_t on) {
    if (!o) return PFB_E_INVALID_ARGUMENT;
    o->persistent = on ? 1 : 0;
    if (!on) return persist_stop(o->ctx);
    return PFB_OK;
}

int pfb_ctx_persist_trace(pfb_ctx* c, uint64_t* out5) {
    if (!c || !out5) return PFB_E_INVALID_ARGUMENT;
    for (int i = 0; i < 5; ++i) out5[i] = c->persist_trace ? c->persist_trace[i] : 0;
    return PFB_OK;
}

int pfb_ctx_persist_stop(pfb_ctx* c) {
    if (!c) return PFB_E_INVALID_ARGUMENT;
    return persist_stop(c);
}

int pfb_objective_destroy(pfb_objective* o) {
    if (o && o->persistent) persist_stop(o->ctx);
    delete o;
    return PFB_OK;
}

}  // extern "C"
