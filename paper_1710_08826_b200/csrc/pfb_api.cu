// pfb_api.cu -- C ABI: contexts, device event stores, plan compilation,
// per-call argument packing, error decoding and the Dalitz grid object.
#include <atomic>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <memory>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <unistd.h>

#include "pfb_internal.cuh"

namespace pfb {
cudaError_t launch_nll(const NllArgs& A, cudaStream_t stream, int sm_count, int nc);
cudaError_t launch_fix(const NllArgs& A, cudaStream_t stream, int sm_count);
int persist_kind(const NllArgs& A, int nc);
cudaError_t launch_persist_kind(int kind, const PersistCtl& P, cudaStream_t stream, int sm_count);
bool sop_batched_in_kernel(const NllArgs& A, int nc);
bool dal_batched_in_kernel(const NllArgs& A);
cudaError_t launch_export(unsigned long long* acc, long long* out, long long* result_i,
                          unsigned long long* fix_counter, unsigned long long* errkey,
                          cudaStream_t stream);
cudaError_t launch_probe(const NllArgs& A, int64_t j, double* out, cudaStream_t stream);
cudaError_t launch_bin_fill(const BinAxes& B, int64_t begin, int64_t n, unsigned long long* counts,
                            cudaStream_t stream, int sm_count);
cudaError_t launch_binned_nll(const NllArgs& A, const double* contents, int64_t nbins, double total,
                              double volume, unsigned long long* expkey, cudaStream_t stream, int sm_count);
cudaError_t launch_quadrature(const NllArgs& A, const double* weights, int64_t n, cudaStream_t stream,
                              int sm_count);
cudaError_t launch_binned_probe(const NllArgs& A, int64_t b, double total, double volume, double* out,
                                cudaStream_t stream);
cudaError_t launch_fp64_peak(double* out, int blocks, int threads, int iters, cudaStream_t stream);
cudaError_t launch_spin_flush(long long cycles, const double* buf, int64_t bytes, double* sink, int sm_count,
                              cudaStream_t stream);
int npy_parse(int fd, int64_t* n_out, int64_t* data_off);
cudaError_t launch_overhead_probe(int mode, const NllArgs& A, double* sink, cudaStream_t stream);
cudaError_t launch_read_bw(int mode, const double* buf, int64_t bytes, int chunk_kb, double* sink,
                           unsigned long long* counter, int sm_count, cudaStream_t stream);
cudaError_t launch_range_check(const double* x, int64_t n, double lo, double hi, unsigned long long* first,
                               cudaStream_t stream, int sm_count);
cudaError_t launch_peer_allreduce(long long* const* mbox, int world, int rank, unsigned long long seq,
                                  long long timeout_cycles, long long* acc, unsigned long long* status,
                                  cudaStream_t stream);
size_t peer_mailbox_bytes();
int peer_max();
struct PcgParams;
struct PcgHostResult {
    int status;
    int64_t attempts, accepted, in_boundary, produced;
    double observed;
    int64_t ambiguous;
};
cudaError_t pcg_generate_entry(const NllArgs& A, int dalitz, const double* box, double envelope,
                               const GridConsts* g, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                               uint64_t inc_lo, int64_t n_wanted, int64_t budget, double* out0, double* out1,
                               cudaStream_t stream, PcgHostResult* R);
cudaError_t pcg_scan_1d(const NllArgs& A, double lo, double hi, int64_t points, double* out_max,
                        unsigned long long* scratch, cudaStream_t stream, int sm_count);
cudaError_t pcg_scan_dalitz(const NllArgs& A, const GridConsts& g, double* out_max, unsigned long long* scratch,
                            cudaStream_t stream, int sm_count);
cudaError_t launch_grid_mask(const GridConsts& g, uint8_t* mask, int* row_count, cudaStream_t st);
cudaError_t launch_grid_compact(const GridConsts& g, const uint8_t* mask, const int* row_offset,
                                double* p12, double* p13, cudaStream_t st);
cudaError_t launch_grid_amp(const DalDesc& D, const DalTerm& T, const double* p12,
                            const double* p13, int64_t n, double2* out, cudaStream_t st,
                            int sm_count);
cudaError_t launch_grid_overlap(const double2* amps, int64_t n, const int2* pairs, int npairs,
                                unsigned long long* acc, cudaStream_t st, int sm_count);
cudaError_t launch_lineshape_cache(const DalDesc& D, const DalTerm& T, const double* s12,
                                   const double* s13, int64_t n, double2* row, cudaStream_t st,
                                   int sm_count);
cudaError_t launch_gen_1d(const Gen1D& G, int64_t n, double* x, double* y, cudaStream_t st, int sm);
cudaError_t run_gen_dalitz(const GenDalitz& G, int64_t n, double* s12, double* s13, cudaStream_t st,
                           int sm, int64_t* candidates_used);
}  // namespace pfb

using namespace pfb;

#define CK(call)                                  \
    do {                                          \
        cudaError_t e_ = (call);                  \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

static int cuda_fail(cudaError_t e) {
    if (e == cudaErrorMemoryAllocation) return PFB_E_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return PFB_E_NO_DEVICE;
    fprintf(stderr, "pfb200: CUDA error %d: %s\n", (int)e, cudaGetErrorString(e));
    return PFB_E_CUDA;
}

static constexpr int kStoreMaxCols = 16;
// result words: a head, one exported accumulator per point, then the heads of
// the quadrature slots (quad_enqueue: up to kMaxPts launches behind one wait)
static constexpr int kResHead = 5;  // [0] deferred-block count, [1] error key, [2] [3] fused exchange
                                    // status, [4] completion sequence (post_seq)
static constexpr int kResQuad = kResHead + kMaxPts * PFB_ACC_WORDS;  // + one accumulator per point
static constexpr int kResWords = kResQuad + kMaxPts * 4;             // + {count, error key} per slot
enum { MODE_EXPORT = 0, MODE_ADD_EXPORT = 1, MODE_ACCUM = 2 };

static constexpr int64_t kIoChunk = 4 << 20;  // doubles per staging buffer (32 MB)
static constexpr int kDlLanes = 8;            // host threads of a large pageable download
static constexpr int64_t kDlChunk = 1 << 20;  // doubles per lane staging buffer (8 MB)

struct pfb_ctx {
    int device = 0;
    int sm_count = 148;
    int clock_khz = 1965000;  // SM clock for the bounded peer waits (queried once)
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    int warps_override = 0;
    int pipeline = 1;  // 1: TMA bulk-copy pipeline where available
    unsigned long long* acc = nullptr;
    unsigned int* ticket = nullptr;
    unsigned long long* work_counter = nullptr;
    unsigned long long* errkey = nullptr;
    double* tail_scratch = nullptr;
    // result words (error key, deferred count, exported accumulator): pinned
    // host memory mapped into the device, so the finishing CTA writes the
    // result straight to the host and a call needs no device-to-host copy
    long long* res_dev = nullptr;   // kResWords, device view
    long long* res_host = nullptr;  // kResWords, host view
    bool res_mapped = false;
    long long call_seq = 0;  // completion sequence numbers posted by the exporting CTA
    unsigned long long* fix_counter = nullptr;
    int64_t* fix_list = nullptr;
    double* gfold = nullptr;       // task kernel: cross-CTA block fold slots (fix_cap blocks)
    int* gbad = nullptr;
    unsigned int* gcnt = nullptr;  // zeroed once, self-resetting
    int64_t fix_cap = 0;
    int64_t fold_cap = 0;
    double* bsums = nullptr;
    int64_t bsums_cap = 0;
    double* probe_dev = nullptr;
    int64_t launches = 0;
    bool timing = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_ms = 0.f;
    // last partial launch, for error decoding
    std::unique_ptr<NllArgs> last_args;
    std::unique_ptr<NllArgs> enqueue_args;  // pfb_nll_enqueue's packing buffer
    const pfb_plan* last_plan = nullptr;
    int64_t last_index_offset = 0;
    int last_frac_rank = -1;
    // end-to-end staging
    double* e2e_dev[kMaxCols] = {nullptr, nullptr, nullptr, nullptr};
    int64_t e2e_cap = 0;
    std::vector<cudaEvent_t> chunk_events;
    // cross-GPU accumulator exchange over peer memory (pfb_peer_*)
    int peer_world = 0, peer_rank = 0;
    long long* peer_ptr[16] = {};
    bool peer_ipc[16] = {};
    unsigned long long peer_seq = 0;
    unsigned long long* peer_status = nullptr;
    // file ingest staging (pfb_store_load_npy)
    double* io_pinned[2] = {nullptr, nullptr};
    cudaEvent_t io_event[2] = {nullptr, nullptr};
    // parallel download lanes (pfb_store_download to pageable memory)
    double* dl_pinned[kDlLanes][2] = {};
    cudaStream_t dl_stream[kDlLanes] = {};
    // persistent NLL kernel (pfb_nll_task.cuh): doorbell + mailbox in mapped
    // pinned memory, their device copies, the kernel's own stream
    int persist_kind = 0;                  // kind of the resident kernel (0: none)
    cudaStream_t persist_stream = nullptr;
    unsigned long long* persist_ctl = nullptr;      // host view [seq, op]
    unsigned long long* persist_ctl_dev = nullptr;  // device view of the same
    PersistBox* persist_box = nullptr;              // host view of the mailbox
    PersistBox* persist_box_dev = nullptr;
    NllArgs* persist_args = nullptr;                // device copy (kMaxArgChunks x 128 B)
    unsigned int* persist_chunks = nullptr;         // device: count + changed chunk indices
    std::unique_ptr<unsigned char[]> persist_shadow;  // the NllArgs bytes the kernel holds
    bool persist_shadow_valid = false;
    unsigned long long* persist_go = nullptr;       // device [seq, op]
    unsigned long long* persist_trace = nullptr;    // mapped %globaltimer stamps of the last call (host view)
    unsigned long long* persist_trace_dev = nullptr;
    // binned data scratch
    void* bin_dev = nullptr;  // bin counts / contents
    int64_t bin_cap = 0;      // bytes
    unsigned long long* bin_key = nullptr;
    // binned contents on the device and the host copy they were uploaded from
    // (a fit calls binned_nll with the same contents every step)
    double* bin_cont = nullptr;
    int64_t bin_cont_cap = 0;
    std::vector<double> bin_cont_host;
};


struct pfb_store {
    pfb_ctx* ctx = nullptr;
    int32_t ncols = 0;
    int64_t n = 0;
    double* cols[kStoreMaxCols] = {};
    bool owned = false;
    bool pooled = false;  // columns from the device's stream-ordered pool
    // content generation: a fresh process-wide number whenever the columns
    // may have changed (create, upload, load, generate, writable pointer
    // handed out).  Caches of per-event data (the Dalitz lineshape cache)
    // key on it, never on the store's address, which the allocator recycles.
    uint64_t gen = 0;
};

static std::atomic<uint64_t> g_store_gen{0};
static inline void store_touched(pfb_store* s) { s->gen = ++g_store_gen; }

struct TermFactor {
    int type;  // 0: weight (node, child index), 1: 1/norm(node)
    int node;
    int child;
};
struct TermStruct {
    uint32_t emask = 0, vmask = 0;
    std::vector<TermFactor> factors;
};

struct pfb_plan {
    pfb_ctx* ctx = nullptr;
    std::vector<pfb_node> nodes;
    std::vector<pfb_dalitz_desc> dal;
    std::vector<std::vector<int>> children;
    std::vector<int> raw_off;       // offset of each node's raw values
    std::vector<int> der_off;       // offset of each node's derived (literal) values
    std::vector<int> rank;          // first check rank per node (-1 none)
    std::vector<int> frac_rank;     // add-node fraction check rank (-1)
    int nraw = 0, nder = 0;
    int final_rank = 0;
    int nslots = 0;
    int slot_col[kMaxCols] = {0, 0, 0, 0};
    std::vector<int> node_slot0, node_slot1;
    int evaluator = EV_LITERAL;
    int dal_node = -1;
    // sum of products
    std::vector<int> leaf_nodes;
    std::vector<TermStruct> terms;
    // lineshape cache
    int lineshape_mode = 0;
    double2* cache = nullptr;
    int64_t cache_cap = 0;
    uint64_t cache_gen = 0;  // pfb_store::gen the cache was computed from (0: none)
    int64_t cache_begin = -1, cache_end = -1;
    bool cache_valid[kMaxDal] = {};
    double cache_mw[kMaxDal][2] = {};
    int64_t cache_recomputes = 0;
};

struct pfb_grid {
    pfb_ctx* ctx = nullptr;
    pfb_dalitz_desc desc{};
    GridConsts g{};
    int64_t n_inside = 0;
    double area = 0.0;
    uint8_t* mask = nullptr;
    double* p12 = nullptr;
    double* p13 = nullptr;
    double2* amps = nullptr;
    int amps_rows = 0;
};

// The persistent kernel owns every SM while it is resident: any other device
// work first stops it (it is restarted by the next persistent call).
static int persist_stop(pfb_ctx* c) {
    if (!c->persist_kind) return PFB_OK;
    c->persist_kind = 0;
    c->persist_ctl[1] = 1;  // op: stop
    std::atomic_thread_fence(std::memory_order_seq_cst);
    reinterpret_cast<volatile unsigned long long*>(c->persist_ctl)[0] = (unsigned long long)(++c->call_seq);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    CK(cudaStreamSynchronize(c->persist_stream));
    return PFB_OK;
}
#define PFB_QUIESCE(c)                              \
    do {                                            \
        if ((c)->persist_kind) {                    \
            const int q_ = persist_stop(c);         \
            if (q_) return q_;                      \
        }                                           \
    } while (0)

// ---------------------------------------------------------------------------
extern "C" {

int pfb_version(void) { return PFB_ABI_VERSION; }

const char* pfb_strerror(int code) {
    switch (code) {
        case PFB_OK: return "ok";
        case PFB_E_NONPOSITIVE_DENSITY: return "non-positive density";
        case PFB_E_NONFINITE_DENSITY: return "non-finite density";
        case PFB_E_NEGATIVE_DENSITY: return "negative density";
        case PFB_E_FRACTION_OUT_OF_RANGE: return "fraction out of range";
        case PFB_E_EMPTY_DATASET: return "empty dataset";
        case PFB_E_NONPOSITIVE_NORM: return "non-positive normalisation";
        case PFB_E_DEGENERATE_GRID: return "degenerate grid";
        case PFB_E_INVALID_SUM: return "-inf + inf in exact sum";
        case PFB_E_NONPOSITIVE_EXPECTATION: return "non-positive binned expectation";
        case PFB_E_ENVELOPE_HIT: return "density above the generation envelope";
        case PFB_E_ATTEMPTS_EXHAUSTED: return "generation attempts exhausted";
        case PFB_E_PEER_TIMEOUT: return "peer rank did not post its accumulator";
        case PFB_E_UNBOUNDED_OBSERVABLE: return "normalisation over an unbounded observable";
        case PFB_E_OUT_OF_BOUNDS: return "parameter outside its bounds";
        case PFB_E_INVALID_ARGUMENT: return "invalid argument";
        case PFB_E_UNSUPPORTED_PLAN: return "unsupported plan";
        case PFB_E_CUDA: return "CUDA error";
        case PFB_E_NO_DEVICE: return "no CUDA device";
        case PFB_E_OUT_OF_MEMORY: return "out of device memory";
        default: return "unknown status";
    }
}

int pfb_device_count(int* out) {
    if (!out) return PFB_E_INVALID_ARGUMENT;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = 0;
        return PFB_OK;
    }
    *out = n;
    return PFB_OK;
}

int pfb_ctx_create(int device, pfb_ctx** out) {
    if (!out) return PFB_E_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        return PFB_E_NO_DEVICE;
    }
    if (device < 0 || device >= n) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(device));
    auto* c = new pfb_ctx();
    c->device = device;
    CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&c->clock_khz, cudaDevAttrClockRate, device));
    {
        // keep freed pool memory for reuse by later stores (see pfb_store_create)
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
        uint64_t keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    CK(cudaMalloc(&c->acc, sizeof(unsigned long long) * kMaxPts * PFB_ACC_WORDS));
    CK(cudaMemset(c->acc, 0, sizeof(unsigned long long) * kMaxPts * PFB_ACC_WORDS));
    CK(cudaMalloc(&c->ticket, sizeof(unsigned int)));
    CK(cudaMemset(c->ticket, 0, sizeof(unsigned int)));
    CK(cudaMalloc(&c->work_counter, sizeof(unsigned long long)));
    CK(cudaMemset(c->work_counter, 0, sizeof(unsigned long long)));
    CK(cudaMalloc(&c->errkey, sizeof(unsigned long long)));
    CK(cudaMemset(c->errkey, 0xff, sizeof(unsigned long long)));
    CK(cudaMalloc(&c->tail_scratch, sizeof(double) * kBlock));
    CK(cudaMalloc(&c->fix_counter, sizeof(unsigned long long)));
    CK(cudaMemset(c->fix_counter, 0, sizeof(unsigned long long)));
    CK(cudaMalloc(&c->probe_dev, sizeof(double) * 2));
#ifndef PFB_RES_DEVICE
    CK(cudaHostAlloc(&c->res_host, sizeof(long long) * kResWords, cudaHostAllocMapped));
    memset(c->res_host, 0, sizeof(long long) * kResWords);
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->res_dev), c->res_host, 0));
    c->res_mapped = true;
#else
    CK(cudaMalloc(&c->res_dev, sizeof(long long) * kResWords));
    CK(cudaMemset(c->res_dev, 0, sizeof(long long) * kResWords));
    CK(cudaMallocHost(&c->res_host, sizeof(long long) * kResWords));
#endif
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    *out = c;
    return PFB_OK;
}

int pfb_ctx_destroy(pfb_ctx* c) {
    if (!c) return PFB_OK;
    cudaSetDevice(c->device);
    persist_stop(c);
    if (c->persist_stream) {
        cudaStreamDestroy(c->persist_stream);
        cudaFreeHost(c->persist_ctl);
        cudaFreeHost(c->persist_box);
        cudaFree(c->persist_args);
        cudaFree(c->persist_go);
        cudaFree(c->persist_chunks);
        cudaFreeHost(c->persist_trace);
    }
    cudaStreamSynchronize(c->stream);
    cudaFree(c->acc);
    cudaFree(c->ticket);
    cudaFree(c->work_counter);
    cudaFree(c->errkey);
    cudaFree(c->tail_scratch);
    if (!c->res_mapped) cudaFree(c->res_dev);
    cudaFree(c->fix_counter);
    cudaFree(c->fix_list);
    cudaFree(c->gfold);
    cudaFree(c->gbad);
    cudaFree(c->gcnt);
    cudaFree(c->probe_dev);
    cudaFree(c->bsums);
    cudaFree(c->bin_dev);
    cudaFree(c->bin_key);
    cudaFree(c->bin_cont);
    for (int q = 0; q < 16; ++q) {
        if (c->peer_ipc[q] && c->peer_ptr[q]) cudaIpcCloseMemHandle(c->peer_ptr[q]);
    }
    if (c->peer_world) cudaFree(c->peer_ptr[c->peer_rank]);
    cudaFree(c->peer_status);
    for (int b = 0; b < 2; ++b) {
        if (c->io_pinned[b]) cudaFreeHost(c->io_pinned[b]);
        if (c->io_event[b]) cudaEventDestroy(c->io_event[b]);
    }
    for (int t = 0; t < kDlLanes; ++t) {
        for (int b = 0; b < 2; ++b)
            if (c->dl_pinned[t][b]) cudaFreeHost(c->dl_pinned[t][b]);
        if (c->dl_stream[t]) cudaStreamDestroy(c->dl_stream[t]);
    }
    for (auto& p : c->e2e_dev) cudaFree(p);
    for (auto& e : c->chunk_events) cudaEventDestroy(e);
    cudaFreeHost(c->res_host);
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    cudaStreamDestroy(c->own_stream);
    cudaStreamDestroy(c->copy_stream);
    delete c;
    return PFB_OK;
}

int pfb_ctx_set_stream(pfb_ctx* c, void* s) {
    if (!c) return PFB_E_INVALID_ARGUMENT;
    c->stream = s ? (cudaStream_t)s : c->own_stream;
    return PFB_OK;
}

void* pfb_ctx_stream(pfb_ctx* c) { return c ? (void*)c->stream : nullptr; }

int pfb_ctx_synchronize(pfb_ctx* c) {
    if (!c) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    CK(cudaStreamSynchronize(c->stream));
    return PFB_OK;
}

int pfb_ctx_set_warps_per_block(pfb_ctx* c, int w) {
    if (!c || !(w == 0 || w == 1 || w == 2 || w == 4 || w == 8)) return PFB_E_INVALID_ARGUMENT;
    c->warps_override = w;
    return PFB_OK;
}

int pfb_ctx_set_pipeline(pfb_ctx* c, int mode) {
    if (!c || mode < 0 || mode > 4) return PFB_E_INVALID_ARGUMENT;
    c->pipeline = mode;
    return PFB_OK;
}

int pfb_ctx_launch_count(pfb_ctx* c, int64_t* out) {
    if (!c || !out) return PFB_E_INVALID_ARGUMENT;
    *out = c->launches;
    return PFB_OK;
}

int pfb_ctx_enable_timing(pfb_ctx* c, int on) {
    if (!c) return PFB_E_INVALID_ARGUMENT;
    c->timing = on != 0;
    return PFB_OK;
}

int pfb_ctx_last_kernel_ms(pfb_ctx* c, float* out) {
    if (!c || !out) return PFB_E_INVALID_ARGUMENT;
    *out = c->last_ms;
    return PFB_OK;
}

// ---- stores ------------------------------------------------------------------

int pfb_store_create(pfb_ctx* c, int32_t ncols, int64_t n, pfb_store** out) {
    if (!c || !out || ncols < 1 || ncols > kStoreMaxCols || n < 0) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto* s = new pfb_store();
    s->ctx = c;
    s->ncols = ncols;
    s->n = n;
    s->owned = true;
    // pad each column to a whole number of 4096-event blocks (+2 for double2 reads)
    // Columns come from the device's stream-ordered pool (kept, not returned
    // to the driver, see pfb_ctx_create): a toy study that generates, fits and
    // drops a dataset per toy reuses the same HBM instead of paying a fresh
    // cudaMalloc (tens of ms for 100 MB-class buffers) every time.
    const int64_t padded = ((n + kBlock - 1) / kBlock) * kBlock + 2;
    s->pooled = true;
    for (int i = 0; i < ncols; ++i) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&s->cols[i]), sizeof(double) * padded, c->stream);
        if (e != cudaSuccess) {
            for (int j = 0; j < i; ++j) cudaFreeAsync(s->cols[j], c->stream);
            delete s;
            return cuda_fail(e);
        }
    }
    // usable from any stream once this returns
    CK(cudaStreamSynchronize(c->stream));
    store_touched(s);
    *out = s;
    return PFB_OK;
}

int pfb_store_upload(pfb_store* s, int32_t col, const double* host, int64_t offset, int64_t count) {
    if (!s || !host || col < 0 || col >= s->ncols || offset < 0 || count < 0 ||
        offset + count > s->n)
        return PFB_E_INVALID_ARGUMENT;
    // a single pageable copy: the source pages are already resident, and the
    // driver's own staging (~10 GB/s measured) beats host_copy's lanes here
    CK(cudaSetDevice(s->ctx->device));
    PFB_QUIESCE(s->ctx);
    store_touched(s);
    CK(cudaMemcpyAsync(s->cols[col] + offset, host, sizeof(double) * count, cudaMemcpyHostToDevice,
                       s->ctx->stream));
    CK(cudaStreamSynchronize(s->ctx->stream));
    return PFB_OK;
}

int pfb_store_wrap(pfb_ctx* c, int32_t ncols, int64_t n, const double* const* dev_cols,
                   pfb_store** out) {
    if (!c || !out || !dev_cols || ncols < 1 || ncols > kStoreMaxCols || n < 0)
        return PFB_E_INVALID_ARGUMENT;
    auto* s = new pfb_store();
    s->ctx = c;
    s->ncols = ncols;
    s->n = n;
    s->owned = false;
    for (int i = 0; i < ncols; ++i) s->cols[i] = const_cast<double*>(dev_cols[i]);
    store_touched(s);
    *out = s;
    return PFB_OK;
}

int pfb_store_device_ptr(pfb_store* s, int32_t col, void** out) {
    if (!s || !out || col < 0 || col >= s->ncols) return PFB_E_INVALID_ARGUMENT;
    store_touched(s);  // the caller may write through the pointer
    *out = s->cols[col];
    return PFB_OK;
}

int pfb_store_destroy(pfb_store* s) {
    if (!s) return PFB_OK;
    if (s->owned) {
        cudaSetDevice(s->ctx->device);
        for (int i = 0; i < s->ncols; ++i) {
            if (s->pooled)
                cudaFreeAsync(s->cols[i], s->ctx->stream);  // after the work queued on the context
            else
                cudaFree(s->cols[i]);
        }
    }
    delete s;
    return PFB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// plan compilation

static int expected_nparam(const pfb_node& n, const std::vector<pfb_dalitz_desc>& dal) {
    switch (n.kind) {
        case PFB_GAUSSIAN: return 2;
        case PFB_EXPONENTIAL: return 1;
        case PFB_POLYNOMIAL: return n.nparam >= 1 ? n.nparam : -1;
        case PFB_ADD: return n.nchild - 1;
        case PFB_PROD: return 0;
        case PFB_DALITZ:
            if (n.aux < 0 || n.aux >= (int)dal.size()) return -1;
            return 4 * dal[n.aux].nterms;
        default: return -1;
    }
}

static int der_size(const pfb_node& n) {
    switch (n.kind) {
        case PFB_GAUSSIAN: return 2;
        case PFB_EXPONENTIAL: return 1;
        case PFB_POLYNOMIAL: return n.nparam;
        case PFB_ADD: return n.nchild;
        default: return 0;
    }
}

static void assign_ranks(pfb_plan* p, int node, int* r) {
    const pfb_node& n = p->nodes[node];
    switch (n.kind) {
        case PFB_ADD:
            p->frac_rank[node] = (*r)++;
            for (int c : p->children[node]) assign_ranks(p, c, r);
            break;
        case PFB_PROD:
            for (int c : p->children[node]) assign_ranks(p, c, r);
            break;
        case PFB_GAUSSIAN:
        case PFB_EXPONENTIAL:
            p->rank[node] = (*r)++;
            break;
        case PFB_POLYNOMIAL:
            p->rank[node] = *r;
            *r += 2;
            break;
        default:
            break;
    }
}

// Expand a subtree into sum-of-products terms over its leaves (unnormalised
// density of the subtree).
static bool expand(const pfb_plan* p, int node, std::vector<TermStruct>* out) {
    const pfb_node& n = p->nodes[node];
    out->clear();
    if (n.kind == PFB_GAUSSIAN || n.kind == PFB_EXPONENTIAL || n.kind == PFB_POLYNOMIAL) {
        int li = -1;
        for (size_t i = 0; i < p->leaf_nodes.size(); ++i)
            if (p->leaf_nodes[i] == node) li = (int)i;
        if (li < 0) return false;
        TermStruct t;
        if (n.kind == PFB_POLYNOMIAL)
            t.vmask = 1u << li;
        else
            t.emask = 1u << li;
        out->push_back(t);
        return true;
    }
    if (n.kind == PFB_ADD) {
        const auto& ch = p->children[node];
        for (size_t k = 0; k < ch.size(); ++k) {
            std::vector<TermStruct> sub;
            if (!expand(p, ch[k], &sub)) return false;
            for (auto& t : sub) {
                t.factors.push_back({0, node, (int)k});
                t.factors.push_back({1, ch[k], 0});
                out->push_back(t);
            }
            if (out->size() > (size_t)kMaxTerms) return false;
        }
        return true;
    }
    if (n.kind == PFB_PROD) {
        std::vector<TermStruct> cur(1);
        for (int c : p->children[node]) {
            std::vector<TermStruct> sub, next;
            if (!expand(p, c, &sub)) return false;
            for (auto& a : cur)
                for (auto& b : sub) {
                    TermStruct t = a;
                    t.emask |= b.emask;
                    t.vmask |= b.vmask;
                    t.factors.insert(t.factors.end(), b.factors.begin(), b.factors.end());
                    t.factors.push_back({1, c, 0});
                    next.push_back(t);
                }
            if (next.size() > (size_t)kMaxTerms) return false;
            cur.swap(next);
        }
        *out = cur;
        return true;
    }
    return false;
}

extern "C" {

int pfb_plan_compile(pfb_ctx* c, const pfb_node* nodes, int32_t nnodes,
                     const pfb_dalitz_desc* dalitz, int32_t ndalitz, pfb_plan** out) {
    if (!c || !nodes || !out || nnodes < 1 || ndalitz < 0 || (ndalitz > 0 && !dalitz))
        return PFB_E_INVALID_ARGUMENT;
    *out = nullptr;
    if (nnodes > kMaxNodes) return PFB_E_UNSUPPORTED_PLAN;
    auto p = std::make_unique<pfb_plan>();
    p->ctx = c;
    p->nodes.assign(nodes, nodes + nnodes);
    p->dal.assign(dalitz, dalitz + ndalitz);
    for (const auto& d : p->dal)
        if (d.nterms < 1 || d.nterms > kMaxDal) return PFB_E_UNSUPPORTED_PLAN;
    p->children.resize(nnodes);
    p->raw_off.resize(nnodes);
    p->der_off.resize(nnodes);
    p->rank.assign(nnodes, -1);
    p->frac_rank.assign(nnodes, -1);
    p->node_slot0.assign(nnodes, -1);
    p->node_slot1.assign(nnodes, -1);
    std::vector<int> stack;
    int ndal_nodes = 0;
    for (int i = 0; i < nnodes; ++i) {
        const pfb_node& n = p->nodes[i];
        const int np = expected_nparam(n, p->dal);
        if (np < 0 || np != n.nparam) return PFB_E_INVALID_ARGUMENT;
        const bool combo = n.kind == PFB_ADD || n.kind == PFB_PROD;
        if (combo != (n.nchild >= 2)) return PFB_E_INVALID_ARGUMENT;
        if (!combo && n.nchild != 0) return PFB_E_INVALID_ARGUMENT;
        if ((int)stack.size() < n.nchild) return PFB_E_INVALID_ARGUMENT;
        p->children[i].assign(stack.end() - n.nchild, stack.end());
        stack.resize(stack.size() - n.nchild);
        stack.push_back(i);
        p->raw_off[i] = p->nraw;
        p->nraw += n.nparam;
        p->der_off[i] = p->nder;
        p->nder += der_size(n);
        if (n.kind == PFB_DALITZ) {
            ++ndal_nodes;
            p->dal_node = i;
        }
        // observable column slots
        auto slot_of = [&](int col) -> int {
            if (col < 0 || col >= kStoreMaxCols) return -2;
            for (int s = 0; s < p->nslots; ++s)
                if (p->slot_col[s] == col) return s;
            if (p->nslots >= kMaxCols) return -3;
            p->slot_col[p->nslots] = col;
            return p->nslots++;
        };
        if (!combo) {
            const int s0 = slot_of(n.col0);
            if (s0 == -2) return PFB_E_INVALID_ARGUMENT;
            if (s0 == -3) return PFB_E_UNSUPPORTED_PLAN;
            p->node_slot0[i] = s0;
            if (n.kind == PFB_DALITZ) {
                const int s1 = slot_of(n.col1);
                if (s1 == -2) return PFB_E_INVALID_ARGUMENT;
                if (s1 == -3) return PFB_E_UNSUPPORTED_PLAN;
                p->node_slot1[i] = s1;
            }
        }
    }
    if (stack.size() != 1 || stack[0] != nnodes - 1) return PFB_E_INVALID_ARGUMENT;
    if (p->nder > kMaxVals) return PFB_E_UNSUPPORTED_PLAN;
    if (ndal_nodes > 1) return PFB_E_UNSUPPORTED_PLAN;
    int r = 0;
    assign_ranks(p.get(), nnodes - 1, &r);
    p->final_rank = r;

    // evaluator choice
    if (nnodes == 1 && p->nodes[0].kind == PFB_DALITZ) {
        p->evaluator = EV_DALITZ;
        // fast path reads s12 from slot 0 and s13 from slot 1
        if (!(p->node_slot0[0] == 0 && p->node_slot1[0] == 1)) p->evaluator = EV_LITERAL;
    } else if (ndal_nodes == 0) {
        for (int i = 0; i < nnodes; ++i) {
            const int k = p->nodes[i].kind;
            if (k == PFB_GAUSSIAN || k == PFB_EXPONENTIAL || k == PFB_POLYNOMIAL)
                p->leaf_nodes.push_back(i);
        }
        std::vector<TermStruct> terms;
        if ((int)p->leaf_nodes.size() <= kMaxLeaves && expand(p.get(), nnodes - 1, &terms) &&
            (int)terms.size() <= kMaxTerms && !terms.empty()) {
            for (auto& t : terms) t.factors.push_back({1, nnodes - 1, 0});
            p->terms = terms;
            p->evaluator = EV_SOP;
        } else {
            p->evaluator = EV_LITERAL;
        }
    } else {
        p->evaluator = EV_LITERAL;
    }
    *out = p.release();
    return PFB_OK;
}

int pfb_plan_destroy(pfb_plan* p) {
    if (!p) return PFB_OK;
    if (p->cache) {
        cudaSetDevice(p->ctx->device);
        cudaFree(p->cache);
    }
    delete p;
    return PFB_OK;
}

int pfb_plan_evaluator(const pfb_plan* p, int32_t* out) {
    if (!p || !out) return PFB_E_INVALID_ARGUMENT;
    *out = (p->evaluator == EV_DALITZ && p->lineshape_mode == 1) ? EV_DALITZ_CACHED : p->evaluator;
    return PFB_OK;
}

int pfb_plan_set_lineshape_cache(pfb_plan* p, int32_t mode) {
    if (!p || mode < 0 || mode > 2) return PFB_E_INVALID_ARGUMENT;
    p->lineshape_mode = mode;
    return PFB_OK;
}

int pfb_plan_cache_recomputes(const pfb_plan* p, int64_t* out) {
    if (!p || !out) return PFB_E_INVALID_ARGUMENT;
    *out = p->cache_recomputes;
    return PFB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// per-call packing

// numpy's float64 add.reduce for a contiguous array (pairwise_sum in
// numpy/_core/src/umath/loops_utils.h): sequential below 8 elements, eight
// interleaved accumulators up to 128, recursive halving (multiple of 8) above.
static double numpy_sum(const double* a, int n) {
    if (n < 8) {
        double r = n ? a[0] : 0.0;
        for (int i = 1; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return numpy_sum(a, n2) + numpy_sum(a + n2, n - n2);
}

static void build_dal(const pfb_plan* p, const double* values, NllArgs* A) {
    DalDesc& D = A->dal;
    memset(&D, 0, sizeof(D));
    if (p->dal_node < 0) return;
    const pfb_node& n = p->nodes[p->dal_node];
    const pfb_dalitz_desc& d = p->dal[n.aux];
    const double* raw = values + p->raw_off[p->dal_node];
    const double M = d.mother_mass;
    const double M2 = M * M, m1sq = d.m1 * d.m1, m2sq = d.m2 * d.m2, m3sq = d.m3 * d.m3;
    D.K = d.nterms;
    D.mss = ((M2 + m1sq) + m2sq) + m3sq;
    D.zc12 = (M2 - m3sq) * (m2sq - m1sq);
    D.zc13 = (M2 - m2sq) * (m3sq - m1sq);
    D.zc23 = (M2 - m1sq) * (m3sq - m2sq);
    for (int k = 0; k < d.nterms; ++k) {
        DalTerm& T = D.t[k];
        const double m = raw[4 * k], w = raw[4 * k + 1], mag = raw[4 * k + 2], ph = raw[4 * k + 3];
        T.pair = d.pair[k];
        T.spin = d.spin[k];
        T.m2 = m * m;
        T.mg = m * w;
        T.mg2 = T.mg * T.mg;
        T.cre = mag * cos(ph);
        T.cim = mag * sin(ph);
        T.alpha = T.cre * T.m2 - T.cim * T.mg;
        T.beta = T.cre * T.mg + T.cim * T.m2;
        T.cached = 0;
        if (T.spin == 1) {
            if (T.pair == 12 && D.zc12 != 0.0) D.need12 = 1;
            if (T.pair == 13 && D.zc13 != 0.0) D.need13 = 1;
            if (T.pair == 23 && D.zc23 != 0.0) D.need23 = 1;
        }
    }
}

// Sum-of-products tables for parameter point m: the structural leaf/term
// layout (A->leaf, A->term masks) and the point's row A->ptv[m] = leaf values
// (mu, 1/sigma, alpha, coefficients) then (log coef, threshold) per term.  A
// zero weight keeps its term with log coef -inf (exactly 0 in the reference).
// Returns false when the leaf values do not fit a row.
static bool fill_sop_point(const pfb_plan* p, const double* values, const double* norms, NllArgs* A,
                           int m) {
    double* row = A->ptv[m];
    int vo = 0;
    A->nleaf = (int)p->leaf_nodes.size();
    for (int l = 0; l < A->nleaf; ++l) {
        const int ni = p->leaf_nodes[l];
        const pfb_node& n = p->nodes[ni];
        SopLeaf& L = A->leaf[l];
        L.kind = n.kind;
        L.col = p->node_slot0[ni];
        L.voff = vo;
        L.nv = n.kind == PFB_GAUSSIAN ? 2 : (n.kind == PFB_EXPONENTIAL ? 1 : n.nparam);
        if (vo + L.nv > kPtLeafWords) return false;
        const double* raw = values + p->raw_off[ni];
        if (n.kind == PFB_GAUSSIAN) {
            row[vo] = raw[0];
            row[vo + 1] = 1.0 / raw[1];
        } else {
            for (int k = 0; k < L.nv; ++k) row[vo + k] = raw[k];
        }
        vo += L.nv;
    }
    const bool g2_shape = A->nleaf == 2 && A->leaf[0].kind == PFB_GAUSSIAN && A->leaf[1].kind == PFB_EXPONENTIAL;
    if (g2_shape) {
        const double mu = row[0], is = row[1], al = row[2];
        A->g2_c2[m] = (-0.5 * is) * is;
        A->g2_amu[m] = al * mu;
        // certified |w| = |x - mu| < min(256 / |alpha| - |mu|, 1000 sigma): |alpha x| < 256
        // (the reference's exp(alpha x) stays normal) and d >= -5e5 - 512 (the
        // exponential's scale index cannot wrap)
        double lim = fmin(256.0 / fabs(al) - fabs(mu), 1000.0 / is);
        if (!(lim > 0.0)) lim = 0.0;
        uint64_t bits;
        memcpy(&bits, &lim, 8);
        A->g2_wlim[m] = (int32_t)(bits >> 32);
    }
    A->nterm = (int)p->terms.size();
    for (int t = 0; t < A->nterm; ++t) {
        const TermStruct& ts = p->terms[t];
        double logc = 0.0, budget = 0.0;
        bool zero = false;
        for (const auto& f : ts.factors) {
            double v;
            if (f.type == 0) {  // weight f.child of add node f.node (pdf._fractions)
                const double* raw = values + p->raw_off[f.node];
                const int nf = p->nodes[f.node].nchild - 1;
                v = f.child < nf ? raw[f.child] : 1.0 - numpy_sum(raw, nf);
            } else {
                v = 1.0 / norms[f.node];
            }
            if (!(v > 0.0) || !isfinite(v)) {
                zero = true;
                break;
            }
            const double lv = log(v);
            logc += lv;
            budget += fabs(lv);
        }
        SopTerm& T = A->term[t];
        T.emask = ts.emask;
        T.vmask = ts.vmask;
        T.logcoef = zero ? -INFINITY : logc;
        T.coef = zero ? 0.0 : exp(logc);
        T.thr = 690.0 - budget;
        row[kPtLeafWords + 2 * t] = T.logcoef;
        row[kPtLeafWords + 2 * t + 1] = T.thr;
    }
    if (m == 0) A->g2_qcert = 0;
    if (g2_shape && A->nterm == 2) {
        // EvSum2GE: q = c1 + c0 e^d with d = u0 - u1 <= alpha^2 sigma^2 / 2 - alpha mu
        // for every x, and q >= c1: when that range sits inside the unit check's
        // [2^-250, 2^251) no event can leave it and the kernel drops the
        // per-event range tracking (EvSum2GE<true>)
        const double mu = row[0], sg = 1.0 / row[1], al = row[2];
        const double c0 = A->term[0].coef, c1 = A->term[1].coef;
        const double qmax = c1 + c0 * exp(0.5 * (al * al) * (sg * sg) - al * mu);
        const int cert = (c1 >= 0x1p-249 && c0 >= 0.0 && qmax * (1.0 + 1e-6) <= 0x1p249) ? 1 : 0;
        A->g2_qcert = m == 0 ? cert : (A->g2_qcert & cert);
        A->g2_c0[m] = c0;
        A->g2_c1[m] = c1;
    }
    return true;
}

// Fills A from the plan and this call's raw values/norms.  Returns the rank of
// a failing fraction check (host-side, FractionOutOfRange) or -1.
static int pack_args(const pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end,
                     const double* values, const double* norms, NllArgs* A) {
    memset(A, 0, sizeof(NllArgs));
    pfb_ctx* c = p->ctx;
    bool aligned = (begin % 2) == 0;
    for (int s = 0; s < p->nslots; ++s) {
        A->col[s] = st->cols[p->slot_col[s]];
        if (((uintptr_t)A->col[s]) % 16) aligned = false;
    }
    A->ncols = p->nslots;
    A->vec2 = aligned ? 1 : 0;
    A->begin = begin;
    const int64_t n = end - begin;
    A->nfull = n / kBlock;
    A->tail = (int32_t)(n % kBlock);
    A->evaluator = p->evaluator;
    // one 4096-event block per 8-warp group: measured fastest for every
    // evaluator at 1M-10M events (scripts/kernel_sweep.py)
    A->warps = c->warps_override;  // 0: the evaluator's default kernel shape
    A->tma = c->pipeline == 4 ? 1 : c->pipeline;  // 4: pipeline 1 with the warp-task C1 shell
    A->task_shell = c->pipeline == 4;
    A->acc = c->acc;
    A->ticket = c->ticket;
    A->work_counter = c->work_counter;
    A->errkey = c->errkey;
    A->tail_scratch = c->tail_scratch;
    A->acc_out = c->res_dev + kResHead;
    A->result_i = c->res_dev;
    A->fix_counter = c->fix_counter;
    A->fix_list = c->fix_list;
    A->fix_count = c->res_dev;
    A->gfold = c->gfold;
    A->gbad = c->gbad;
    A->gcnt = c->gcnt;
    A->block_base = 0;
    A->mode = MODE_EXPORT;
    A->nops = (int)p->nodes.size();
    A->final_rank = p->final_rank;
    int frac_fail = -1;
    for (int i = 0; i < A->nops; ++i) {
        const pfb_node& n = p->nodes[i];
        LitOp& op = A->ops[i];
        op.kind = n.kind;
        op.nchild = n.nchild;
        op.col0 = p->node_slot0[i] < 0 ? 0 : p->node_slot0[i];
        op.col1 = p->node_slot1[i] < 0 ? 0 : p->node_slot1[i];
        op.voff = p->der_off[i];
        op.nv = der_size(n);
        op.rank = p->rank[i];
        op.dal = 0;
        A->norm[i] = norms[i];
        const double* raw = values + p->raw_off[i];
        double* der = A->v + p->der_off[i];
        switch (n.kind) {
            case PFB_GAUSSIAN:
                der[0] = raw[0];
                der[1] = raw[1];
                break;
            case PFB_EXPONENTIAL:
                der[0] = raw[0];
                break;
            case PFB_POLYNOMIAL:
                for (int k = 0; k < n.nparam; ++k) der[k] = raw[k];
                break;
            case PFB_ADD: {
                // pdf._fractions (pdf.py:205-210)
                const int nf = n.nchild - 1;
                const double rest = 1.0 - numpy_sum(raw, nf);
                bool bad = rest < 0.0;
                for (int k = 0; k < nf; ++k) {
                    der[k] = raw[k];
                    if (raw[k] < 0.0 || raw[k] > 1.0) bad = true;
                }
                der[nf] = rest;
                if (bad && (frac_fail < 0 || p->frac_rank[i] < frac_fail)) frac_fail = p->frac_rank[i];
                break;
            }
            default:
                break;
        }
    }
    build_dal(p, values, A);
    A->inv_norm = 1.0 / norms[A->nops - 1];
    {
        const double sn = sqrt(A->inv_norm);
        for (int k = 0; k < A->dal.K && k < kMaxDal; ++k) {
            DalTerm& T = A->dal.t[k];
            T.scre = T.cre * sn;
            T.scim = T.cim * sn;
            T.salpha = T.alpha * sn;
            T.sbeta = T.beta * sn;
        }
    }
    // sum of products
    A->npts = 1;
    A->fix_point = 0;
    if (p->evaluator == EV_SOP && !fill_sop_point(p, values, norms, A, 0)) A->evaluator = EV_LITERAL;
    return frac_fail;
}

// The kernels stream double2 pairs from an even start of 16-byte aligned
// columns.  Ranges that violate this (odd shard starts of small unaligned
// shards, foreign device pointers) are copied once into context staging.
static bool range_aligned(const pfb_plan* p, const pfb_store* st, int64_t begin) {
    if (begin % 2) return false;
    for (int s = 0; s < p->nslots; ++s)
        if (((uintptr_t)st->cols[p->slot_col[s]]) % 16) return false;
    return true;
}

static int restage(pfb_ctx* c, const pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end,
                   pfb_store* tmp) {
    const int64_t n = end - begin;
    if (c->e2e_cap < n) {
        for (auto& ptr : c->e2e_dev) {
            cudaFree(ptr);
            ptr = nullptr;
        }
        const int64_t padded = ((n + kBlock - 1) / kBlock) * kBlock + 2;
        for (int i = 0; i < kMaxCols; ++i) CK(cudaMalloc(&c->e2e_dev[i], sizeof(double) * padded));
        c->e2e_cap = n;
    }
    tmp->ctx = c;
    tmp->owned = false;
    store_touched(tmp);  // staging holds a different range every call
    tmp->n = n;
    tmp->ncols = st->ncols;
    for (int i = 0; i < kStoreMaxCols; ++i) tmp->cols[i] = nullptr;
    for (int s = 0; s < p->nslots; ++s) {
        const int col = p->slot_col[s];
        tmp->cols[col] = c->e2e_dev[s];
        CK(cudaMemcpyAsync(tmp->cols[col], st->cols[col] + begin, sizeof(double) * n,
                           cudaMemcpyDeviceToDevice, c->stream));
    }
    return PFB_OK;
}

static int sop_ncols(const pfb_plan* p) { return p->nslots < 1 ? 1 : p->nslots; }

static int ensure_cache(pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end,
                        NllArgs* A) {
    pfb_ctx* c = p->ctx;
    const int K = A->dal.K;
    const int64_t n = end - begin;
    if (p->cache_gen != st->gen || p->cache_begin != begin || p->cache_end != end) {
        if (p->cache_cap < (int64_t)K * n) {
            if (p->cache) cudaFree(p->cache);
            p->cache = nullptr;
            p->cache_cap = 0;
            CK(cudaMalloc(&p->cache, sizeof(double2) * (size_t)K * (size_t)(n > 0 ? n : 1)));
            p->cache_cap = (int64_t)K * n;
        }
        p->cache_gen = st->gen;
        p->cache_begin = begin;
        p->cache_end = end;
        for (int k = 0; k < kMaxDal; ++k) p->cache_valid[k] = false;
    }
    for (int k = 0; k < K; ++k) {
        DalTerm& T = A->dal.t[k];
        // shape fingerprint (dalitz.py:108-117): mass and width values
        const double m2 = T.m2, mg = T.mg;
        if (!p->cache_valid[k] || memcmp(&p->cache_mw[k][0], &m2, 8) != 0 ||
            memcmp(&p->cache_mw[k][1], &mg, 8) != 0) {
            CK(launch_lineshape_cache(A->dal, T, A->col[0] + begin, A->col[1] + begin, n,
                                      p->cache + (int64_t)k * n, c->stream, c->sm_count));
            ++c->launches;
            p->cache_valid[k] = true;
            p->cache_mw[k][0] = m2;
            p->cache_mw[k][1] = mg;
            ++p->cache_recomputes;
        }
        T.cached = 1;
    }
    A->dal.cache = p->cache;
    A->dal.cache_stride = n;
    A->evaluator = EV_DALITZ_CACHED;
    return PFB_OK;
}

static int launch_eval(pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end, NllArgs* A,
                       bool allow_cache = true) {
    pfb_ctx* c = p->ctx;
    if (allow_cache && p->evaluator == EV_DALITZ && p->lineshape_mode == 1) {
        const int rc = ensure_cache(p, st, begin, end, A);
        if (rc) return rc;
    }
    if (c->timing) CK(cudaEventRecord(c->ev0, c->stream));
    CK(launch_nll(*A, c->stream, c->sm_count, sop_ncols(p)));
    ++c->launches;
    if (c->timing) CK(cudaEventRecord(c->ev1, c->stream));
    return PFB_OK;
}

// Decode an error key into the reference's exception semantics.
static int decode_error(pfb_ctx* c, const pfb_plan* p, const NllArgs& A, unsigned long long key,
                        int frac_rank, int64_t index_offset, pfb_err* err) {
    pfb_err e;
    e.code = PFB_OK;
    e.node = -1;
    e.index = -1;
    e.value = NAN;
    if (key == ~0ull) {
        if (frac_rank >= 0) e.code = PFB_E_FRACTION_OUT_OF_RANGE;
    } else {
        const int rank = (int)(key >> 40);
        const int64_t local = (int64_t)(key & ((1ull << 40) - 1));
        if (frac_rank >= 0 && frac_rank < rank) {
            e.code = PFB_E_FRACTION_OUT_OF_RANGE;
        } else if (rank == p->final_rank) {
            e.code = PFB_E_NONPOSITIVE_DENSITY;
            e.index = index_offset + local;
        } else {
            for (int i = 0; i < (int)p->nodes.size(); ++i) {
                if (p->rank[i] < 0) continue;
                if (rank == p->rank[i]) {
                    e.code = PFB_E_NONFINITE_DENSITY;
                    e.node = i;
                } else if (p->nodes[i].kind == PFB_POLYNOMIAL && rank == p->rank[i] + 1) {
                    e.code = PFB_E_NEGATIVE_DENSITY;
                    e.node = i;
                }
            }
            e.index = local;
        }
        if (e.code == PFB_E_NONPOSITIVE_DENSITY || e.code == PFB_E_NEGATIVE_DENSITY) {
            // the offending value: re-evaluate that one event literally
            const int64_t j = A.begin + local - A.idx_base;
            CK(launch_probe(A, j, c->probe_dev, c->stream));
            ++c->launches;
            double pv[2];
            CK(cudaMemcpyAsync(pv, c->probe_dev, sizeof(pv), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            e.value = pv[1];
        }
    }
    if (err) *err = e;
    return e.code;
}

static int read_result(pfb_ctx* c, int npts = 1) {
    if (!c->res_mapped)
        CK(cudaMemcpyAsync(c->res_host, c->res_dev, sizeof(long long) * (kResHead + npts * PFB_ACC_WORDS),
                           cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->timing) cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    return PFB_OK;
}

// Wait for a launch whose exporting CTA posts `seq` (NllArgs::seq) into the
// mapped result block: the host spins on that word instead of a stream
// synchronize (no driver round trip on the critical path of a minimiser
// call).  Every 1024 polls the stream is queried, so an error or a launch
// that does not post falls back to the ordinary synchronize.
static bool poll_results() {
    // opt-in: measured no faster than a stream synchronize for one-shot
    // launches, and the post costs the exporting CTA a system fence
    // (profiles/r2_persistent.md); the persistent kernel always posts
    static const bool on = getenv("PFB_POLL") != nullptr;
    return on;
}

static int wait_result(pfb_ctx* c, long long seq) {
    if (c->timing || !c->res_mapped || seq <= 0) return read_result(c);
    volatile long long* flag = c->res_host + 4;
    for (unsigned spins = 1;; ++spins) {
        if (*flag == seq) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return PFB_OK;
        }
        if ((spins & 1023u) == 0u) {
            const cudaError_t e = cudaStreamQuery(c->stream);
            if (e != cudaErrorNotReady) {
                if (e != cudaSuccess) return cuda_fail(e);
                if (*flag != seq) return read_result(c);
            }
        }
    }
}

// Deferred-block list for up to `nentries` (block, point) pairs, and the task
// kernel's cross-CTA fold slots for `nblocks` blocks (one parameter point).
static int ensure_fix(pfb_ctx* c, int64_t nentries, int64_t nblocks = -1) {
    if (nblocks < 0) nblocks = nentries;
    if (c->fix_cap < nentries) {
        cudaFree(c->fix_list);
        c->fix_list = nullptr;
        c->fix_cap = 0;
        CK(cudaMalloc(&c->fix_list, sizeof(int64_t) * (size_t)(nentries > 0 ? nentries : 1)));
        c->fix_cap = nentries;
    }
    if (c->fold_cap < nblocks) {
        cudaFree(c->gfold);
        cudaFree(c->gbad);
        cudaFree(c->gcnt);
        c->gfold = nullptr;
        c->gbad = nullptr;
        c->gcnt = nullptr;
        c->fold_cap = 0;
        const size_t nb = (size_t)(nblocks > 0 ? nblocks : 1);
        CK(cudaMalloc(&c->gfold, sizeof(double) * 8 * 32 * nb));
        CK(cudaMalloc(&c->gbad, sizeof(int) * 8 * nb));
        CK(cudaMalloc(&c->gcnt, sizeof(unsigned int) * nb));
        CK(cudaMemset(c->gcnt, 0, sizeof(unsigned int) * nb));
        c->fold_cap = nblocks;
    }
    return PFB_OK;
}

// Exact fix-up of the blocks a fast launch deferred (listed on the device).
static int launch_fixup(pfb_ctx* c, const NllArgs& A, long long* out) {
    NllArgs F = A;
    F.mode = MODE_ADD_EXPORT;
    F.acc_out = out;
    F.fix_count = c->res_dev;
    CK(launch_fix(F, c->stream, c->sm_count));
    ++c->launches;
    return PFB_OK;
}

// Host rounding of the exported accumulator words in res_host[0..72).
static int round_result(pfb_ctx* c, double* out, int point = 0) {
    double r = 0.0;
    const int st = acc_round(c->res_host + kResHead + point * PFB_ACC_WORDS, &r);
    if (out) *out = r;
    return st;
}

static void clear_err(pfb_err* e) {
    if (!e) return;
    e->code = PFB_OK;
    e->node = -1;
    e->index = -1;
    e->value = NAN;
}

static int nll_common(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int64_t begin,
                      int64_t end, int64_t index_offset, const double* values, int32_t nvalues,
                      const double* norms, int32_t nnorms, double* block_sums_host, int64_t n_out,
                      double* out_nll, pfb_err* out_err) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !values || !norms || p->ctx != c || st->ctx != c)
        return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end < begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    for (int s = 0; s < p->nslots; ++s)
        if (p->slot_col[s] >= st->ncols) return PFB_E_INVALID_ARGUMENT;
    clear_err(out_err);
    if (end == begin) {
        if (out_err) out_err->code = PFB_E_EMPTY_DATASET;
        return PFB_E_EMPTY_DATASET;
    }
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    pfb_store staged;
    const bool restaged = !range_aligned(p, st, begin);
    if (restaged) {
        const int rs = restage(c, p, st, begin, end, &staged);
        if (rs) return rs;
        st = &staged;
        end -= begin;
        begin = 0;
    }
    const int64_t nb = (end - begin + kBlock - 1) / kBlock;
    int rc = ensure_fix(c, nb);
    if (rc) return rc;
    auto A = std::make_unique<NllArgs>();
    const int frac = pack_args(p, st, begin, end, values, norms, A.get());
    if (block_sums_host) {
        if (n_out < nb) return PFB_E_INVALID_ARGUMENT;
        if (c->bsums_cap < nb) {
            cudaFree(c->bsums);
            c->bsums = nullptr;
            CK(cudaMalloc(&c->bsums, sizeof(double) * nb));
            c->bsums_cap = nb;
        }
        A->block_sums = c->bsums;
    }
    A->seq = poll_results() ? ++c->call_seq : 0;
    rc = launch_eval(p, st, begin, end, A.get(), !restaged);
    if (rc) return rc;
    rc = wait_result(c, A->seq);
    if (rc) return rc;
    if (c->res_host[0] > 0) {  // deferred blocks: exact fix-up
        A->seq = poll_results() ? ++c->call_seq : 0;
        rc = launch_fixup(c, *A, c->res_dev + kResHead);
        if (rc) return rc;
        const float fast_ms = c->last_ms;
        rc = wait_result(c, A->seq);
        if (rc) return rc;
        c->last_ms = fast_ms;
    }
    const unsigned long long key = (unsigned long long)c->res_host[1];
    const int code = decode_error(c, p, *A, key, frac, index_offset, out_err);
    if (code) return code;
    if (block_sums_host)
        CK(cudaMemcpy(block_sums_host, c->bsums, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    const int st_round = round_result(c, out_nll);
    if (st_round && out_err) out_err->code = st_round;
    return st_round;
}

extern "C" {

int pfb_nll(pfb_ctx* c, const pfb_plan* p, const pfb_store* st, int64_t begin, int64_t end,
            int64_t index_offset, const double* values, int32_t nvalues, const double* norms,
            int32_t nnorms, double* out_nll, pfb_err* out_err) {
    return nll_common(c, p, st, begin, end, index_offset, values, nvalues, norms, nnorms, nullptr,
                      0, out_nll, out_err);
}

int pfb_nll_block_sums(pfb_ctx* c, const pfb_plan* p, const pfb_store* st, int64_t begin,
                       int64_t end, int64_t index_offset, const double* values, int32_t nvalues,
                       const double* norms, int32_t nnorms, double* out_block_sums, int64_t n_out,
                       pfb_err* out_err) {
    if (!out_block_sums) return PFB_E_INVALID_ARGUMENT;
    return nll_common(c, p, st, begin, end, index_offset, values, nvalues, norms, nnorms,
                      out_block_sums, n_out, nullptr, out_err);
}

int pfb_nll_batch(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int64_t begin, int64_t end,
                  int64_t index_offset, const double* values, int32_t npts, int32_t nvalues,
                  const double* norms, int32_t nnorms, double* out_nll, pfb_err* out_err) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !values || !norms || !out_nll || p->ctx != c || st->ctx != c)
        return PFB_E_INVALID_ARGUMENT;
    if (npts < 1 || npts > kMaxPts) return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end < begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    for (int m = 0; m < npts; ++m) clear_err(out_err ? out_err + m : nullptr);
    if (end == begin) {
        for (int m = 0; m < npts; ++m)
            if (out_err) out_err[m].code = PFB_E_EMPTY_DATASET;
        return PFB_E_EMPTY_DATASET;
    }
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    pfb_store staged;
    if (!range_aligned(p, st, begin)) {
        const int rs = restage(c, p, st, begin, end, &staged);
        if (rs) return rs;
        st = &staged;
        end -= begin;
        begin = 0;
    }
    // the batched kernels list one deferred entry per (block, point) pair
    int rc = ensure_fix(c, (end - begin + kBlock - 1) / kBlock * npts, (end - begin + kBlock - 1) / kBlock);
    if (rc) return rc;
    auto A = std::make_unique<NllArgs>();
    int frac0 = pack_args(p, st, begin, end, values, norms, A.get());
    bool in_kernel = A->evaluator == EV_SOP && sop_batched_in_kernel(*A, sop_ncols(p));
    int first = PFB_OK;
    if (in_kernel) {
        for (int m = 1; m < npts; ++m)
            fill_sop_point(p, values + (int64_t)m * nvalues, norms + (int64_t)m * nnorms, A.get(), m);
        A->npts = npts;
        // every point must meet the batched evaluator's preconditions
        in_kernel = sop_batched_in_kernel(*A, sop_ncols(p));
    }
    if (!in_kernel && npts > 1 && A->evaluator == EV_DALITZ && dal_batched_in_kernel(*A)) {
        // the D0 ratio form: every point's four scaled coefficients per term go
        // into its ptv row -- when the shapes (masses, widths) are point 0's
        static_assert(kPtWords >= 4 * 4, "ptv row holds 4 Dalitz terms x 4 coefficients");
        bool same = true;
        auto Am = std::make_unique<NllArgs>();
        for (int m = 0; m < npts && same; ++m) {
            const NllArgs* S = A.get();
            if (m > 0) {
                pack_args(p, st, begin, end, values + (int64_t)m * nvalues, norms + (int64_t)m * nnorms, Am.get());
                S = Am.get();
            }
            for (int k = 0; k < 4; ++k) {
                const DalTerm& T = S->dal.t[k];
                const DalTerm& T0 = A->dal.t[k];
                if (!(T.m2 == T0.m2 && T.mg == T0.mg && T.mg2 == T0.mg2)) same = false;
                A->ptv[m][4 * k] = T.scre;
                A->ptv[m][4 * k + 1] = T.scim;
                A->ptv[m][4 * k + 2] = T.salpha;
                A->ptv[m][4 * k + 3] = T.sbeta;
            }
        }
        if (same) {
            A->npts = npts;
            in_kernel = true;
        }
    }
    if (in_kernel) {
        // one pass over the data for all points (TMA pipeline kernel)
        rc = launch_eval(p, st, begin, end, A.get(), false);
        if (rc) return rc;
        rc = read_result(c, npts);
        if (rc) return rc;
        const bool deferred = c->res_host[0] > 0;
        std::vector<long long> accs(c->res_host + kResHead, c->res_host + kResHead + npts * PFB_ACC_WORDS);
        for (int m = 0; m < npts; ++m) {
            // point m's literal tables (weights, norms) for the fix-up and errors
            auto Am = std::make_unique<NllArgs>();
            const int frac = m == 0 ? frac0
                                    : pack_args(p, st, begin, end, values + (int64_t)m * nvalues,
                                                norms + (int64_t)m * nnorms, Am.get());
            const NllArgs& Ap = m == 0 ? *A : *Am;
            unsigned long long key = ~0ull;
            if (deferred) {
                NllArgs F = Ap;
                F.fix_point = m;
                rc = launch_fixup(c, F, c->res_dev + kResHead + m * PFB_ACC_WORDS);
                if (rc) return rc;
                rc = read_result(c, npts);
                if (rc) return rc;
                key = (unsigned long long)c->res_host[1];
                std::copy(c->res_host + kResHead + m * PFB_ACC_WORDS,
                          c->res_host + kResHead + (m + 1) * PFB_ACC_WORDS, accs.begin() + m * PFB_ACC_WORDS);
            }
            pfb_err e;
            int code = decode_error(c, p, Ap, key, frac, index_offset, &e);
            double r = 0.0;
            if (!code) code = acc_round(accs.data() + m * PFB_ACC_WORDS, &r);
            out_nll[m] = r;
            e.code = code;
            if (out_err) out_err[m] = e;
            if (code && !first) first = code;
        }
        return first;
    }
    // other evaluators: one fused launch per point, back to back in C++
    for (int m = 0; m < npts; ++m) {
        pfb_err e;
        const int code = nll_common(c, p, st, begin, end, index_offset, values + (int64_t)m * nvalues,
                                    nvalues, norms + (int64_t)m * nnorms, nnorms, nullptr, 0, out_nll + m, &e);
        if (code >= PFB_E_INVALID_ARGUMENT) return code;
        if (out_err) out_err[m] = e;
        if (code && !first) first = code;
    }
    return first;
}

int pfb_nll_enqueue(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int64_t begin, int64_t end,
                    const double* values, int32_t nvalues, const double* norms, int32_t nnorms, int64_t* dev_acc,
                    int64_t* dev_status) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !values || !norms || !dev_acc || !dev_status || p->ctx != c || st->ctx != c)
        return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end <= begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    if (!range_aligned(p, st, begin)) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = ensure_fix(c, (end - begin + kBlock - 1) / kBlock);
    if (rc) return rc;
    NllArgs* A = c->enqueue_args.get();
    if (!A) {
        c->enqueue_args.reset(new NllArgs());
        A = c->enqueue_args.get();
    }
    if (pack_args(p, st, begin, end, values, norms, A) >= 0) return PFB_E_FRACTION_OUT_OF_RANGE;
    A->acc_out = (long long*)dev_acc;
    A->result_i = (long long*)dev_status;
    A->seq = 0;
    return launch_eval(p, st, begin, end, A, true);
}

int pfb_nll_partial_async(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int64_t begin,
                          int64_t end, int64_t index_offset, const double* values,
                          int32_t nvalues, const double* norms, int32_t nnorms, int64_t* dev_acc) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !values || !norms || !dev_acc || p->ctx != c || st->ctx != c)
        return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end < begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    pfb_store staged;
    const bool restaged = end > begin && !range_aligned(p, st, begin);
    if (restaged) {
        const int rs = restage(c, p, st, begin, end, &staged);
        if (rs) return rs;
        st = &staged;
        end -= begin;
        begin = 0;
    }
    int rc = ensure_fix(c, (end - begin + kBlock - 1) / kBlock);
    if (rc) return rc;
    c->last_args.reset(new NllArgs());
    NllArgs* A = c->last_args.get();
    c->last_frac_rank = pack_args(p, st, begin, end, values, norms, A);
    c->last_plan = p;
    c->last_index_offset = index_offset;
    if (end == begin) {  // empty shard: a zero partial (sharding.partial_nll, sharding.py:110-111)
        CK(cudaMemsetAsync(dev_acc, 0, sizeof(int64_t) * PFB_ACC_WORDS, c->stream));
        CK(cudaMemsetAsync(c->res_dev, 0, sizeof(long long), c->stream));
        CK(cudaMemsetAsync(c->res_dev + 1, 0xff, sizeof(long long), c->stream));
        return PFB_OK;
    }
    A->acc_out = (long long*)dev_acc;
    rc = launch_eval(p, st, begin, end, A, !restaged);
    if (rc) return rc;
    // no host round trip: the fix-up launch reads the deferred count on the device
    return launch_fixup(c, *A, (long long*)dev_acc);
}

int pfb_finalize(pfb_ctx* c, const int64_t* dev_acc, double* out_nll, int64_t* out_fails) {
    if (!c || !dev_acc) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    long long h[PFB_ACC_WORDS];
    CK(cudaMemcpyAsync(h, dev_acc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    double r = 0.0;
    const int st = acc_round(h, &r);
    if (out_nll) *out_nll = r;
    // failed events/blocks of every rank, plus this call's fraction check
    // (host-side, so it never reaches the accumulator)
    if (out_fails) *out_fails = (int64_t)h[PFB_ACC_FAILS] + (c->last_frac_rank >= 0 ? 1 : 0);
    return st;
}

int pfb_ctx_last_fraction_failure(pfb_ctx* c, int32_t* out) {
    if (!c || !out) return PFB_E_INVALID_ARGUMENT;
    *out = (c->last_args && c->last_frac_rank >= 0) ? 1 : 0;
    return PFB_OK;
}

int pfb_last_error(pfb_ctx* c, pfb_err* out_err) {
    if (!c || !out_err || !c->last_args) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = read_result(c);
    if (rc) return rc;
    const unsigned long long key = (unsigned long long)c->res_host[1];
    decode_error(c, c->last_plan, *c->last_args, key, c->last_frac_rank, c->last_index_offset,
                 out_err);
    return PFB_OK;
}

int pfb_nll_host(pfb_ctx* c, const pfb_plan* pc, const double* const* host_cols, int32_t ncols,
                 int64_t n, const double* values, int32_t nvalues, const double* norms,
                 int32_t nnorms, double* out_nll, pfb_err* out_err) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !host_cols || ncols < 1 || ncols > kMaxCols || n < 0 || !values || !norms)
        return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    for (int s = 0; s < p->nslots; ++s)
        if (p->slot_col[s] >= ncols) return PFB_E_INVALID_ARGUMENT;
    clear_err(out_err);
    if (n == 0) {
        if (out_err) out_err->code = PFB_E_EMPTY_DATASET;
        return PFB_E_EMPTY_DATASET;
    }
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    if (c->e2e_cap < n) {
        for (auto& ptr : c->e2e_dev) {
            cudaFree(ptr);
            ptr = nullptr;
        }
        const int64_t padded = ((n + kBlock - 1) / kBlock) * kBlock + 2;
        for (int i = 0; i < kMaxCols; ++i) CK(cudaMalloc(&c->e2e_dev[i], sizeof(double) * padded));
        c->e2e_cap = n;
    }
    int rc = ensure_fix(c, (n + kBlock - 1) / kBlock);
    if (rc) return rc;
    pfb_store st;
    st.ctx = c;
    st.ncols = ncols;
    st.n = n;
    for (int i = 0; i < ncols; ++i) st.cols[i] = c->e2e_dev[i];
    // chunks of 256 blocks (1 Mi events); copies on the copy stream, one
    // accumulate-mode launch per landed chunk on the compute stream.
    const int64_t chunk = 256LL * kBlock;
    const int64_t nchunks = (n + chunk - 1) / chunk;
    while ((int64_t)c->chunk_events.size() < nchunks) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->chunk_events.push_back(e);
    }
    // the copy stream must not overwrite staging still read by a previous call
    cudaEvent_t prior;
    CK(cudaEventCreateWithFlags(&prior, cudaEventDisableTiming));
    CK(cudaEventRecord(prior, c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, prior, 0));
    cudaEventDestroy(prior);
    NllArgs A0;
    const int frac = pack_args(p, &st, 0, n, values, norms, &A0);
    for (int64_t k = 0; k < nchunks; ++k) {
        const int64_t b = k * chunk, e = std::min(n, b + chunk);
        for (int s = 0; s < ncols; ++s)
            CK(cudaMemcpyAsync(c->e2e_dev[s] + b, host_cols[s] + b, sizeof(double) * (e - b),
                               cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaEventRecord(c->chunk_events[k], c->copy_stream));
        CK(cudaStreamWaitEvent(c->stream, c->chunk_events[k], 0));
        auto A = std::make_unique<NllArgs>();
        pack_args(p, &st, b, e, values, norms, A.get());
        A->idx_base = b;
        A->block_base = b / kBlock;
        A->mode = MODE_ACCUM;
        rc = launch_eval(p, &st, b, e, A.get(), /*allow_cache=*/false);
        if (rc) return rc;
    }
    CK(launch_export(c->acc, c->res_dev + kResHead, c->res_dev, c->fix_counter, c->errkey,
                     c->stream));
    ++c->launches;
    rc = read_result(c);
    if (rc) return rc;
    if (c->res_host[0] > 0) {
        rc = launch_fixup(c, A0, c->res_dev + kResHead);
        if (rc) return rc;
        rc = read_result(c);
        if (rc) return rc;
    }
    const unsigned long long key = (unsigned long long)c->res_host[1];
    const int code = decode_error(c, p, A0, key, frac, 0, out_err);
    if (code) return code;
    const int st_round = round_result(c, out_nll);
    if (st_round && out_err) out_err->code = st_round;
    return st_round;
}

int pfb_terms_block_sums(pfb_ctx* c, const double* host_terms, int64_t n, double* out_block_sums,
                         double* out_total) {
    if (!c || (!host_terms && n) || n < 0) return PFB_E_INVALID_ARGUMENT;
    if (n == 0) {
        if (out_total) *out_total = 0.0;
        return PFB_OK;
    }
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    pfb_store* st = nullptr;
    int rc = pfb_store_create(c, 1, n, &st);
    if (rc) return rc;
    std::unique_ptr<pfb_store, int (*)(pfb_store*)> guard(st, pfb_store_destroy);
    rc = pfb_store_upload(st, 0, host_terms, 0, n);
    if (rc) return rc;
    const int64_t nb = (n + kBlock - 1) / kBlock;
    rc = ensure_fix(c, nb);
    if (rc) return rc;
    auto A = std::make_unique<NllArgs>();
    memset(A.get(), 0, sizeof(NllArgs));
    A->col[0] = st->cols[0];
    A->ncols = 1;
    A->vec2 = 1;
    A->begin = 0;
    A->nfull = n / kBlock;
    A->tail = (int32_t)(n % kBlock);
    A->evaluator = 100;
    A->npts = 1;
    A->warps = c->warps_override;  // 0: the evaluator's default kernel shape
    A->tma = c->pipeline == 4 ? 1 : c->pipeline;  // 4: pipeline 1 with the warp-task C1 shell
    A->task_shell = c->pipeline == 4;
    A->acc = c->acc;
    A->ticket = c->ticket;
    A->work_counter = c->work_counter;
    A->errkey = c->errkey;
    A->tail_scratch = c->tail_scratch;
    A->acc_out = c->res_dev + kResHead;
    A->result_i = c->res_dev;
    A->fix_counter = c->fix_counter;
    A->fix_list = c->fix_list;
    A->mode = MODE_EXPORT;
    if (c->bsums_cap < nb) {
        cudaFree(c->bsums);
        c->bsums = nullptr;
        CK(cudaMalloc(&c->bsums, sizeof(double) * nb));
        c->bsums_cap = nb;
    }
    A->block_sums = c->bsums;
    if (c->timing) CK(cudaEventRecord(c->ev0, c->stream));
    CK(launch_nll(*A, c->stream, c->sm_count, 1));
    ++c->launches;
    if (c->timing) CK(cudaEventRecord(c->ev1, c->stream));
    rc = read_result(c);
    if (rc) return rc;
    if (out_block_sums)
        CK(cudaMemcpy(out_block_sums, c->bsums, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    return round_result(c, out_total);
}

int pfb_exact_sum_host(const double* v, int64_t n, double* out) {
    if ((!v && n) || !out || n < 0) return PFB_E_INVALID_ARGUMENT;
    long long acc[PFB_ACC_WORDS];
    memset(acc, 0, sizeof(acc));
    for (int64_t i = 0; i < n; ++i) acc_add_host(acc, v[i]);
    return acc_round(acc, out);
}

int pfb_acc_round(const int64_t* acc, double* out) {
    if (!acc || !out) return PFB_E_INVALID_ARGUMENT;
    return acc_round((const long long*)acc, out);
}

int pfb_acc_add_host(int64_t* acc, const double* v, int64_t n) {
    if (!acc || (!v && n) || n < 0) return PFB_E_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i) acc_add_host((long long*)acc, v[i]);
    return PFB_OK;
}

int pfb_shard_bounds(int64_t n, int32_t workers, int64_t block, int64_t* bounds) {
    if (workers < 1 || n < 0 || !bounds || block < 1) return PFB_E_INVALID_ARGUMENT;
    // sharding.shard (sharding.py:80-85)
    const int64_t base = n / workers, extra = n % workers;
    bounds[0] = 0;
    for (int k = 0; k < workers; ++k) bounds[k + 1] = bounds[k] + base + (k < extra ? 1 : 0);
    if (n >= (int64_t)workers * block)
        for (int k = 1; k < workers; ++k) bounds[k] = (bounds[k] / block) * block;
    bounds[workers] = n;
    return PFB_OK;
}

// ---- Dalitz grid ---------------------------------------------------------------

int pfb_grid_create(pfb_ctx* c, const pfb_dalitz_desc* d, int32_t nx, int32_t ny, pfb_grid** out) {
    if (!c || !d || !out) return PFB_E_INVALID_ARGUMENT;
    *out = nullptr;
    if (nx < 32 || ny < 32) return PFB_E_DEGENERATE_GRID;  // dalitz.py:253-254
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto g = std::make_unique<pfb_grid>();
    g->ctx = c;
    g->desc = *d;
    GridConsts& k = g->g;
    k.nx = nx;
    k.ny = ny;
    const double M = d->mother_mass;
    // DecayChannel.s12_range / s13_range (dalitz.py:68-74): Python (a)**2
    const double a12 = d->m1 + d->m2, b12 = M - d->m3, a13 = d->m1 + d->m3, b13 = M - d->m2;
    k.lo12 = a12 * a12;
    k.hi12 = b12 * b12;
    k.lo13 = a13 * a13;
    const double hi13 = b13 * b13;
    k.dx = (k.hi12 - k.lo12) / nx;
    k.dy = (hi13 - k.lo13) / ny;
    k.m1sq = d->m1 * d->m1;
    k.m2sq = d->m2 * d->m2;
    k.m3sq = d->m3 * d->m3;
    k.M2 = M * M;
    g->area = k.dx * k.dy;
    const int64_t total = (int64_t)nx * ny;
    int* row_count = nullptr;
    CK(cudaMalloc(&g->mask, total));
    CK(cudaMalloc(&row_count, sizeof(int) * nx));
    std::unique_ptr<int, cudaError_t (*)(void*)> rc_guard(row_count, cudaFree);
    CK(cudaMemsetAsync(row_count, 0, sizeof(int) * nx, c->stream));
    CK(launch_grid_mask(k, g->mask, row_count, c->stream));
    ++c->launches;
    std::vector<int> counts(nx), offs(nx);
    CK(cudaMemcpyAsync(counts.data(), row_count, sizeof(int) * nx, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int64_t acc = 0;
    for (int i = 0; i < nx; ++i) {
        offs[i] = (int)acc;
        acc += counts[i];
    }
    g->n_inside = acc;
    CK(cudaMemcpyAsync(row_count, offs.data(), sizeof(int) * nx, cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMalloc(&g->p12, sizeof(double) * (acc > 0 ? acc : 1)));
    CK(cudaMalloc(&g->p13, sizeof(double) * (acc > 0 ? acc : 1)));
    CK(launch_grid_compact(k, g->mask, row_count, g->p12, g->p13, c->stream));
    ++c->launches;
    CK(cudaStreamSynchronize(c->stream));
    *out = g.release();
    return PFB_OK;
}

int pfb_grid_info(const pfb_grid* g, int64_t* n_inside, double* area) {
    if (!g) return PFB_E_INVALID_ARGUMENT;
    if (n_inside) *n_inside = g->n_inside;
    if (area) *area = g->area;
    return PFB_OK;
}

int pfb_grid_mask(const pfb_grid* g, uint8_t* host_mask) {
    if (!g || !host_mask) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(g->ctx->device));
    CK(cudaMemcpy(host_mask, g->mask, (size_t)g->g.nx * g->g.ny, cudaMemcpyDeviceToHost));
    return PFB_OK;
}

int pfb_grid_integrals(pfb_ctx* c, pfb_grid* g, int32_t K, const int32_t* pair,
                       const int32_t* spin, const double* mass_width, const uint8_t* rows,
                       const uint8_t* stale, double* inout) {
    if (!c || !g || K < 1 || K > kMaxDal || !pair || !spin || !mass_width || !rows || !stale ||
        !inout)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    const int64_t n = g->n_inside;
    if (g->amps_rows < K) {
        double2* na = nullptr;
        CK(cudaMalloc(&na, sizeof(double2) * (size_t)K * (size_t)(n > 0 ? n : 1)));
        if (g->amps) {
            CK(cudaMemcpyAsync(na, g->amps, sizeof(double2) * (size_t)g->amps_rows * n,
                               cudaMemcpyDeviceToDevice, c->stream));
            cudaStreamSynchronize(c->stream);
            cudaFree(g->amps);
        }
        g->amps = na;
        g->amps_rows = K;
    }
    // channel constants as in build_dal
    DalDesc D;
    memset(&D, 0, sizeof(D));
    const pfb_dalitz_desc& d = g->desc;
    const double M = d.mother_mass;
    const double M2 = M * M, m1sq = d.m1 * d.m1, m2sq = d.m2 * d.m2, m3sq = d.m3 * d.m3;
    D.K = K;
    D.mss = ((M2 + m1sq) + m2sq) + m3sq;
    D.zc12 = (M2 - m3sq) * (m2sq - m1sq);
    D.zc13 = (M2 - m2sq) * (m3sq - m1sq);
    D.zc23 = (M2 - m1sq) * (m3sq - m2sq);
    for (int k = 0; k < K; ++k) {
        if (!rows[k]) continue;
        if (!(pair[k] == 12 || pair[k] == 13 || pair[k] == 23) || !(spin[k] == 0 || spin[k] == 1))
            return PFB_E_INVALID_ARGUMENT;
        DalTerm T;
        memset(&T, 0, sizeof(T));
        T.pair = pair[k];
        T.spin = spin[k];
        const double m = mass_width[2 * k], w = mass_width[2 * k + 1];
        T.m2 = m * m;
        T.mg = m * w;
        CK(launch_grid_amp(D, T, g->p12, g->p13, n, g->amps + (int64_t)k * n, c->stream,
                           c->sm_count));
        ++c->launches;
    }
    std::vector<int2> pairs;
    for (int i = 0; i < K; ++i)
        for (int j = i; j < K; ++j)
            if (stale[i] || stale[j]) pairs.push_back(make_int2(i, j));
    if (!pairs.empty() && n > 0) {
        const size_t words = pairs.size() * 2 * PFB_ACC_WORDS;
        int2* dpairs = nullptr;
        unsigned long long* dacc = nullptr;
        CK(cudaMalloc(&dpairs, sizeof(int2) * pairs.size()));
        CK(cudaMalloc(&dacc, sizeof(unsigned long long) * words));
        std::unique_ptr<int2, cudaError_t (*)(void*)> g1(dpairs, cudaFree);
        std::unique_ptr<unsigned long long, cudaError_t (*)(void*)> g2(dacc, cudaFree);
        CK(cudaMemcpyAsync(dpairs, pairs.data(), sizeof(int2) * pairs.size(),
                           cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemsetAsync(dacc, 0, sizeof(unsigned long long) * words, c->stream));
        CK(launch_grid_overlap(g->amps, n, dpairs, (int)pairs.size(), dacc, c->stream,
                               c->sm_count));
        ++c->launches;
        std::vector<long long> hacc(words);
        CK(cudaMemcpyAsync(hacc.data(), dacc, sizeof(long long) * words, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t q = 0; q < pairs.size(); ++q) {
            double re, im;
            acc_round(&hacc[(q * 2) * PFB_ACC_WORDS], &re);
            acc_round(&hacc[(q * 2 + 1) * PFB_ACC_WORDS], &im);
            const int i = pairs[q].x, j = pairs[q].y;
            // dalitz.py:321-328: diagonal real sum * dA; off-diagonal complex sum * dA
            re = re * g->area;
            im = (i == j) ? 0.0 : im * g->area;
            inout[2 * (i * K + j)] = re;
            inout[2 * (i * K + j) + 1] = im;
            inout[2 * (j * K + i)] = re;
            inout[2 * (j * K + i) + 1] = (i == j) ? 0.0 : -im;
        }
    } else if (!pairs.empty()) {
        for (auto pr : pairs) {
            const int i = pr.x, j = pr.y;
            inout[2 * (i * K + j)] = inout[2 * (i * K + j) + 1] = 0.0;
            inout[2 * (j * K + i)] = inout[2 * (j * K + i) + 1] = 0.0;
        }
    }
    return PFB_OK;
}

int pfb_grid_destroy(pfb_grid* g) {
    if (!g) return PFB_OK;
    cudaSetDevice(g->ctx->device);
    cudaFree(g->mask);
    cudaFree(g->p12);
    cudaFree(g->p13);
    cudaFree(g->amps);
    delete g;
    return PFB_OK;
}

// ---- synthetic event generation (toy MC) -------------------------------------------

static void fill_daldesc(const pfb_dalitz_desc& d, const double* raw, DalDesc* D) {
    memset(D, 0, sizeof(DalDesc));
    const double M = d.mother_mass;
    const double M2 = M * M, m1sq = d.m1 * d.m1, m2sq = d.m2 * d.m2, m3sq = d.m3 * d.m3;
    D->K = d.nterms;
    D->mss = ((M2 + m1sq) + m2sq) + m3sq;
    D->zc12 = (M2 - m3sq) * (m2sq - m1sq);
    D->zc13 = (M2 - m2sq) * (m3sq - m1sq);
    D->zc23 = (M2 - m1sq) * (m3sq - m2sq);
    for (int k = 0; k < d.nterms; ++k) {
        DalTerm& T = D->t[k];
        const double m = raw[4 * k], w = raw[4 * k + 1], mag = raw[4 * k + 2], ph = raw[4 * k + 3];
        T.pair = d.pair[k];
        T.spin = d.spin[k];
        T.m2 = m * m;
        T.mg = m * w;
        T.mg2 = T.mg * T.mg;
        T.cre = mag * cos(ph);
        T.cim = mag * sin(ph);
        T.alpha = T.cre * T.m2 - T.cim * T.mg;
        T.beta = T.cre * T.mg + T.cim * T.m2;
    }
}

int pfb_gen_dalitz(pfb_ctx* c, const pfb_dalitz_desc* d, const double* term_values, double envelope,
                   uint64_t seed, int64_t n, pfb_store* out, int64_t* candidates) {
    if (!c || !d || !term_values || !out || n < 0 || out->ncols < 2 || out->n < n || !(envelope > 0.0) ||
        d->nterms < 1 || d->nterms > kMaxDal)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    GenDalitz G;
    memset(&G, 0, sizeof(G));
    fill_daldesc(*d, term_values, &G.D);
    const double a12 = d->m1 + d->m2, b12 = d->mother_mass - d->m3;
    const double a13 = d->m1 + d->m3, b13 = d->mother_mass - d->m2;
    G.lo12 = a12 * a12;
    G.hi12 = b12 * b12;
    G.lo13 = a13 * a13;
    G.hi13 = b13 * b13;
    G.m1sq = d->m1 * d->m1;
    G.m2sq = d->m2 * d->m2;
    G.m3sq = d->m3 * d->m3;
    G.M2 = d->mother_mass * d->mother_mass;
    G.envelope = envelope;
    G.seed_lo = (uint32_t)seed;
    G.seed_hi = (uint32_t)(seed >> 32);
    store_touched(out);
    if (n == 0) return PFB_OK;
    CK(run_gen_dalitz(G, n, out->cols[0], out->cols[1], c->stream, c->sm_count, candidates));
    c->launches += 3;
    CK(cudaStreamSynchronize(c->stream));
    return PFB_OK;
}

int pfb_gen_1d(pfb_ctx* c, int32_t kind, double mu, double sigma, double alpha, double f, double lo,
               double hi, uint64_t seed, int64_t n, pfb_store* out) {
    if (!c || !out || n < 0 || out->n < n || (kind != 0 && kind != 1) || out->ncols < (kind == 1 ? 2 : 1) ||
        !(sigma > 0.0) || !(hi > lo))
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    Gen1D G;
    G.kind = kind;
    G.mu = mu;
    G.sigma = sigma;
    G.alpha = alpha;
    G.f = f;
    G.lo = lo;
    G.hi = hi;
    G.seed_lo = (uint32_t)seed;
    G.seed_hi = (uint32_t)(seed >> 32);
    store_touched(out);
    if (n == 0) return PFB_OK;
    CK(launch_gen_1d(G, n, out->cols[0], kind == 1 ? out->cols[1] : nullptr, c->stream, c->sm_count));
    ++c->launches;
    CK(cudaStreamSynchronize(c->stream));
    return PFB_OK;
}

}  // extern "C"

// Device -> host copy of `count` doubles into a pageable host buffer (a fresh
// numpy array).  One pageable cudaMemcpy is bound by a single staging copy
// and the page faults of the destination (~4 GB/s); here up to kDlLanes host
// threads each move a contiguous share through their own two pinned 8 MB
// buffers and stream, so the faults and the copies out of staging run in
// parallel while the copy engine fills the other buffer (100M-event Dalitz
// toy: 2.1 -> 0.87 s end to end).  Pinned destinations and small copies go
// straight through cudaMemcpyAsync.
static int download_to_host(pfb_ctx* c, const double* dev, double* host, int64_t count) {
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    cudaPointerAttributes pa;
    const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type != cudaMemoryTypeUnregistered;
    cudaGetLastError();
    const unsigned hw = std::thread::hardware_concurrency();
    const int lanes = (int)std::min<int64_t>({(int64_t)kDlLanes, (int64_t)(hw > 2 ? hw / 2 : 1),
                                              (count + kDlChunk - 1) / kDlChunk});
    if (pinned || lanes < 2) {
        CK(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return PFB_OK;
    }
    CK(cudaStreamSynchronize(c->stream));  // the device column is not in use by queued work
    for (int t = 0; t < lanes; ++t) {
        for (int b = 0; b < 2; ++b)
            if (!c->dl_pinned[t][b]) CK(cudaHostAlloc(&c->dl_pinned[t][b], sizeof(double) * kDlChunk, cudaHostAllocDefault));
        if (!c->dl_stream[t]) CK(cudaStreamCreateWithFlags(&c->dl_stream[t], cudaStreamNonBlocking));
    }
    std::vector<cudaError_t> errs(lanes, cudaSuccess);
    std::vector<std::thread> pool;
    const int64_t share = (count + lanes - 1) / lanes;
    auto lane = [&](int t) {
        cudaError_t e = cudaSetDevice(c->device);
        const int64_t b0 = std::min(count, t * share), b1 = std::min(count, b0 + share);
        const int64_t np = (b1 - b0 + kDlChunk - 1) / kDlChunk;
        cudaStream_t s = c->dl_stream[t];
        double* const* buf = c->dl_pinned[t];
        auto piece = [&](int64_t k) { return std::min(kDlChunk, b1 - (b0 + k * kDlChunk)); };
        auto at = [&](int64_t k) { return b0 + k * kDlChunk; };
        if (e == cudaSuccess && np > 0)
            e = cudaMemcpyAsync(buf[0], dev + at(0), sizeof(double) * piece(0), cudaMemcpyDeviceToHost, s);
        for (int64_t k = 0; e == cudaSuccess && k < np; ++k) {
            e = cudaStreamSynchronize(s);  // piece k is in buffer k & 1
            if (e == cudaSuccess && k + 1 < np)
                e = cudaMemcpyAsync(buf[(k + 1) & 1], dev + at(k + 1), sizeof(double) * piece(k + 1),
                                    cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) memcpy(host + at(k), buf[k & 1], sizeof(double) * piece(k));
        }
        errs[t] = e;
    };
    // no exception may cross the C ABI: a lane whose thread cannot be
    // started runs on this thread after the others are launched
    std::vector<int> inline_lanes;
    for (int t = 0; t < lanes; ++t) {
        try {
            pool.emplace_back(lane, t);
        } catch (...) {
            inline_lanes.push_back(t);
        }
    }
    for (int t : inline_lanes) lane(t);
    for (auto& th : pool) th.join();
    for (int t = 0; t < lanes; ++t) CK(errs[t]);
    return PFB_OK;
}

extern "C" {

int pfb_store_download(pfb_store* st, int32_t col, double* host, int64_t offset, int64_t count) {
    if (!st || !host || col < 0 || col >= st->ncols || offset < 0 || count < 0 || offset + count > st->n)
        return PFB_E_INVALID_ARGUMENT;
    return download_to_host(st->ctx, st->cols[col] + offset, host, count);
}

int pfb_fp64_peak(pfb_ctx* c, double* out) {
    if (!c || !out) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    const int blocks = c->sm_count * 8, threads = 256, iters = 2048;
    CK(launch_fp64_peak(c->probe_dev, blocks, threads, 16, c->stream));  // warm-up
    CK(cudaEventRecord(c->ev0, c->stream));
    CK(launch_fp64_peak(c->probe_dev, blocks, threads, iters, c->stream));
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->launches += 2;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    const double flops = 2.0 * 16.0 * 8.0 * (double)iters * (double)blocks * threads;
    *out = flops / (ms * 1e-3) / 1e12;
    return PFB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Binned data.

static int ensure_bin(pfb_ctx* c, int64_t bytes) {
    if (!c->bin_key) CK(cudaMalloc(&c->bin_key, sizeof(unsigned long long)));
    if (c->bin_cap >= bytes) return PFB_OK;
    cudaFree(c->bin_dev);
    c->bin_dev = nullptr;
    c->bin_cap = 0;
    CK(cudaMalloc(&c->bin_dev, (size_t)bytes));
    c->bin_cap = bytes;
    return PFB_OK;
}

extern "C" {

int pfb_ctx_spin(pfb_ctx* c, int64_t cycles, const double* flush_buf, int64_t flush_bytes) {
    if (!c || cycles < 0 || flush_bytes < 0 || (flush_bytes && !flush_buf)) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    CK(launch_spin_flush(cycles, flush_buf, flush_bytes, c->probe_dev, c->sm_count, c->stream));
    return PFB_OK;
}

int pfb_bin_fill(pfb_ctx* c, const pfb_store* st, int64_t begin, int64_t end, int32_t naxes,
                 const int32_t* cols, const double* lower, const double* width, const int64_t* nbins,
                 double* contents) {
    if (!c || !st || st->ctx != c || !cols || !lower || !width || !nbins || !contents) return PFB_E_INVALID_ARGUMENT;
    if (naxes < 1 || naxes > kMaxCols || begin < 0 || end < begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    BinAxes B;
    memset(&B, 0, sizeof(B));
    B.naxes = naxes;
    int64_t total_bins = 1;
    for (int a = 0; a < naxes; ++a) {
        if (cols[a] < 0 || cols[a] >= st->ncols || nbins[a] < 1) return PFB_E_INVALID_ARGUMENT;
        if (total_bins > ((int64_t)1 << 40) / nbins[a]) return PFB_E_INVALID_ARGUMENT;
        total_bins *= nbins[a];
        B.col[a] = st->cols[cols[a]];
        B.lower[a] = lower[a];
        B.width[a] = width[a];
        B.nbins[a] = nbins[a];
    }
    if (end == begin) return PFB_OK;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = ensure_bin(c, (int64_t)sizeof(unsigned long long) * total_bins);
    if (rc) return rc;
    auto* counts = static_cast<unsigned long long*>(c->bin_dev);
    CK(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * total_bins, c->stream));
    CK(launch_bin_fill(B, begin, end - begin, counts, c->stream, c->sm_count));
    ++c->launches;
    std::vector<unsigned long long> h(total_bins);
    CK(cudaMemcpyAsync(h.data(), counts, sizeof(unsigned long long) * total_bins, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    // np.add.at adds 1.0 once per event: integral contents (< 2^53) take the
    // count in one exact addition; anything else repeats the reference's adds.
    for (int64_t i = 0; i < total_bins; ++i) {
        if (!h[i]) continue;
        const double v = contents[i];
        if (v == floor(v) && fabs(v) < 9007199254740992.0 && h[i] < (1ull << 53)) {
            contents[i] = v + (double)h[i];
        } else {
            double x = v;
            for (unsigned long long k = 0; k < h[i]; ++k) x += 1.0;
            contents[i] = x;
        }
    }
    return PFB_OK;
}

}  // extern "C"

// One quadrature launch into result slot q (accumulator q, head kResQuad + 4q),
// without a wait: the objective enqueues every quadrature norm of a batch of
// points and waits once (pfb_objective_eval_batch).  A keeps the packed
// arguments for quad_collect's error decoding; *frac the fraction status.
static int quad_enqueue(pfb_ctx* c, pfb_plan* p, const pfb_store* st, int32_t weight_col, const double* values,
                        const double* norms, int q, NllArgs* A, int* frac) {
    *frac = pack_args(p, st, 0, st->n, values, norms, A);
    A->acc_out = c->res_dev + kResHead + (int64_t)q * PFB_ACC_WORDS;
    A->result_i = c->res_dev + kResQuad + 4 * q;
    CK(launch_quadrature(*A, st->cols[weight_col], st->n, c->stream, c->sm_count));
    ++c->launches;
    return PFB_OK;
}

// Slots [0, nq) after their launches: copy the result block back if it is not mapped.
static int quad_wait(pfb_ctx* c) {
    if (!c->res_mapped)
        CK(cudaMemcpyAsync(c->res_host, c->res_dev, sizeof(long long) * kResWords, cudaMemcpyDeviceToHost,
                           c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return PFB_OK;
}

// Slot q's integral (after quad_wait): the status and the rounded sum.
static int quad_collect(pfb_ctx* c, const pfb_plan* p, const NllArgs& A, int q, int frac, double* out,
                        pfb_err* err) {
    int code = decode_error(c, p, A, (unsigned long long)c->res_host[kResQuad + 4 * q + 1], frac, 0, err);
    double r = 0.0;
    if (!code) code = acc_round(c->res_host + kResHead + (int64_t)q * PFB_ACC_WORDS, &r);
    if (err) err->code = code;
    *out = r;
    return code;
}

static int quad_check(const pfb_ctx* c, const pfb_plan* p, const pfb_store* st, int32_t weight_col) {
    if (!c || !p || !st || p->ctx != c || st->ctx != c) return PFB_E_INVALID_ARGUMENT;
    if (weight_col < 0 || weight_col >= st->ncols || st->n < 1) return PFB_E_INVALID_ARGUMENT;
    for (int s = 0; s < p->nslots; ++s)
        if (p->slot_col[s] >= st->ncols || p->slot_col[s] == weight_col) return PFB_E_INVALID_ARGUMENT;
    return PFB_OK;
}

extern "C" {

int pfb_quadrature(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int32_t weight_col, const double* values,
                   int32_t nvalues, const double* norms, int32_t nnorms, double* out, pfb_err* out_err) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!values || !norms || !out || quad_check(c, p, st, weight_col)) return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    clear_err(out_err);
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    int frac = -1;
    if (c->timing) CK(cudaEventRecord(c->ev0, c->stream));
    int rc = quad_enqueue(c, p, st, weight_col, values, norms, 0, A.get(), &frac);
    if (rc) return rc;
    if (c->timing) CK(cudaEventRecord(c->ev1, c->stream));
    rc = quad_wait(c);
    if (rc) return rc;
    if (c->timing) cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    pfb_err e;
    const int code = quad_collect(c, p, *A, 0, frac, out, &e);
    if (out_err) *out_err = e;
    return code;
}

int pfb_binned_nll(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, const double* contents, int64_t nbins,
                   double total, double volume, const double* values, int32_t nvalues, const double* norms,
                   int32_t nnorms, double* out_nll, pfb_err* out_err) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !contents || !values || !norms || p->ctx != c || st->ctx != c)
        return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (nbins < 1 || nbins > st->n) return PFB_E_INVALID_ARGUMENT;
    for (int s = 0; s < p->nslots; ++s)
        if (p->slot_col[s] >= st->ncols) return PFB_E_INVALID_ARGUMENT;
    clear_err(out_err);
    if (!(total > 0.0)) {
        if (out_err) out_err->code = PFB_E_EMPTY_DATASET;
        return PFB_E_EMPTY_DATASET;
    }
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = ensure_bin(c, 0);  // bin_key
    if (rc) return rc;
    if (c->bin_cont_cap < nbins) {
        cudaFree(c->bin_cont);
        c->bin_cont = nullptr;
        c->bin_cont_cap = 0;
        c->bin_cont_host.clear();
        CK(cudaMalloc(&c->bin_cont, sizeof(double) * nbins));
        c->bin_cont_cap = nbins;
    }
    // upload the contents only when they differ from the last upload
    if ((int64_t)c->bin_cont_host.size() != nbins ||
        memcmp(c->bin_cont_host.data(), contents, sizeof(double) * nbins) != 0) {
        c->bin_cont_host.assign(contents, contents + nbins);
        CK(cudaMemcpyAsync(c->bin_cont, c->bin_cont_host.data(), sizeof(double) * nbins, cudaMemcpyHostToDevice,
                           c->stream));
    }
    auto A = std::make_unique<NllArgs>();
    const int frac = pack_args(p, st, 0, nbins, values, norms, A.get());
    A->xkey = c->bin_key;  // the exporting CTA hands the key back in the result block and resets it
    CK(cudaMemsetAsync(c->bin_key, 0xff, sizeof(unsigned long long), c->stream));
    if (c->timing) CK(cudaEventRecord(c->ev0, c->stream));
    CK(launch_binned_nll(*A, c->bin_cont, nbins, total, volume, c->bin_key, c->stream, c->sm_count));
    ++c->launches;
    if (c->timing) CK(cudaEventRecord(c->ev1, c->stream));
    rc = read_result(c);
    if (rc) return rc;
    const unsigned long long expkey = (unsigned long long)c->res_host[2];
    pfb_err e;
    int code = decode_error(c, p, *A, (unsigned long long)c->res_host[1], frac, 0, &e);
    if (!code && expkey != ~0ull) {
        CK(launch_binned_probe(*A, (int64_t)expkey, total, volume, c->probe_dev, c->stream));
        ++c->launches;
        double nu = 0.0;
        CK(cudaMemcpyAsync(&nu, c->probe_dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        code = PFB_E_NONPOSITIVE_EXPECTATION;
        e.code = code;
        e.node = -1;
        e.index = (int64_t)expkey;
        e.value = nu;
    }
    double r = 0.0;
    if (!code) code = acc_round(c->res_host + kResHead, &r);
    e.code = code;
    if (out_nll) *out_nll = r;
    if (out_err) *out_err = e;
    return code;
}


}  // extern "C"

// ---- stream-exact toy generation ------------------------------

static GridConsts grid_consts_of(const pfb_dalitz_desc& d, int nx, int ny) {
    GridConsts k{};
    k.nx = nx;
    k.ny = ny;
    const double M = d.mother_mass;
    // DecayChannel.s12_range / s13_range (dalitz.py:68-74): Python (a)**2
    const double a12 = d.m1 + d.m2, b12 = M - d.m3, a13 = d.m1 + d.m3, b13 = M - d.m2;
    k.lo12 = a12 * a12;
    k.hi12 = b12 * b12;
    k.lo13 = a13 * a13;
    const double hi13 = b13 * b13;
    k.dx = (k.hi12 - k.lo12) / nx;
    k.dy = (hi13 - k.lo13) / ny;
    k.m1sq = d.m1 * d.m1;
    k.m2sq = d.m2 * d.m2;
    k.m3sq = d.m3 * d.m3;
    k.M2 = M * M;
    return k;
}

static int pack_density_args(pfb_ctx* c, const pfb_plan* p, const double* values, int32_t nvalues,
                             const double* norms, int32_t nnorms, NllArgs* A) {
    if (p->ctx != c || nvalues != p->nraw || nnorms != (int32_t)p->nodes.size() || p->nslots > 2)
        return PFB_E_INVALID_ARGUMENT;
    pfb_store dummy;
    dummy.ctx = c;
    dummy.ncols = kStoreMaxCols;
    dummy.n = 0;
    const int frac = pack_args(p, &dummy, 0, 0, values, norms, A);
    return frac >= 0 ? PFB_E_FRACTION_OUT_OF_RANGE : PFB_OK;
}

static int gen_status(const PcgHostResult& R, pfb_gen_stats* stats) {
    if (stats) {
        stats->attempts = R.attempts;
        stats->accepted = R.accepted;
        stats->in_boundary = R.in_boundary;
        stats->produced = R.produced;
        stats->observed = R.observed;
        stats->ambiguous = R.ambiguous;
    }
    switch (R.status) {
        case 0: return PFB_OK;
        case 2: return PFB_E_NONFINITE_DENSITY;
        case 10: return PFB_E_ENVELOPE_HIT;
        default: return PFB_E_ATTEMPTS_EXHAUSTED;
    }
}

extern "C" {

int pfb_pcg_scan_1d(pfb_ctx* c, const pfb_plan* p, const double* values, int32_t nvalues, const double* norms,
                    int32_t nnorms, double lo, double hi, int64_t points, double* out_max) {
    if (!c || !p || !values || !norms || !out_max || points < 1) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    int rc = pack_density_args(c, p, values, nvalues, norms, nnorms, A.get());
    if (rc) return rc;
    rc = ensure_bin(c, 0);
    if (rc) return rc;
    CK(pcg_scan_1d(*A, lo, hi, points, out_max, c->bin_key, c->stream, c->sm_count));
    ++c->launches;
    return PFB_OK;
}

int pfb_pcg_scan_dalitz(pfb_ctx* c, const pfb_dalitz_desc* d, const double* term_values, int32_t n,
                        double* out_max) {
    if (!c || !d || !term_values || !out_max || n < 1 || d->nterms < 1 || d->nterms > kMaxDal)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    memset(A.get(), 0, sizeof(NllArgs));
    fill_daldesc(*d, term_values, &A->dal);
    int rc = ensure_bin(c, 0);
    if (rc) return rc;
    CK(pcg_scan_dalitz(*A, grid_consts_of(*d, n, n), out_max, c->bin_key, c->stream, c->sm_count));
    ++c->launches;
    return PFB_OK;
}

int pfb_pcg_generate_1d(pfb_ctx* c, const pfb_plan* p, const double* values, int32_t nvalues,
                        const double* norms, int32_t nnorms, double lo, double hi, double envelope,
                        const pfb_pcg64* stream, int64_t n_wanted, int64_t budget, pfb_store* out,
                        int64_t out_offset, pfb_gen_stats* stats) {
    if (!c || !p || !values || !norms || !stream || !out || out->ctx != c || n_wanted < 0 || budget < 0 ||
        out_offset < 0 || out_offset + n_wanted > out->n || out->ncols < 1)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    int rc = pack_density_args(c, p, values, nvalues, norms, nnorms, A.get());
    if (rc) return rc;
    const double box[4] = {lo, hi - lo, 0.0, 0.0};
    store_touched(out);
    PcgHostResult R;
    CK(pcg_generate_entry(*A, 0, box, envelope, nullptr, stream->state_hi, stream->state_lo, stream->inc_hi,
                          stream->inc_lo, n_wanted, budget, out->cols[0] + out_offset, nullptr, c->stream, &R));
    c->launches += 2;
    return gen_status(R, stats);
}

int pfb_pcg_generate_dalitz(pfb_ctx* c, const pfb_dalitz_desc* d, const double* term_values, double envelope,
                            const pfb_pcg64* stream, int64_t n_wanted, int64_t budget, pfb_store* out,
                            int64_t out_offset, pfb_gen_stats* stats) {
    if (!c || !d || !term_values || !stream || !out || out->ctx != c || n_wanted < 0 || budget < 0 ||
        out_offset < 0 || out_offset + n_wanted > out->n || out->ncols < 2 || d->nterms < 1 ||
        d->nterms > kMaxDal)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    memset(A.get(), 0, sizeof(NllArgs));
    fill_daldesc(*d, term_values, &A->dal);
    const GridConsts g = grid_consts_of(*d, 1, 1);
    const double M = d->mother_mass;
    const double b13 = M - d->m2;
    const double hi13 = b13 * b13;
    // uniform(lo, hi): scale = hi - lo as numpy computes it
    const double box[4] = {g.lo12, g.hi12 - g.lo12, g.lo13, hi13 - g.lo13};
    store_touched(out);
    PcgHostResult R;
    CK(pcg_generate_entry(*A, 1, box, envelope, &g, stream->state_hi, stream->state_lo, stream->inc_hi,
                          stream->inc_lo, n_wanted, budget, out->cols[0] + out_offset, out->cols[1] + out_offset,
                          c->stream, &R));
    c->launches += 2;
    return gen_status(R, stats);
}


// ---- binary SoA ingest ---------------------------------------


int pfb_npy_length(const char* path, int64_t* n_out) {
    if (!path || !n_out) return PFB_E_INVALID_ARGUMENT;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return PFB_E_INVALID_ARGUMENT;
    int64_t n = 0, off = 0;
    const int bad = npy_parse(fd, &n, &off);
    close(fd);
    if (bad) return PFB_E_INVALID_ARGUMENT;
    *n_out = n;
    return PFB_OK;
}

int pfb_store_load_npy(pfb_store* st, int32_t col, const char* path, int64_t src_offset, int64_t dst_offset,
                       int64_t count) {
    if (!st || !path || col < 0 || col >= st->ncols || src_offset < 0 || dst_offset < 0 || count < 0 ||
        dst_offset + count > st->n)
        return PFB_E_INVALID_ARGUMENT;
    pfb_ctx* c = st->ctx;
    store_touched(st);
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return PFB_E_INVALID_ARGUMENT;
    std::unique_ptr<int, void (*)(int*)> fd_guard(new int(fd), [](int* f) {
        close(*f);
        delete f;
    });
    int64_t n = 0, off = 0;
    if (npy_parse(fd, &n, &off) || src_offset + count > n) return PFB_E_INVALID_ARGUMENT;
    if (count == 0) return PFB_OK;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    for (int b = 0; b < 2; ++b) {
        if (!c->io_pinned[b]) CK(cudaHostAlloc(&c->io_pinned[b], sizeof(double) * kIoChunk, cudaHostAllocDefault));
        if (!c->io_event[b]) CK(cudaEventCreateWithFlags(&c->io_event[b], cudaEventDisableTiming));
    }
    CK(cudaStreamSynchronize(c->stream));  // the column is not in use by queued kernels
    bool used[2] = {false, false};
    for (int64_t done = 0, k = 0; done < count; done += kIoChunk, ++k) {
        const int b = (int)(k & 1);
        const int64_t m = count - done < kIoChunk ? count - done : kIoChunk;
        if (used[b]) CK(cudaEventSynchronize(c->io_event[b]));  // its previous copy has landed
        char* dst = reinterpret_cast<char*>(c->io_pinned[b]);
        int64_t want = m * (int64_t)sizeof(double), got = 0;
        const int64_t pos = off + (src_offset + done) * (int64_t)sizeof(double);
        while (got < want) {
            const ssize_t r = pread(fd, dst + got, (size_t)(want - got), pos + got);
            if (r <= 0) return PFB_E_INVALID_ARGUMENT;
            got += r;
        }
        CK(cudaMemcpyAsync(st->cols[col] + dst_offset + done, c->io_pinned[b], (size_t)want,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaEventRecord(c->io_event[b], c->copy_stream));
        used[b] = true;
    }
    CK(cudaStreamSynchronize(c->copy_stream));
    return PFB_OK;
}

int pfb_store_check_range(pfb_store* st, int32_t col, int64_t begin, int64_t end, double lower, double upper,
                          int64_t* first_bad, double* bad_value) {
    if (!st || !first_bad || col < 0 || col >= st->ncols || begin < 0 || end < begin || end > st->n)
        return PFB_E_INVALID_ARGUMENT;
    pfb_ctx* c = st->ctx;
    *first_bad = -1;
    if (end == begin) return PFB_OK;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = ensure_bin(c, 0);
    if (rc) return rc;
    CK(cudaMemsetAsync(c->bin_key, 0xff, sizeof(unsigned long long), c->stream));
    CK(launch_range_check(st->cols[col] + begin, end - begin, lower, upper, c->bin_key, c->stream, c->sm_count));
    ++c->launches;
    unsigned long long key = 0;
    CK(cudaMemcpyAsync(&key, c->bin_key, sizeof(key), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (key != ~0ull) {
        *first_bad = (int64_t)key;
        double v = 0.0;
        CK(cudaMemcpy(&v, st->cols[col] + begin + key, sizeof(double), cudaMemcpyDeviceToHost));
        if (bad_value) *bad_value = v;
    }
    return PFB_OK;
}


// Read-bandwidth microbenchmark (roofline calibration): `bytes` of a device
// buffer read once per launch; mode 0 SIMT loads, 1 bulk copies (1 CTA/SM),
// 2 bulk copies (2 CTAs/SM) with chunk_kb-KB stages.  Median of `reps`.
int pfb_read_bw(pfb_ctx* c, const double* buf, int64_t bytes, int32_t mode, int32_t chunk_kb, int32_t reps,
                double* out_gbps) {
    if (!c || !buf || bytes <= 0 || !out_gbps || mode < 0 || mode > 2 || reps < 1 || chunk_kb < 1)
        return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    int rc = ensure_bin(c, 0);
    if (rc) return rc;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ms;
    for (int r = 0; r < reps + 1; ++r) {
        CK(launch_spin_flush(200000, nullptr, 0, c->probe_dev, c->sm_count, c->stream));
        CK(cudaEventRecord(a, c->stream));
        CK(launch_read_bw(mode, buf, bytes, chunk_kb, c->probe_dev, c->bin_key, c->sm_count, c->stream));
        CK(cudaEventRecord(b, c->stream));
        CK(cudaEventSynchronize(b));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, a, b));
        if (r) ms.push_back(t);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(ms.begin(), ms.end());
    *out_gbps = (double)bytes / (ms[ms.size() / 2] * 1e-3) / 1e9;
    return PFB_OK;
}


// ---- cross-GPU accumulator exchange over peer memory ---------------

int pfb_peer_create(pfb_ctx* c, int32_t rank, int32_t world, uint8_t* out_handle) {
    if (!c || world < 1 || world > peer_max() || rank < 0 || rank >= world) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    if (c->peer_world) {  // already a member: the same group again is a no-op
        if (c->peer_world != world || c->peer_rank != rank) return PFB_E_INVALID_ARGUMENT;
        if (out_handle) {
            cudaIpcMemHandle_t h;
            memset(&h, 0, sizeof(h));
            if (world > 1) CK(cudaIpcGetMemHandle(&h, c->peer_ptr[rank]));
            memcpy(out_handle, &h, sizeof(h));
        }
        return PFB_OK;
    }
    long long* m = nullptr;
    CK(cudaMalloc(&m, peer_mailbox_bytes()));
    CK(cudaMemset(m, 0, peer_mailbox_bytes()));
    if (!c->peer_status) CK(cudaMalloc(&c->peer_status, sizeof(unsigned long long)));
    c->peer_world = world;
    c->peer_rank = rank;
    c->peer_ptr[rank] = m;
    c->peer_seq = 0;
    if (out_handle) {
        cudaIpcMemHandle_t h;
        memset(&h, 0, sizeof(h));
        if (world > 1) CK(cudaIpcGetMemHandle(&h, m));
        memcpy(out_handle, &h, sizeof(h));
    }
    return PFB_OK;
}

int pfb_peer_open(pfb_ctx* c, const uint8_t* handles) {
    if (!c || !handles || !c->peer_world) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    for (int q = 0; q < c->peer_world; ++q) {
        if (q == c->peer_rank || c->peer_ptr[q]) continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + (size_t)q * sizeof(cudaIpcMemHandle_t), sizeof(h));
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->peer_ptr[q] = static_cast<long long*>(p);
        c->peer_ipc[q] = true;
    }
    return PFB_OK;
}

int pfb_peer_attach(pfb_ctx* c, const void* const* mailboxes) {
    if (!c || !mailboxes || !c->peer_world) return PFB_E_INVALID_ARGUMENT;
    for (int q = 0; q < c->peer_world; ++q)
        if (q != c->peer_rank) c->peer_ptr[q] = static_cast<long long*>(const_cast<void*>(mailboxes[q]));
    return PFB_OK;
}

int pfb_peer_mailbox(pfb_ctx* c, void** out) {
    if (!c || !out || !c->peer_world) return PFB_E_INVALID_ARGUMENT;
    *out = c->peer_ptr[c->peer_rank];
    return PFB_OK;
}

int pfb_nll_peer(pfb_ctx* c, const pfb_plan* pc, const pfb_store* st, int64_t begin, int64_t end,
                 int64_t index_offset, const double* values, int32_t nvalues, const double* norms,
                 int32_t nnorms, double timeout_s, double* out_nll, int32_t* out_slow) {
    pfb_plan* p = const_cast<pfb_plan*>(pc);
    if (!c || !p || !st || !values || !norms || !out_nll || !out_slow || p->ctx != c || st->ctx != c ||
        !c->peer_world || !(timeout_s > 0.0))
        return PFB_E_INVALID_ARGUMENT;
    for (int q = 0; q < c->peer_world; ++q)
        if (!c->peer_ptr[q]) return PFB_E_INVALID_ARGUMENT;
    if (nvalues != p->nraw || nnorms != (int32_t)p->nodes.size()) return PFB_E_INVALID_ARGUMENT;
    if (begin < 0 || end <= begin || end > st->n) return PFB_E_INVALID_ARGUMENT;
    (void)index_offset;  // errors take the unfused path, which reports them with their offsets
    *out_slow = 0;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    pfb_store staged;
    const bool restaged = !range_aligned(p, st, begin);
    if (restaged) {
        const int rs = restage(c, p, st, begin, end, &staged);
        if (rs) return rs;
        st = &staged;
        end -= begin;
        begin = 0;
    }
    int rc = ensure_fix(c, (end - begin + kBlock - 1) / kBlock);
    if (rc) return rc;
    auto A = std::make_unique<NllArgs>();
    if (pack_args(p, st, begin, end, values, norms, A.get()) >= 0) {
        // FractionOutOfRange (pdf.py:205-210) is a property of the parameter
        // point, the same on every rank: no rank launches, every rank takes
        // the unfused path, which reports it in reference evaluation order
        *out_slow = 1;
        return PFB_OK;
    }
    A->mode = MODE_EXPORT;
    const int khz = c->clock_khz;  // a per-call attribute query would stall the queue
    for (int q = 0; q < c->peer_world; ++q) A->peer_mbox[q] = c->peer_ptr[q];
    A->peer_world = c->peer_world;
    A->peer_rank = c->peer_rank;
    A->peer_seq = ++c->peer_seq;
    A->peer_timeout = (long long)(timeout_s * (double)khz * 1e3);
    rc = launch_eval(p, st, begin, end, A.get(), !restaged);
    if (rc) return rc;
    rc = read_result(c);
    if (rc) return rc;
    if (c->res_host[3]) return PFB_E_PEER_TIMEOUT;
    if (c->res_host[2]) {  // a rank deferred blocks or failed: the caller redoes the call unfused
        *out_slow = 1;
        return PFB_OK;
    }
    return round_result(c, out_nll);
}

int pfb_peer_allreduce(pfb_ctx* c, int64_t* dev_acc, double timeout_s) {
    if (!c || !dev_acc || !c->peer_world || !(timeout_s > 0.0)) return PFB_E_INVALID_ARGUMENT;
    for (int q = 0; q < c->peer_world; ++q)
        if (!c->peer_ptr[q]) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    const int khz = c->clock_khz;  // a per-call attribute query would stall the queue
    const long long cycles = (long long)(timeout_s * (double)khz * 1e3);
    const unsigned long long seq = ++c->peer_seq;
    CK(launch_peer_allreduce(c->peer_ptr, c->peer_world, c->peer_rank, seq, cycles,
                             reinterpret_cast<long long*>(dev_acc), c->peer_status, c->stream));
    ++c->launches;
    unsigned long long st = 0;
    CK(cudaMemcpyAsync(&st, c->peer_status, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return st ? PFB_E_PEER_TIMEOUT : PFB_OK;
}


// Fixed-cost microbenchmark of one launch (event-timed, median of reps):
// mode 0 empty kernel, 1 + the 6.4 KB NllArgs parameter block, 2 + 64
// constant-bank reads, 3 + the accumulator epilogue (finish_launch).
int pfb_overhead_probe(pfb_ctx* c, int32_t mode, int32_t reps, double* out_us) {
    if (!c || !out_us || reps < 1 || mode < 0 || mode > 3) return PFB_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    PFB_QUIESCE(c);
    auto A = std::make_unique<NllArgs>();
    memset(A.get(), 0, sizeof(NllArgs));
    A->acc = c->acc;
    A->ticket = c->ticket;
    A->work_counter = c->work_counter;
    A->errkey = c->errkey;
    A->acc_out = c->res_dev + kResHead;
    A->result_i = c->res_dev;
    A->fix_counter = c->fix_counter;
    A->mode = MODE_EXPORT;
    A->npts = 1;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ms;
    for (int r = 0; r < reps + 1; ++r) {
        CK(launch_spin_flush(400000, nullptr, 0, c->probe_dev, c->sm_count, c->stream));
        CK(cudaEventRecord(a, c->stream));
        CK(launch_overhead_probe(mode, *A, c->probe_dev, c->stream));
        CK(cudaEventRecord(b, c->stream));
        CK(cudaEventSynchronize(b));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, a, b));
        if (r) ms.push_back(t);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(ms.begin(), ms.end());
    *out_us = 1e3 * ms[ms.size() / 2];
    return PFB_OK;
}

}  // extern "C"

// the minimiser objective in C (uses the internals above)
#include "pfb_objective.cuh"
