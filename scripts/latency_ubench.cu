// Launch / completion latency micro-benchmark on one B200 (what bounds a
// small-N NLL call): CUDA-event time and host round trip of
//   empty kernels (1 CTA / 148 CTAs), a 6.4 KB __grid_constant__ parameter
//   block, a final write of the result block into mapped pinned host memory,
//   the same launches through a CUDA graph, and a persistent kernel that
//   polls a mapped doorbell.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/latency_ubench scripts/latency_ubench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <functional>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

struct Big {
    double v[800];  // 6.4 KB
};

__global__ void empty_k(int* sink) {
    if (sink && threadIdx.x == 1023) sink[0] = 1;
}
__global__ void big_k(const __grid_constant__ Big b, double* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && b.v[799] == 12345.0) sink[0] = b.v[3];
}
extern __shared__ double dyn_smem[];
__global__ void big_smem_k(const __grid_constant__ Big b, double* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && b.v[799] == 12345.0) sink[0] = dyn_smem[threadIdx.x];
}
__global__ void small_smem_k(double* sink) {
    if (threadIdx.x == 100000) sink[0] = dyn_smem[threadIdx.x];
}
__global__ void mapped_k(volatile long long* host_res, int words) {
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < words) host_res[threadIdx.x] = threadIdx.x + 1;
}
__global__ void spin_k(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}
// persistent: one CTA polls a doorbell in mapped host memory; on a new
// sequence number it "computes" (a grid-wide nothing) and posts the result
__global__ void persistent_k(volatile unsigned* bell, volatile unsigned long long* res, int iters) {
    unsigned seen = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) {
            unsigned s;
            do {
                s = *bell;
            } while (s == seen);
            seen = s;
            __threadfence_system();
            res[0] = ((unsigned long long)s << 32) | 1ull;
        }
        __syncthreads();
    }
}

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    int* sink;
    CK(cudaMalloc(&sink, 64));
    long long* hres;
    CK(cudaHostAlloc(&hres, 4096, cudaHostAllocMapped));
    long long* dres;
    CK(cudaHostGetDevicePointer((void**)&dres, hres, 0));
    Big big;
    for (int i = 0; i < 800; ++i) big.v[i] = i;
    CK(cudaFuncSetAttribute(big_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608));
    CK(cudaFuncSetAttribute(small_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608));
    const int reps = 200;

    auto ev_time = [&](auto launch, bool spin_before) -> double {
        std::vector<double> t;
        for (int r = 0; r < reps + 10; ++r) {
            if (spin_before) spin_k<<<148, 32, 0, s>>>(400000);
            cudaEventRecord(a, s);
            launch();
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 10) t.push_back(ms * 1e3);
        }
        return median(t);
    };
    auto host_time = [&](auto launch) -> double {
        std::vector<double> t;
        for (int r = 0; r < reps + 10; ++r) {
            auto t0 = std::chrono::high_resolution_clock::now();
            launch();
            cudaStreamSynchronize(s);
            auto t1 = std::chrono::high_resolution_clock::now();
            if (r >= 10) t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        return median(t);
    };

    struct Case {
        const char* name;
        std::function<void()> f;
    };
    std::vector<std::pair<const char*, std::function<void()>>> cases = {
        {"empty 1x32", [&] { empty_k<<<1, 32, 0, s>>>(sink); }},
        {"empty 148x256", [&] { empty_k<<<148, 256, 0, s>>>(sink); }},
        {"empty 592x256", [&] { empty_k<<<592, 256, 0, s>>>(sink); }},
        {"6.4KB param 148x256", [&] { big_k<<<148, 256, 0, s>>>(big, (double*)sink); }},
        {"mapped result 148x256", [&] { mapped_k<<<148, 256, 0, s>>>(dres, 80); }},
        // the C2 TMA unit kernel's launch shape: 148 CTAs x 544 threads, 196 KB dynamic shared memory
        {"148x544 + 196KB smem + 6.4KB param", [&] { big_smem_k<<<148, 544, 196608, s>>>(big, (double*)sink); }},
        {"148x544 + 196KB smem", [&] { small_smem_k<<<148, 544, 196608, s>>>((double*)sink); }},
        {"148x544, no smem", [&] { small_smem_k<<<148, 544, 0, s>>>((double*)sink); }},
    };
    for (auto& c : cases) {
        printf("{\"case\": \"%s\", \"event_us\": %.2f, \"event_us_after_spin\": %.2f, \"host_roundtrip_us\": %.2f}\n",
               c.first, ev_time(c.second, false), ev_time(c.second, true), host_time(c.second));
    }
    // CUDA graph of the 6.4 KB-param kernel + mapped write
    {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        big_k<<<148, 256, 0, s>>>(big, (double*)sink);
        mapped_k<<<148, 256, 0, s>>>(dres, 80);
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        auto f = [&] { cudaGraphLaunch(ge, s); };
        printf("{\"case\": \"graph(6.4KB param + mapped)\", \"event_us\": %.2f, \"event_us_after_spin\": %.2f, "
               "\"host_roundtrip_us\": %.2f}\n",
               ev_time(f, false), ev_time(f, true), host_time(f));
        auto f2 = [&] {
            big_k<<<148, 256, 0, s>>>(big, (double*)sink);
            mapped_k<<<148, 256, 0, s>>>(dres, 80);
        };
        printf("{\"case\": \"stream(6.4KB param + mapped)\", \"event_us\": %.2f, \"event_us_after_spin\": %.2f, "
               "\"host_roundtrip_us\": %.2f}\n",
               ev_time(f2, false), ev_time(f2, true), host_time(f2));
    }
    // one kernel of the C2 launch shape as a single-node graph vs a stream launch
    {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        big_smem_k<<<148, 544, 196608, s>>>(big, (double*)sink);
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        auto f = [&] { cudaGraphLaunch(ge, s); };
        printf("{\"case\": \"graph(148x544 + 196KB smem + 6.4KB param)\", \"event_us\": %.2f, "
               "\"event_us_after_spin\": %.2f, \"host_roundtrip_us\": %.2f}\n",
               ev_time(f, false), ev_time(f, true), host_time(f));
        // the same graph with the kernel's 6.4 KB parameter block replaced before
        // every launch (what a per-call NLL launch through a cached graph does)
        cudaGraphNode_t nodes[4];
        size_t nn = 4;
        CK(cudaGraphGetNodes(g, nodes, &nn));
        cudaKernelNodeParams kp;
        CK(cudaGraphKernelNodeGetParams(nodes[0], &kp));
        Big big2 = big;
        double* sinkd = (double*)sink;
        void* args[2] = {&big2, &sinkd};
        kp.kernelParams = args;
        int flip = 0;
        auto fset = [&] {
            big2.v[0] = (double)(++flip);
            cudaGraphExecKernelNodeSetParams(ge, nodes[0], &kp);
            cudaGraphLaunch(ge, s);
        };
        printf("{\"case\": \"graph + SetParams each call (148x544 + 196KB smem + 6.4KB param)\", \"event_us\": %.2f, "
               "\"event_us_after_spin\": %.2f, \"host_roundtrip_us\": %.2f}\n",
               ev_time(fset, false), ev_time(fset, true), host_time(fset));
        // events inside the graph's stream order but around nothing: the event pair's own floor
        auto nothing = [&] {};
        printf("{\"case\": \"event pair around nothing\", \"event_us\": %.2f, \"event_us_after_spin\": %.2f}\n",
               ev_time(nothing, false), ev_time(nothing, true));
    }
    // persistent doorbell round trip (host write -> device poll -> mapped result -> host poll)
    {
        unsigned* hbell;
        CK(cudaHostAlloc(&hbell, 64, cudaHostAllocMapped));
        unsigned long long* hr;
        CK(cudaHostAlloc(&hr, 64, cudaHostAllocMapped));
        unsigned* dbell;
        unsigned long long* dr;
        CK(cudaHostGetDevicePointer((void**)&dbell, hbell, 0));
        CK(cudaHostGetDevicePointer((void**)&dr, hr, 0));
        *(volatile unsigned*)hbell = 0;
        *(volatile unsigned long long*)hr = 0;
        const int iters = reps + 10;
        persistent_k<<<1, 32, 0, s>>>(dbell, dr, iters);
        std::vector<double> t;
        for (int i = 1; i <= iters; ++i) {
            auto t0 = std::chrono::high_resolution_clock::now();
            *(volatile unsigned*)hbell = (unsigned)i;
            while (((*(volatile unsigned long long*)hr) >> 32) != (unsigned long long)i) {
            }
            auto t1 = std::chrono::high_resolution_clock::now();
            if (i > 10) t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        CK(cudaStreamSynchronize(s));
        printf("{\"case\": \"persistent doorbell round trip\", \"host_roundtrip_us\": %.2f}\n", median(t));
    }
    return 0;
}
