// scripts/exp_stream_ubench.cu -- microbenchmark for DESIGN §6: stream N doubles with a
// plain grid-stride kernel, per-event exp (table + polynomial, as EvSum2GE), unit
// product + log per 16 events; no certificates, no exact fold.  Compares the
// instruction budget of the production C1 kernels with a bare-minimum kernel.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o scripts/exp_stream_ubench scripts/exp_stream_ubench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>
__constant__ double kTab[64];
constexpr double kExpK = 92.33248261689366;
constexpr double kLn2o64Hi = 0x1.62e42fee00000p-7;
constexpr double kLn2o64Lo = 0x1.a39ef35793c76p-39;
__device__ __forceinline__ double cexp(double d, const double* tab, double a) {
    const double t = fma(d, kExpK, 0x1.8p52);
    const int k = __double2loint(t);
    const double kd = t - 0x1.8p52;
    double r = fma(kd, -kLn2o64Hi, d);
    r = fma(kd, -kLn2o64Lo, r);
    double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    const double tv = tab[k & 63];
    const double cs = __hiloint2double(__double2hiint(tv) + ((k >> 6) << 20), __double2loint(tv));
    return fma(cs, q, a);
}
template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const double* __restrict__ x, long n, double mu, double c2, double al, double amu, double c1, double* out) {
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = kTab[threadIdx.x] * 0.7;
    __syncthreads();
    double acc = 0.0;
    const long nunits = n / 16;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < nunits; u += (long)gridDim.x * blockDim.x) {
        // unit u: 16 events, 8 rows of 2 (coalesced: row r at u-block offset)
        const long wbase = (u / 32) * 512 + (u % 32) * 2;
        double m = 1.0, ls = 0.0;
        int ex = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(x + wbase + r * 64));
            if (MODE == 0) { m = m * (1.0 + v.x * 1e-9) * (1.0 + v.y * 1e-9); ls += v.x + v.y; }
            else {
                double w0 = v.x - mu, w1 = v.y - mu;
                double d0 = fma(w0, fma(c2, w0, -al), -amu), d1 = fma(w1, fma(c2, w1, -al), -amu);
                double q0 = cexp(d0, tab, c1), q1 = cexp(d1, tab, c1);
                m = (m * q0) * q1;
                ls = (ls + v.x) + v.y;
                if (r & 1) { int hi = __double2hiint(m); ex += (hi >> 20) - 1023; m = __hiloint2double((hi & 0xfffff) | 0x3ff00000, __double2loint(m)); }
            }
        }
        acc += log(m) + ls * al + ex * 0.6931471805599453;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}
template <int MODE, int MINB>
float run(const double* x, long n, double* out, int grid, int reps, void* flush) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9, tot = 0; int cnt = 0;
    for (int i = 0; i < reps + 3; ++i) {
        cudaMemsetAsync(flush, i, 256 << 20);
        cudaEventRecord(a);
        k<MODE, MINB><<<grid, 256>>>(x, n, 5.0, -2.0, -0.3, -1.5, 0.4, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (i >= 3) { tot += ms; ++cnt; if (ms < best) best = ms; }
    }
    return tot / cnt * 1000.0f;
}
int main() {
    double h[64]; for (int j = 0; j < 64; ++j) h[j] = exp2(j / 64.0);
    cudaMemcpyToSymbol(kTab, h, sizeof h);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (long n : {1000000L, 10000000L, 40000000L}) {
        n = n / 8192 * 8192;
        double* x; cudaMalloc(&x, n * 8); double* out; cudaMalloc(&out, 8);
        void* flush; cudaMalloc(&flush, 256 << 20);
        double* hx = new double[n]; for (long i = 0; i < n; ++i) hx[i] = 5.0 + ((i * 2654435761L) % 1000) * 0.003;
        cudaMemcpy(x, hx, n * 8, cudaMemcpyHostToDevice); delete[] hx;
        for (int g : {sms * 2, sms * 4, sms * 8}) {
            printf("n %ld grid %d  nocompute(minb4) %.2f us  exp(minb2) %.2f  exp(minb3) %.2f  exp(minb4) %.2f\n", n, g,
                   run<0, 4>(x, n, out, g, 20, flush), run<1, 2>(x, n, out, g, 20, flush), run<1, 3>(x, n, out, g, 20, flush),
                   run<1, 4>(x, n, out, g, 20, flush));
        }
        cudaFree(x); cudaFree(out); cudaFree(flush);
    }
    // empty kernel
    return 0;
}
