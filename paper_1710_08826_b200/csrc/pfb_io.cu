// pfb_io.cu -- binary SoA event ingest straight into device columns
// (SURVEY 8(f) row 3).
//
// The reference reads events from CSV through Python lists (dataio.py:20-83,
// core.py:259-282).  For 100M-event runs each observable is kept as one
// little-endian float64 .npy column; pfb_store_load_npy streams any row range
// of it (a GPU's shard) from the file into a device column through two pinned
// staging buffers, so file reads overlap the host-to-device copies and no
// host copy of the data is ever materialised.  The reference's strict range
// check (core.py:262-272: x < lower, x > upper or non-finite -> OutOfRange at
// the first such row) runs on the device (pfb_store_check_range).
#include <fcntl.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "pfb_internal.cuh"

namespace pfb {

// Parses the .npy header: 1-D, '<f8', C order.  Returns the data offset.
int npy_parse(int fd, int64_t* n_out, int64_t* data_off) {
    unsigned char pre[12];
    if (pread(fd, pre, 10, 0) != 10) return -1;
    if (memcmp(pre, "\x93NUMPY", 6) != 0) return -1;
    const int major = pre[6];
    int64_t hlen, hoff;
    if (major == 1) {
        hlen = pre[8] | (pre[9] << 8);
        hoff = 10;
    } else if (major == 2 || major == 3) {
        if (pread(fd, pre, 12, 0) != 12) return -1;
        hlen = (int64_t)pre[8] | ((int64_t)pre[9] << 8) | ((int64_t)pre[10] << 16) | ((int64_t)pre[11] << 24);
        hoff = 12;
    } else {
        return -1;
    }
    if (hlen <= 0 || hlen > (1 << 20)) return -1;
    std::string h(hlen, '\0');
    if (pread(fd, &h[0], hlen, hoff) != hlen) return -1;
    auto has = [&](const char* s) { return h.find(s) != std::string::npos; };
    if (!(has("'descr': '<f8'") || has("'descr':'<f8'"))) return -1;
    if (!has("'fortran_order': False") && !has("'fortran_order':False")) return -1;
    const size_t sp = h.find("'shape':");
    if (sp == std::string::npos) return -1;
    const size_t lp = h.find('(', sp), rp = h.find(')', sp);
    if (lp == std::string::npos || rp == std::string::npos || rp < lp) return -1;
    const std::string dims = h.substr(lp + 1, rp - lp - 1);  // "N," for 1-D
    const size_t comma = dims.find(',');
    if (comma == std::string::npos || dims.find_first_not_of(" ", comma + 1) != std::string::npos) return -1;
    char* end = nullptr;
    const long long n = strtoll(dims.c_str(), &end, 10);
    if (n < 0) return -1;
    *n_out = n;
    *data_off = hoff + hlen;
    return 0;
}

__global__ void range_check_kernel(const double* x, int64_t n, double lo, double hi, unsigned long long* first) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (v < lo || v > hi || !isfinite(v)) atomicMin(first, (unsigned long long)i);
    }
}

cudaError_t launch_range_check(const double* x, int64_t n, double lo, double hi, unsigned long long* first,
                               cudaStream_t stream, int sm_count) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
    range_check_kernel<<<(unsigned)grid, 256, 0, stream>>>(x, n, lo, hi, first);
    return cudaGetLastError();
}

}  // namespace pfb
