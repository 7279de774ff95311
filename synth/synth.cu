// synth.cu -- device twin of synth/__init__.py (seeded input generator).
// Holds none of the codec's arithmetic: only the counter-based splitmix64
// stream of DESIGN.md "Input recipe", so multi-GiB inputs (configs 3 and 5)
// can be generated in HBM without a host copy.  Checked bit-exact against the
// numpy generator by tests/test_gpu_parity.py::test_synth_device_matches_host.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// byte i (global) = (W[i/8] >> 8*(i%8)) & 0xff, W[j] = mix64(key + (j+1)*gamma)
__global__ void fill_kernel(uint8_t* __restrict__ d, int64_t n, uint64_t key, int64_t offset) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // head bytes until (offset + i) % 8 == 0
    const int64_t head = (8 - (offset & 7)) & 7;
    const int64_t h = head < n ? head : n;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < h) {
        const int64_t g = offset + t;
        d[t] = uint8_t(mix64(key + uint64_t(g / 8 + 1) * 0x9E3779B97F4A7C15ULL) >> (8 * (g & 7)));
    }
    const int64_t nw = (n - h) / 8;
    const int64_t j0 = (offset + h) / 8;
    const bool aligned = ((reinterpret_cast<uintptr_t>(d + h) & 7) == 0);
    for (int64_t w = t; w < nw; w += stride) {
        const uint64_t v = mix64(key + uint64_t(j0 + w + 1) * 0x9E3779B97F4A7C15ULL);
        uint8_t* p = d + h + 8 * w;
        if (aligned) {
            *reinterpret_cast<uint64_t*>(p) = v;
        } else {
            for (int k = 0; k < 8; ++k) p[k] = uint8_t(v >> (8 * k));
        }
    }
    const int64_t tail0 = h + 8 * nw;
    if (t < n - tail0) {
        const int64_t i = tail0 + t;
        const int64_t g = offset + i;
        d[i] = uint8_t(mix64(key + uint64_t(g / 8 + 1) * 0x9E3779B97F4A7C15ULL) >> (8 * (g & 7)));
    }
}

}  // namespace

extern "C" int synth_fill(uint8_t* d, int64_t n, uint64_t seed, uint64_t sid, int64_t offset, cudaStream_t s) {
    if (n <= 0) return 0;
    const uint64_t key = (seed << 32) + sid;
    int64_t blocks = (n / 8 + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_kernel<<<unsigned(blocks), 256, 0, s>>>(d, n, key, offset);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}
