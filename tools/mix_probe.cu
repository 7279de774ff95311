// mix_probe.cu -- HBM bandwidth of pure streaming kernels by read:write mix
// (DESIGN.md "Kernels and their rooflines").  Not part of the product: a
// yardstick for the codec kernels, whose traffic is 3:4 (encode: n read,
// 4n/3 written) and 4:3 (decode).  Each kernel is grid-stride over warp
// "rounds"; a round reads R x 512 B and writes W x 512 B with lane-linear
// 16-byte vectors (whole sectors), D rounds of loads in flight per warp.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_probe tools/mix_probe.cu
//   ./mix_probe [GiB=1]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1); } } while (0)

template <int R, int W, int U = 4>
__global__ void __launch_bounds__(256) mix_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                  long rounds) {
    const int lane = threadIdx.x & 31;
    const long warp = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long nwarp = (long(gridDim.x) * blockDim.x) >> 5;
    uint4 acc = make_uint4(0, 0, 0, 0);
    // U rounds per iteration (warp, warp + nwarp, ...): all their loads are issued first
    for (long r0 = warp; r0 < rounds; r0 += U * nwarp) {
        uint4 v[U][R > 0 ? R : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long r = r0 + u * nwarp;
#pragma unroll
            for (int i = 0; i < R; ++i) v[u][i] = r < rounds ? in[(r * R + i) * 32 + lane] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long r = r0 + u * nwarp;
#pragma unroll
            for (int i = 0; i < R; ++i) { acc.x ^= v[u][i].x; acc.y += v[u][i].y; acc.z ^= v[u][i].z; acc.w += v[u][i].w; }
            if (r < rounds) {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    uint4 o = acc;
                    o.x += j;
                    out[(r * W + j) * 32 + lane] = o;
                }
            }
        }
    }
    if (R > 0 && W == 0 && acc.x == 0x12345678u && acc.y == 0x9abcdef0u) out[0] = acc;  // keep the loads alive
}

template <int R, int W>
double run(const uint4* in, uint4* out, long bytes_budget, int sms, int bps) {
    const long per_round = long(R + W) * 512;
    const long rounds = bytes_budget / per_round;
    const int blocks = sms * bps;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int it = 0; it < 12; ++it) {
        CK(cudaEventRecord(a));
        mix_kernel<R, W><<<blocks, 256>>>(in, out, rounds);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it >= 2 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return double(rounds * per_round) / (best * 1e-3) / 1e9;
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? std::atof(argv[1]) : 1.0;
    const long budget = long(gib * (1L << 30)) * 2;  // read + write bytes per launch
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint4 *in, *out;
    CK(cudaMalloc(&in, budget));
    CK(cudaMalloc(&out, budget));
    CK(cudaMemset(in, 1, budget));
    CK(cudaMemset(out, 0, budget));
    std::printf("{\"traffic_bytes\": %ld, \"results_gbs\": {", budget);
    for (int bps : {4, 6, 8}) {
        std::printf("%s\"bps%d\": {\"read\": %.1f, \"write\": %.1f, \"copy_1_1\": %.1f, \"enc_3_4\": %.1f, "
                    "\"dec_4_3\": %.1f}",
                    bps == 4 ? "" : ", ", bps, run<1, 0>(in, out, budget, sms, bps), run<0, 1>(in, out, budget, sms, bps),
                    run<1, 1>(in, out, budget, sms, bps), run<3, 4>(in, out, budget, sms, bps),
                    run<4, 3>(in, out, budget, sms, bps));
    }
    std::printf("}}\n");
    return 0;
}
