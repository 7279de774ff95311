// small.cu -- single-launch validating decode for small inputs (SURVEY.md
// Sec. 8(f) f1, the paper's small-input regime).
//
// b64_decode_ex on a large input is three stream operations: initialise the
// error word, the bulk kernel (whose CTAs lower it with atomicMin), and a
// one-thread finalize.  For inputs up to kSmallMax chars the whole call is ONE
// launch of a thread-block CLUSTER (up to 16 CTAs, one per SM): each CTA keeps
// its first error in shared memory, the cluster barriers, and CTA 0 gathers
// the 16 minima through distributed shared memory (DSMEM) and writes
// err_off / status / out_len itself -- no global scratch, no init, no second
// kernel.  The per-chunk work is dec_fast_kernel's (same per-lane code).
#include <cooperative_groups.h>

#include "b64_device.cuh"

namespace b64 {

namespace cg = cooperative_groups;

#ifndef B64_SMALL_THREADS
#define B64_SMALL_THREADS 512
#endif
constexpr int kSmallThreads = B64_SMALL_THREADS;  // 16 warps per CTA (1024 measured slower below 1 MiB)
constexpr int kSmallCluster = 16;                // CTAs (non-portable cluster size, one per SM)
constexpr int64_t kSmallMax = int64_t(512) << 10;  // chars handled by the single-launch path (tools/small_sweep.py)

__global__ void __launch_bounds__(kSmallThreads)
dec_small_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab,
                 int64_t* __restrict__ err_off, int32_t* __restrict__ status, int64_t* __restrict__ out_len) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(128) uint32_t s_stage[kSmallThreads / 32][768 / 4];
    __shared__ unsigned long long s_min;
    cg::cluster_group cluster = cg::this_cluster();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    if (threadIdx.x == 0) s_min = kErrNone;
    griddep_wait();
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);

    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // grid == one cluster
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int32_t W = int32_t(gthreads >> 5);
    const int64_t Q = m >> 2;
    const int64_t Qint = Q > 0 ? Q - 1 : 0;
    const int32_t C = int32_t(Qint >> 8);

    // one chunk per warp in flight ahead of the one being translated (the data is
    // usually L2-resident here: latency, not bandwidth, bounds a 16-SM grid)
    uint32_t xn[8];
    int32_t c = int32_t(gtid >> 5);
    if (c < C) ld256_stream(in + int64_t(c) * 1024 + lane * 32, xn);
    for (; c < C; c += W) {
        uint32_t x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = xn[j];
        const uint8_t* src = in + int64_t(c) * 1024 + lane * 32;
        if (c + W < C) ld256_stream(src + int64_t(W) * 1024, xn);
        uint32_t err = 0, v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(x[q], lb, err);
        uint32_t o[6];
        dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
        dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
        sts64(sb + lane * 24, o[0], o[1]);
        sts64(sb + lane * 24 + 8, o[2], o[3]);
        sts64(sb + lane * 24 + 16, o[4], o[5]);
        __syncwarp();
        uint8_t* dst = out + int64_t(c) * 768 + lane * 8;
        const uint2 s0 = lds64(sb + lane * 8), s1 = lds64(sb + 256 + lane * 8), s2 = lds64(sb + 512 + lane * 8);
        st64(dst, s0.x, s0.y);
        st64(dst + 256, s1.x, s1.y);
        st64(dst + 512, s2.x, s2.y);
        __syncwarp();
        const bool bad = (err & kInvalid) != 0;
        if (__any_sync(kFull, bad)) {
            uint32_t rel = 0xffffffffu;
            if (bad) {
                rel = scan_first_bad(src, 8, lut);
                if (rel != 0xffffffffu) rel += lane * 32;
            }
            const uint32_t r = __reduce_min_sync(kFull, bad ? rel : 0xffffffffu);
            if (lane == 0) atomicMin(&s_min, pack_err(int64_t(c) * 1024 + r, kBadChar));
        }
    }
    for (int64_t q = (int64_t(C) << 8) + gtid; q < Qint; q += gthreads) {
        const uint32_t x = ld32(in + 4 * q);
        uint32_t err = 0;
        const uint32_t v = dec_quad(x, lut, err);
        store_bytes(out + 3 * q, v, 3);
        if (err & kInvalid) atomicMin(&s_min, pack_err(4 * q + first_bad_in_quad(x, lut), kBadChar));
    }
    int k_final = 3;
    if (gtid == gthreads - 1 && Q > 0) {
        const int64_t q = Q - 1;
        int bad;
        uint32_t v;
        const uint32_t kind = final_quad(ld32(in + 4 * q), lut, tab.pad, tab.lenient, &bad, &k_final, &v);
        if (kind == kOk) store_bytes(out + 3 * q, v, k_final);
        else atomicMin(&s_min, pack_err(4 * q + bad, kind));
    }

    // cluster-wide minimum through DSMEM; CTA 0 writes the results
    cluster.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long mn = kErrNone;
        for (unsigned r = 0; r < cluster.num_blocks(); ++r) {
            const unsigned long long v = *cluster.map_shared_rank(&s_min, r);
            mn = v < mn ? v : mn;
        }
        if (mn >= kErrNone) {
            *err_off = -1;
            if (status) *status = kOk;
            if (out_len) {
                int64_t ol = 3 * Q;
                if (Q > 0) ol -= (in[m - 2] == tab.pad) ? 2 : (in[m - 1] == tab.pad ? 1 : 0);
                *out_len = ol;
            }
        } else {
            const int64_t pos = int64_t(mn >> 3);
            *err_off = pos;
            if (status) *status = int32_t(mn & 7);
            if (out_len) *out_len = 3 * (pos >> 2);
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
    (void)k_final;
}

}  // namespace b64
