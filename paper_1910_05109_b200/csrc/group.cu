// group.cu -- grouped launches: up to kGroupMax independent streams (each with
// its own alphabet, length, input and output) encoded or decoded by ONE kernel.
//
// A launch has a fixed cost (~3-4 us on B200: CTA launch, first DRAM latency,
// tail) that a 64 MiB op (~25 us of HBM time) does not amortise; one grid that
// sweeps the concatenated chunk space of several streams pays it once
// (DESIGN.md "Grouped launches").  Per stream the work is exactly the single
// stream kernels' (enc_fast_kernel / dec_fast_kernel): same per-lane code, same
// warp-chunk split, same tail / final-quad / error handling.
#include "b64_device.cuh"

namespace b64 {

constexpr int kGroupMax = 8;

struct EncGroup {
    const uint8_t* in[kGroupMax];
    uint8_t* out[kGroupMax];
    int64_t n[kGroupMax];
    int64_t cstart[kGroupMax + 1];  // exclusive scan of warp-chunks per stream
    uint32_t pad[kGroupMax];
    uint32_t lut[kGroupMax][16];    // enc[64] per stream
    int count;
};

struct DecGroup {
    const uint8_t* in[kGroupMax];
    uint8_t* out[kGroupMax];
    int64_t m[kGroupMax];
    int64_t base[kGroupMax];
    unsigned long long* cell[kGroupMax];
    int64_t cstart[kGroupMax + 1];
    int32_t is_final[kGroupMax];
    uint32_t pad[kGroupMax];
    uint32_t lut[kGroupMax][64];    // dec[256] per stream
    int count;
};

// Monotone cursor over the concatenated chunk space of a group.  A warp visits
// chunks c0, c0 + W, c0 + 2W, ... so the owning stream only moves forward:
// `next` is one compare and one pointer add per chunk; the stream's base
// pointer is re-read from the parameter bank only when a stream boundary is
// crossed (a per-chunk search cost ~35 % more instructions, profiles/).
template <int UNIT, bool IN>
struct GroupCursor {
    int it;
    int32_t lo, hi;   // chunk range [lo, hi) of stream it (a group holds < 2^31 chunks)
    const uint8_t* p; // address of the current chunk (+ the lane offset)
    template <typename G>
    __device__ __forceinline__ void locate(const G& g, int32_t c, int lane_off) {
        while (c >= hi && it + 1 < g.count) {
            ++it;
            lo = hi;
            hi = int32_t(g.cstart[it + 1]);
        }
        p = (IN ? g.in[it] : static_cast<const uint8_t*>(g.out[it])) + int64_t(c - lo) * UNIT + lane_off;
    }
    template <typename G>
    __device__ __forceinline__ void start(const G& g, int32_t c, int lane_off) {
        it = 0;
        lo = int32_t(g.cstart[0]);
        hi = int32_t(g.cstart[1]);
        locate(g, c, lane_off);
    }
    template <typename G>
    __device__ __forceinline__ void next(const G& g, int32_t c, int64_t step, int lane_off) {
        if (c < hi) p += step;
        else locate(g, c, lane_off);
    }
};

template <int D>
__global__ void __launch_bounds__(kThreads) enc_group_kernel(const __grid_constant__ EncGroup g) {
    __shared__ __align__(64) uint32_t s_lut[kGroupMax][16];
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int32_t W = int32_t(nwarp), w = int32_t(gtid >> 5);
    const int64_t sin = nwarp * 768, sout = nwarp * 1024;

    griddep_wait();
    if (threadIdx.x < g.count * 16) (&s_lut[0][0])[threadIdx.x] = (&g.lut[0][0])[threadIdx.x];
    __syncthreads();
    const uint32_t lb0 = smem_u32(&s_lut[0][0]);

    // Stream by stream, the warp walks the chunks c == w (mod W) of the
    // concatenated chunk space -- within a stream exactly enc_fast_kernel's
    // loop (pointer increments, D chunks prefetched in registers).
    for (int it = 0; it < g.count; ++it) {
        const int32_t lo = int32_t(g.cstart[it]), hi = int32_t(g.cstart[it + 1]);
        const int32_t first = lo + int32_t((int64_t(w) - lo % W + W) % W);
        if (first >= hi) continue;
        const int32_t nloc = (hi - first + W - 1) / W;  // chunks of this stream for this warp
        const uint8_t* pin = g.in[it] + int64_t(first - lo) * 768 + lane * 24;
        uint8_t* pout = g.out[it] + int64_t(first - lo) * 1024 + lane * 32;
        const uint32_t lb = lb0 + 64 * it;
        uint32_t wv[D][6];
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (i < nloc) {
                enc_lane24(pin, wv[i]);
                pin += sin;
            }
        for (int32_t k = 0; k < nloc; k += D) {
#pragma unroll
            for (int i = 0; i < D; ++i) {
                if (k + i < nloc) {
                    uint32_t yv[6], o[8];
                    if (k + i + D < nloc) {
                        enc_lane24(pin, yv);
                        pin += sin;
                    }
                    enc_lane_compute(wv[i], o, lb);
                    st256(pout, o);
                    pout += sout;
#pragma unroll
                    for (int j = 0; j < 6; ++j) wv[i][j] = yv[j];
                }
            }
        }
    }

    // per-stream remainder quads (whole triples + the padded tail), one per thread
    for (int it = 0; it < g.count; ++it) {
        const int64_t n = g.n[it];
        const int64_t T = n / 3, Q = (n + 2) / 3;
        const uint8_t* in = g.in[it];
        const uint8_t* lut = reinterpret_cast<const uint8_t*>(&s_lut[it][0]);
        for (int64_t q = (g.cstart[it + 1] - g.cstart[it]) * 256 + gtid; q < Q; q += gthreads) {
            const uint8_t* s = in + 3 * q;
            uint32_t word;
            if (q < T) {
                word = enc_triple((uint32_t(s[0]) << 24) | (uint32_t(s[1]) << 16) | (uint32_t(s[2]) << 8), lut);
            } else {
                const int r = int(n - 3 * q);
                word = enc_partial(s[0], r == 2 ? s[1] : 0u, r, lut, g.pad[it]);
            }
            *reinterpret_cast<uint32_t*>(g.out[it] + 4 * q) = word;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads) dec_group_kernel(const __grid_constant__ DecGroup g) {
    __shared__ __align__(256) uint32_t s_lut[kGroupMax][64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int32_t C = int32_t(g.cstart[g.count]);
    const int32_t c0 = int32_t(gtid >> 5);
    const int32_t W = int32_t(nwarp);
    const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);
    GroupCursor<1024, true> pre;  // input of the chunk being prefetched
    GroupCursor<768, false> cur;  // output of the chunk being decoded

    griddep_wait();
    uint32_t xr[D][8];
    if (c0 < C) {
        pre.start(g, c0, lane * 32);
        cur.start(g, c0, lane * 8);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const int32_t c = c0 + j * W;
        if (c < C) {
            if (j) pre.next(g, c, nwarp * 1024, lane * 32);
            ld256_stream(pre.p, xr[j]);
        }
    }
    for (int t = threadIdx.x; t < g.count * 64; t += blockDim.x) (&s_lut[0][0])[t] = (&g.lut[0][0])[t];
    __syncthreads();
    const uint32_t lb0 = smem_u32(&s_lut[0][0]);

    for (int32_t cb = c0; cb < C; cb += D * W) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const int32_t c = cb + j * W;
            if (c < C) {
                uint32_t y[8];
                const int32_t cn = c + D * W;
                if (cn < C) {
                    pre.next(g, cn, nwarp * 1024, lane * 32);
                    ld256_stream(pre.p, y);
                }
                if (c != c0) cur.next(g, c, nwarp * 768, lane * 8);
                const int it = cur.it;
                const uint32_t lb = lb0 + 256 * it;
                uint32_t err = 0, v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(xr[j][q], lb, err);
                uint32_t o[6];
                dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
                dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
                sts64(sb + lane * 24, o[0], o[1]);
                sts64(sb + lane * 24 + 8, o[2], o[3]);
                sts64(sb + lane * 24 + 16, o[4], o[5]);
                __syncwarp();
                uint8_t* dst = const_cast<uint8_t*>(cur.p);
                const uint2 s0 = lds64(sb + lane * 8), s1 = lds64(sb + 256 + lane * 8), s2 = lds64(sb + 512 + lane * 8);
                st64(dst, s0.x, s0.y);
                st64(dst + 256, s1.x, s1.y);
                st64(dst + 512, s2.x, s2.y);
                __syncwarp();
                const bool bad = (err & kInvalid) != 0;
                if (__any_sync(kFull, bad)) {
                    const uint8_t* lut = reinterpret_cast<const uint8_t*>(&s_lut[it][0]);
                    const int64_t lc = int64_t(c - cur.lo);
                    uint32_t rel = 0xffffffffu;
                    if (bad) {
                        rel = scan_first_bad(g.in[it] + lc * 1024 + lane * 32, 8, lut);
                        if (rel != 0xffffffffu) rel += lane * 32;
                    }
                    warp_report(bad, rel, g.base[it] + lc * 1024, g.cell[it]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) xr[j][k] = y[k];
            }
        }
    }

    // per-stream leftover interior quads, then the final quad (grid's last thread)
    for (int it = 0; it < g.count; ++it) {
        const uint8_t* lut = reinterpret_cast<const uint8_t*>(&s_lut[it][0]);
        const int64_t Q = g.m[it] >> 2;
        const int64_t Qint = (g.is_final[it] && Q > 0) ? Q - 1 : Q;
        const uint8_t* in = g.in[it];
        uint8_t* out = g.out[it];
        for (int64_t q = (g.cstart[it + 1] - g.cstart[it]) * 256 + gtid; q < Qint; q += gthreads) {
            const uint32_t x = ld32(in + 4 * q);
            uint32_t err = 0;
            const uint32_t v = dec_quad(x, lut, err);
            store_bytes(out + 3 * q, v, 3);
            if (err & kInvalid)
                atomicMin(g.cell[it], pack_err(g.base[it] + 4 * q + first_bad_in_quad(x, lut), kBadChar));
        }
        if (gtid == gthreads - 1 && g.is_final[it] && Q > 0) {
            const int64_t q = Q - 1;
            int bad, k;
            uint32_t v;
            const uint32_t kind = final_quad(ld32(in + 4 * q), lut, g.pad[it], &bad, &k, &v);
            if (kind == kOk) store_bytes(out + 3 * q, v, k);
            else atomicMin(g.cell[it], pack_err(g.base[it] + 4 * q + bad, kind));
        }
    }
}

// Packed error words -> (err_off, status) for count streams.
__global__ void dec_finalize_n_kernel(const int64_t* cells, int64_t count, int64_t* err_off, int32_t* status) {
    griddep_wait();
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long wv = static_cast<unsigned long long>(cells[i]);
        if (wv >= kErrNone) {
            err_off[i] = -1;
            if (status) status[i] = kOk;
        } else {
            err_off[i] = int64_t(wv >> 3);
            if (status) status[i] = int32_t(wv & 7);
        }
    }
}

}  // namespace b64
