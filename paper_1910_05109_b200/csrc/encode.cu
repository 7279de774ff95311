// encode.cu -- sm_100a base64 encode kernels (Sec. 2 / Sec. 3.1).
//
// enc_fast_kernel<D>: one stream, d_in 8-byte and d_out 32-byte aligned.
//   Warp-chunk = 768 input bytes (256 triples) -> 1024 chars.  Lane l owns
//   bytes [24l, 24l+24) = 8 triples -> 32 chars: three LDG.64 at a lane stride
//   of 24 B (together one contiguous 768 B range: the first brings every
//   sector into L1, the other two hit) and ONE lane-linear STG.256 (32 lanes x
//   32 B = 1 KiB, whole sectors).  Grid-stride over chunks with D chunks per
//   warp prefetched in registers (Little's law).  The
//   < 768 B remainder (full triples + the 1-2 byte padded tail, PAPER.md:84-87,
//   251) is done by the first threads of the grid, one output quad each.
// enc_generic_kernel: any alignment, one stream or a batch of strings
//   (BASELINE.json configs[3]).  The concatenated input is split into equal
//   byte ranges, one per warp; a warp encodes every 24-byte unit (8 triples ->
//   32 chars) whose first byte lies in its range, so long strings spread over
//   many warps and short strings pack many per warp.
#include <cstddef>

#include "b64_device.cuh"

namespace b64 {

__device__ __forceinline__ void enc_lane24(const uint8_t* __restrict__ src, uint32_t (&w)[6]) {
    const uint2 a = ld64_l1(src), b = ld64_l1(src + 8), c = ld64_l1(src + 16);
    w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y; w[4] = c.x; w[5] = c.y;
}

__device__ __forceinline__ void enc_lane_compute(const uint32_t (&w)[6], uint32_t (&o)[8], uint32_t lb) {
    o[0] = enc_triple_s(__byte_perm(w[0], w[1], 0x0122), lb);
    o[1] = enc_triple_s(__byte_perm(w[0], w[1], 0x3455), lb);
    o[2] = enc_triple_s(__byte_perm(w[1], w[2], 0x2344), lb);
    o[3] = enc_triple_s(__byte_perm(w[2], w[3], 0x1233), lb);
    o[4] = enc_triple_s(__byte_perm(w[3], w[4], 0x0122), lb);
    o[5] = enc_triple_s(__byte_perm(w[3], w[4], 0x3455), lb);
    o[6] = enc_triple_s(__byte_perm(w[4], w[5], 0x2344), lb);
    o[7] = enc_triple_s(__byte_perm(w[5], w[5], 0x1233), lb);
}

// The bulk loop of one stream as seen by one warp of a grouped launch
// (enc_group_kernel; enc_fast_kernel keeps its own copy): chunks c0, c0 + W, ... of
// the stream's C warp-chunks (768 B -> 1024 chars), D of them in flight in
// registers ahead of the one being encoded.  prime() issues the first loads
// (before the alphabet is staged, so the table set-up hides under the first
// DRAM latency); run() is the steady state.  int32 chunk indices (an
// HBM-resident stream has < 2^31 chunks) and pointers advanced by the stride:
// no 64-bit index math per chunk.
template <int D>
struct EncBulk {
    const uint8_t* pin;  // next chunk to load
    uint8_t* pout;       // next chunk to store
    int32_t c0, C, W;
    int64_t sin, sout;
    uint32_t wv[D][6];

    __device__ __forceinline__ void prime(const uint8_t* in, uint8_t* out, int32_t c0_, int32_t C_, int32_t W_,
                                          int lane) {
        c0 = c0_; C = C_; W = W_;
        sin = int64_t(W) * 768;
        sout = int64_t(W) * 1024;
        pin = in + int64_t(c0) * 768 + lane * 24;
        pout = out + int64_t(c0) * 1024 + lane * 32;
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (c0 + i * W < C) {
                enc_lane24(pin, wv[i]);
                pin += sin;
            }
    }
    __device__ __forceinline__ void run(uint32_t lb) {
        for (int32_t c = c0; c < C; c += D * W) {
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const int32_t ci = c + i * W;
                if (ci < C) {
                    uint32_t yv[6], o[8];
                    if (ci + D * W < C) {
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
};

template <int D>
__global__ void __launch_bounds__(kThreads)
enc_fast_kernel(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out, EncTab tab, uint32_t pad) {
    __shared__ __align__(64) uint32_t s_lut[16];
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int64_t nchunk = n / 768;
    const int64_t c0 = gtid >> 5;

    // Grid-stride over warp-chunks: at any moment the whole grid works on one
    // contiguous window of memory (DRAM row locality).  Software pipeline: D
    // chunks per warp are in flight ahead of the one being encoded.  The first
    // loads are issued before the alphabet is staged, so the table set-up
    // hides under the first DRAM latency.
    // int32 chunk indices (an HBM-resident stream has < 2^31 chunks) and
    // pointers advanced by the grid stride: no 64-bit index math per chunk.
    griddep_wait();
    const int32_t C = int32_t(nchunk), W = int32_t(nwarp), c0i = int32_t(c0);
    const int64_t sin = nwarp * 768, sout = nwarp * 1024;
    const uint8_t* pin = in + c0 * 768 + lane * 24;  // next chunk to load
    uint8_t* pout = out + c0 * 1024 + lane * 32;     // next chunk to store
    uint32_t wv[D][6];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (c0i + i * W < C) {
            enc_lane24(pin, wv[i]);
            pin += sin;
        }
    if (threadIdx.x == 0) {  // static indices: the table stays in the constant bank, no stack copy
#pragma unroll
        for (int i = 0; i < 16; ++i) s_lut[i] = tab.w[i];
    }
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    for (int32_t c = c0i; c < C; c += D * W) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int32_t ci = c + i * W;
            if (ci < C) {
                uint32_t yv[6], o[8];
                if (ci + D * W < C) {
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

    // remainder: output quads [256*nchunk, ceil(n/3)), one per thread
    const int64_t T = n / 3;
    const int64_t Q = (n + 2) / 3;
    for (int64_t q = nchunk * 256 + gtid; q < Q; q += gthreads) {
        const uint8_t* s = in + 3 * q;
        uint32_t word;
        if (q < T) {
            const uint32_t x = (uint32_t(s[0]) << 24) | (uint32_t(s[1]) << 16) | (uint32_t(s[2]) << 8);
            word = enc_triple(x, lut);
        } else {
            const int r = int(n - 3 * q);
            word = enc_partial(s[0], r == 2 ? s[1] : 0u, r, lut, pad);
        }
        *reinterpret_cast<uint32_t*>(out + 4 * q) = word;  // out 32-aligned => 4-aligned
    }
}

// The join of a streaming encode (stream.cu, R15), one thread: carry[0..H) are
// held input bytes (H <= 2), in[0..n) the new piece.  If H > 0 and H + n >= 3 the straddling
// triple carry ++ in[0 .. 3-H) is encoded to out[0..4).  The new carry is the last
// (H + n) % 3 bytes of carry ++ in (read before the old carry is overwritten).
__device__ __forceinline__ void enc_stream_join(uint8_t* carry, int H, const uint8_t* in, int64_t n, uint8_t* out,
                                                const uint8_t* lut) {
    const uint8_t c0 = carry[0], c1 = carry[1];
    auto at = [&](int64_t i) -> uint32_t { return i < H ? (i == 0 ? c0 : c1) : in[i - H]; };
    const int64_t A = H + n;
    const int R = int(A % 3);
    if (H > 0 && A >= 3) {
        const uint32_t v = enc_triple((at(0) << 24) | (at(1) << 16) | (at(2) << 8), lut);
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = uint8_t(v >> (8 * k));
    }
    for (int k = 0; k < R; ++k) carry[k] = uint8_t(at(A - R + k));
}

// ---------------------------------------------------------------- generic / batch

__device__ __forceinline__ void store16(uint8_t* dst, const uint32_t (&o)[4]) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(dst);
    if ((u & 15) == 0) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
    } else if ((u & 3) == 0) {
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        d[0] = o[0]; d[1] = o[1]; d[2] = o[2]; d[3] = o[3];
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[i] = uint8_t(o[i >> 2] >> (8 * (i & 3)));
    }
}

// Path B (output not 4-byte aligned: only the single-stream API with a
// misaligned d_out): 12-byte units -> 16 chars with byte-granular stores.
__device__ __forceinline__ void enc_string_unaligned_out(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                                         int64_t a, int64_t L, int64_t ob, int64_t lo, int64_t hi,
                                                         int lane, const uint8_t* __restrict__ lut, uint32_t pad) {
    const int64_t nunit = (L + 11) / 12;
    const int64_t kb = lo > a ? (lo - a + 11) / 12 : 0;
    const int64_t ke = min(nunit, (hi - a + 11) / 12);
    for (int64_t k = kb + lane; k < ke; k += 32) {
        const uint8_t* src = in + a + 12 * k;
        uint8_t* dst = out + ob + 16 * k;
        const int64_t rem = L - 12 * k;
        if (rem >= 12) {
            uint32_t wv[3], o[4];
            ld_unaligned<3>(src, wv);
            enc12(wv[0], wv[1], wv[2], o, lut);
            store16(dst, o);
        } else {
            int t = 0;
            for (; 3 * t + 3 <= rem; ++t) {
                const uint32_t x = (uint32_t(src[3 * t]) << 24) | (uint32_t(src[3 * t + 1]) << 16) |
                                   (uint32_t(src[3 * t + 2]) << 8);
                const uint32_t v = enc_triple(x, lut);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[4 * t + i] = uint8_t(v >> (8 * i));
            }
            const int r = int(rem - 3 * t);
            if (r > 0) {
                const uint32_t v = enc_partial(src[3 * t], r == 2 ? src[3 * t + 1] : 0u, r, lut, pad);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[4 * t + i] = uint8_t(v >> (8 * i));
            }
        }
    }
}

// A short string encoded whole by one lane (enc_generic_kernel): plain triples
// then the padded tail, 4-byte stores when the output is 4-byte aligned
// (always, in a batch).
#ifndef B64_SHORT_ENC
#define B64_SHORT_ENC 96
#endif
constexpr int64_t kShortEnc = B64_SHORT_ENC;  // bytes
__device__ __forceinline__ void enc_short_lane(const uint8_t* __restrict__ src, int64_t L, uint8_t* __restrict__ o,
                                               const uint8_t* __restrict__ lut, uint32_t pad) {
    const int64_t T = L / 3;
    const int r = int(L - 3 * T);
    const bool al = (reinterpret_cast<uintptr_t>(o) & 3) == 0;
    for (int64_t t = 0; t <= T; ++t) {
        uint32_t word;
        if (t < T) {
            word = enc_triple((uint32_t(src[3 * t]) << 24) | (uint32_t(src[3 * t + 1]) << 16) |
                              (uint32_t(src[3 * t + 2]) << 8), lut);
        } else if (r) {
            word = enc_partial(src[3 * t], r == 2 ? src[3 * t + 1] : 0u, r, lut, pad);
        } else {
            break;
        }
        if (al) {
            *reinterpret_cast<uint32_t*>(o + 4 * t) = word;
        } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) o[4 * t + b] = uint8_t(word >> (8 * b));
        }
    }
}

// Per-warp work lists of enc_generic_kernel (one 32-string batch at a time): the
// 24-byte units of the batch's long strings, flattened into one index space so the
// warp's lanes stay busy across string boundaries and the next unit's loads are in
// flight while the current one is encoded; then the scalar triples (heads, tails and
// padded partial triples) flattened the same way.
struct EncWarpList {
    int64_t pre[33];  // exclusive prefix of per-string item counts; pre[32] = total
    int64_t src[32];  // units: input offset of the string's first unit in range; scalars: string start
    int64_t dst[32];  // units: its output offset;  scalars: output offset of the string
    int32_t h[32];    // scalars: head triples, then the first tail triple and T (packed below)
    int32_t t0[32];
    int32_t T[32];
};

// The loads of one 24-byte unit at any alignment (the LDG.64 half of ld24_unaligned),
// kept raw so they can be issued one unit ahead; fix24 does the select / funnel half.
struct Raw24 {
    uint2 a, b, c, d;
    uint32_t sb;
};
__device__ __forceinline__ void ld24_raw(const uint8_t* p, Raw24& r) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const uint2* pa = reinterpret_cast<const uint2*>(u & ~uintptr_t(7));
    r.sb = uint32_t(u & 7);
    r.a = ld64_l1(pa);
    r.b = ld64_l1(pa + 1);
    r.c = ld64_l1(pa + 2);
    r.d = r.sb ? ld64_l1(pa + 3) : make_uint2(0u, 0u);
}
__device__ __forceinline__ void fix24(const Raw24& r, uint32_t (&w)[6]) {
    const uint32_t v[8] = {r.a.x, r.a.y, r.b.x, r.b.y, r.c.x, r.c.y, r.d.x, r.d.y};
    const bool ws = r.sb >= 4;
    const uint32_t sh = (r.sb & 3) * 8;
#pragma unroll
    for (int i = 0; i < 6; ++i) w[i] = __funnelshift_r(ws ? v[i + 1] : v[i], ws ? v[i + 2] : v[i + 1], sh);
}

__device__ __forceinline__ int64_t lds_s64(uint32_t a) {
    int64_t v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ int64_t warp_exclusive_scan(int64_t v, int lane, int64_t* total) {
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    *total = __shfl_sync(kFull, x, 31);
    return x - v;
}

// Any alignment, one stream or a batch.  The concatenated input is cut into
// equal byte ranges, one per warp; a warp owns every work item whose first
// input byte lies in its range.  Strings are visited 32 at a time (lane i
// holds string s0 + i's offsets):
//   * a short string (<= kShortEnc bytes) is encoded whole by its own lane;
//   * the long ones (output 4-byte aligned: always in a batch, whose output
//     offsets are multiples of 4) are split into h < 8 head triples that
//     bring the output to a 32-byte boundary, units of 8 triples (24 bytes,
//     read at any alignment as 8-byte-aligned LDG.64 + funnel shifts) -> 32
//     chars with one STG.256 (the same per-lane code as enc_fast_kernel), and
//     the < 8 tail triples + the padded partial triple; the units of all the
//     batch's long strings form ONE flattened list the warp sweeps with a
//     one-unit-ahead prefetch, the scalar triples a second one;
//   * a long string with a misaligned output (single-stream API only) takes
//     the byte-store path.
#ifndef B64_ENC_GEN_MINB
#define B64_ENC_GEN_MINB 5
#endif
__global__ void __launch_bounds__(kThreads, B64_ENC_GEN_MINB)
enc_generic_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, Offsets off, EncTab tab, uint32_t pad) {
    __shared__ __align__(64) uint32_t s_lut[16];
    __shared__ EncWarpList s_list[kThreads / 32];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) s_lut[i] = tab.w[i];
    }
    __syncthreads();
    griddep_wait();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);

    const int lane = threadIdx.x & 31;
    EncWarpList& wl = s_list[threadIdx.x >> 5];
    const int64_t W = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t base = off.in(0);
    const int64_t total = off.in(off.count) - base;
    if (total <= 0) return;
    const int64_t lo = base + (total * w) / W;
    const int64_t hi = base + (total * (w + 1)) / W;
    if (lo >= hi) return;

    for (int64_t s0 = first_string_ending_after(off, lo); s0 < off.count; s0 += 32) {
        const int64_t si = s0 + lane;
        const bool valid = si < off.count;
        int64_t ai = 0, Li = 0, obi = 0;
        if (valid) {
            ai = off.in(si);
            Li = off.in(si + 1) - ai;
            obi = off.out(si);
        }
        const bool started = valid && ai < hi;  // strings from hi on belong to later warps
        if (started && Li > 0 && Li <= kShortEnc && ai >= lo) enc_short_lane(in + ai, Li, out + obi, lut, pad);
        const bool lng = started && Li > kShortEnc;
        const bool lng_al = lng && ((reinterpret_cast<uintptr_t>(out + obi) & 3) == 0);
        // this lane's long string: units [kb, ke) whose first byte lies in [lo, hi)
        int64_t nu = 0, src = 0, dst = 0, ns = 0;
        int32_t h = 0, t0 = 0, T = 0;
        if (lng_al) {
            const uintptr_t oa = reinterpret_cast<uintptr_t>(out + obi);
            T = int32_t(Li / 3);
            const int r = int(Li - 3 * int64_t(T));
            h = int32_t(min(int64_t(T), int64_t(((32 - (oa & 31)) & 31) >> 2)));
            const int64_t U = (T - h) >> 3;
            const int64_t ua = ai + 3 * h;
            const int64_t kb = lo > ua ? (lo - ua + 23) / 24 : 0;
            const int64_t ke = min(U, (hi - ua + 23) / 24);
            nu = ke > kb ? ke - kb : 0;
            src = ua + 24 * kb;
            dst = obi + 4 * h + 32 * kb;
            t0 = int32_t(h + 8 * U);
            ns = h + (T - t0) + (r > 0 ? 1 : 0);  // scalar triples (range-checked per item)
        }
        int64_t nu_all;
        const int64_t pre = warp_exclusive_scan(nu, lane, &nu_all);
        wl.pre[lane] = pre;
        wl.src[lane] = src;
        wl.dst[lane] = dst;
        if (lane == 31) wl.pre[32] = nu_all;
        __syncwarp();
        // flattened units of the batch's long strings, one unit ahead in flight; each lane's
        // owner string only moves forward (j grows), so it is tracked, not searched
        // (the owner is tracked as the shared address of its pre[] entry: one register, and
        // no per-unit recomputation of the list's base under the 48-register cap)
        int64_t j = lane;
        uint32_t oa = smem_u32(&wl.pre[0]);
        constexpr uint32_t kSrc = offsetof(EncWarpList, src) - offsetof(EncWarpList, pre);
        constexpr uint32_t kDst = offsetof(EncWarpList, dst) - offsetof(EncWarpList, pre);
        Raw24 nr;
        int64_t ndst = 0;
        if (j < nu_all) {
            while (lds_s64(oa + 8) <= j) oa += 8;
            const int64_t po = lds_s64(oa);
            ld24_raw(in + lds_s64(oa + kSrc) + 24 * (j - po), nr);
            ndst = lds_s64(oa + kDst) + 32 * (j - po);
        }
        for (; j < nu_all; j += 32) {
            const Raw24 cr = nr;
            const int64_t cdst = ndst;
            const int64_t jn = j + 32;
            if (jn < nu_all) {
                while (lds_s64(oa + 8) <= jn) oa += 8;
                const int64_t po = lds_s64(oa);
                ld24_raw(in + lds_s64(oa + kSrc) + 24 * (jn - po), nr);
                ndst = lds_s64(oa + kDst) + 32 * (jn - po);
            }
            uint32_t wv[6], ov[8];
            fix24(cr, wv);
            enc_lane_compute(wv, ov, lb);
            st256(out + cdst, ov);
        }
        __syncwarp();
        // flattened scalar triples: head [0, h), tail [t0, T), and the padded partial triple T
        int64_t ns_all;
        const int64_t spre = warp_exclusive_scan(ns, lane, &ns_all);
        wl.pre[lane] = spre;
        wl.src[lane] = ai;
        wl.dst[lane] = obi;
        wl.h[lane] = h;
        wl.t0[lane] = t0;
        wl.T[lane] = T;
        if (lane == 31) wl.pre[32] = ns_all;
        __syncwarp();
        int os = 0;
        for (int64_t k = lane; k < ns_all; k += 32) {
            while (wl.pre[os + 1] <= k) ++os;
            const int o = os;
            const int32_t t = int32_t(k - wl.pre[o]);
            const int32_t ho = wl.h[o], To = wl.T[o];
            const int64_t tri = t < ho ? t : int64_t(wl.t0[o]) + (t - ho);  // == To for the partial triple
            const int64_t p = wl.src[o] + 3 * tri;
            if (p >= lo && p < hi) {
                const uint8_t* sp = in + p;
                uint32_t word;
                if (tri < To) {
                    word = enc_triple((uint32_t(sp[0]) << 24) | (uint32_t(sp[1]) << 16) | (uint32_t(sp[2]) << 8), lut);
                } else {
                    const int64_t L = off.in(s0 + o + 1) - wl.src[o];
                    const int r = int(L - 3 * int64_t(To));
                    word = enc_partial(sp[0], r == 2 ? sp[1] : 0u, r, lut, pad);
                }
                *reinterpret_cast<uint32_t*>(out + wl.dst[o] + 4 * tri) = word;
            }
        }
        __syncwarp();
        // long strings with a misaligned output (single-stream API): byte-granular path
        for (uint32_t mis = __ballot_sync(kFull, lng && !lng_al); mis; mis &= mis - 1) {
            const int jl = __ffs(mis) - 1;
            const int64_t a = __shfl_sync(kFull, ai, jl);
            const int64_t L = __shfl_sync(kFull, Li, jl);
            const int64_t ob = __shfl_sync(kFull, obi, jl);
            enc_string_unaligned_out(in, out, a, L, ob, lo, hi, lane, lut, pad);
        }
        if (__any_sync(kFull, !started)) break;  // a string at or after hi (or the end): done
    }
}

}  // namespace b64
