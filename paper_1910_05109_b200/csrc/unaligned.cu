// unaligned.cu -- the bulk decode for inputs / outputs at any byte alignment
// (dec_fastu_kernel): misaligned single calls, shards and, above all, the pieces
// of a streaming decode, whose quads start wherever the previous piece left off
// (R15) -- before, all of those took the per-unit generic kernel.
//
// Quad k of the text is at in + 4k, its 3 bytes at out + 3k.  The bulk starts at
// the first quad q0 whose OUTPUT is 8-byte aligned (q0 = 3 * (-out mod 8) mod 8
// < 8), so the chunks' 768-byte outputs are 8-byte aligned and go out exactly as
// in dec_fast_kernel (per-warp shared re-layout, lane-linear STG.64).  On the
// input side chunk c's 1024 chars start at in + 4 q0 + 1024 c, i.e. at word WS
// and byte b of an aligned 32-byte block (WS, b the same for every chunk): lane l
// loads its aligned block with ONE LDG.256, takes the next lane's first WS + 1
// words by SHFL (lane 31 loads the next block itself) and funnel-shifts its 8
// quads out of words WS .. WS + 8.  WS is a template parameter (8 kernels per
// prefetch depth; no dynamic register indexing), b a runtime shift.  The < 8
// quads before q0, the < 256 after the last full chunk and the final quad (R6)
// are done one per thread with byte loads.
#include "b64_device.cuh"

namespace b64 {

struct UnalignedBulk {
    const uint8_t* A0;  // aligned 32-byte block holding the first bulk quad's first byte
    uint8_t* out0;      // output of the first bulk quad (8-byte aligned)
    int64_t q0;         // quad index of the first bulk quad (= head quads, < 8)
    int32_t nchunk;     // full 256-quad chunks
    uint32_t b;         // in & 3
};

__device__ __forceinline__ uint32_t ld_u8x4(const uint8_t* p) {  // 4 bytes at any alignment
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

// The first NX words of the next aligned block, loaded only where `pred` (lane 31).
template <int NX>
__device__ __forceinline__ void ld_next_block(const uint8_t* p, bool pred, uint32_t (&w)[NX]) {
    if (NX == 8) {
        uint32_t t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (pred) ld256_stream(p, t);
#pragma unroll
        for (int k = 0; k < NX; ++k) w[k] = t[k & 7];
    } else {
        uint4 t = make_uint4(0, 0, 0, 0);
        if (pred) t = ld128_nc(p);
        w[0] = t.x; w[1 & (NX - 1)] = t.y; w[2 & (NX - 1)] = t.z; w[3 & (NX - 1)] = t.w;
    }
}

template <int D, int WS, bool EARLY>
__global__ void __launch_bounds__(kThreads, D == 1 ? 5 : 4)
dec_fastu_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab, int64_t base,
                 int is_final, unsigned long long* __restrict__ err_cell, int64_t* __restrict__ out_len,
                 UnalignedBulk ub, StreamJoin join) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];
    griddep_launch_dependents();
    if (!EARLY) griddep_wait();  // (EARLY: a B64_STREAM_OVERLAP piece -- the bulk runs before the wait)
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int64_t Q = m >> 2;
    const int64_t Qint = (is_final && Q > 0) ? Q - 1 : Q;
    const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);
    const uint32_t bsh = ub.b * 8;
    const bool need_next = (WS > 0) || (ub.b != 0);  // the last quad of a lane runs into the next block

    const int64_t c0 = gtid >> 5;
    const int32_t C = ub.nchunk, W = int32_t(nwarp), c0i = int32_t(c0);
    const int64_t sin = nwarp * 1024, sout = nwarp * 768;
    const uint8_t* pin = ub.A0 + c0 * 1024 + lane * 32;  // next block to load
    uint8_t* pout = ub.out0 + c0 * 768;
    int64_t cur = c0;                                    // chunk being decoded
    // lane 31 also loads the next aligned block (the next chunk's first), in ONE LDG.128 / LDG.256
    constexpr int NX = WS < 4 ? 4 : 8;
    const bool ld_next = need_next && lane == 31;
    uint32_t xr[D][8], xe[D][NX];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (c0i + i * W < C) {
            ld256_stream(pin, xr[i]);
            ld_next_block<NX>(pin + 32, ld_next, xe[i]);
            pin += sin;
        }
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    for (int32_t cb = c0i; cb < C; cb += D * W) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int32_t c = cb + i * W;
            if (c < C) {
                uint32_t y[8], ye[NX];
                if (c + D * W < C) {
                    ld256_stream(pin, y);
                    ld_next_block<NX>(pin + 32, ld_next, ye);
                    pin += sin;
                }
                // the lane's 8 quads: words WS .. WS + 8 of its block and the next one, shifted by b
                uint32_t nx[WS + 1];
#pragma unroll
                for (int k = 0; k <= WS; ++k) {
                    const uint32_t t = __shfl_down_sync(kFull, xr[i][k], 1);
                    nx[k] = lane == 31 ? xe[i][k] : t;
                }
                uint32_t err = 0, v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t lo = (WS + q < 8) ? xr[i][(WS + q) & 7] : nx[(WS + q - 8) & 7];
                    const uint32_t hi = (WS + q + 1 < 8) ? xr[i][(WS + q + 1) & 7] : nx[(WS + q + 1 - 8) & 7];
                    v[q] = dec_quad_s(__funnelshift_r(lo, hi, bsh), lb, err);
                }
                uint32_t o[6];
                dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
                dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
                sts64(sb + lane * 24, o[0], o[1]);
                sts64(sb + lane * 24 + 8, o[2], o[3]);
                sts64(sb + lane * 24 + 16, o[4], o[5]);
                __syncwarp();
                uint8_t* dst = pout + lane * 8;
                const uint2 s0 = lds64(sb + lane * 8), s1 = lds64(sb + 256 + lane * 8), s2 = lds64(sb + 512 + lane * 8);
                st64(dst, s0.x, s0.y);
                st64(dst + 256, s1.x, s1.y);
                st64(dst + 512, s2.x, s2.y);
                __syncwarp();
                const bool bad = (err & kInvalid) != 0;
                if (__any_sync(kFull, bad)) {  // rare: locate the first invalid char of the chunk
                    uint32_t rel = 0xffffffffu;
                    if (bad) {
                        const uint8_t* p = in + 4 * (ub.q0 + cur * 256) + lane * 32;
                        for (int t = 0; t < 32; ++t)
                            if (lut[p[t]] & kInvalid) { rel = uint32_t(lane * 32 + t); break; }
                    }
                    const uint32_t r = __reduce_min_sync(kFull, rel);
                    if (EARLY) griddep_wait();
                    if (lane == 0) atomicMin(err_cell, pack_err(base + 4 * (ub.q0 + cur * 256) + int64_t(r), kBadChar));
                }
                pout += sout;
                cur += W;
#pragma unroll
                for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
#pragma unroll
                for (int k = 0; k < NX; ++k) xe[i][k] = ye[k];
            }
        }
    }

    if (EARLY) griddep_wait();  // the previous piece done: the rest touches shared state
    // the head quads [0, q0), the quads after the last full chunk, one per thread (byte loads)
    const int64_t qt = ub.q0 + int64_t(C) * 256;
    const int64_t nh = ub.q0, nrest = nh + (Qint - qt);
    for (int64_t t = gtid; t < nrest; t += gthreads) {
        const int64_t q = t < nh ? t : qt + (t - nh);
        const uint32_t x = ld_u8x4(in + 4 * q);
        uint32_t err = 0;
        const uint32_t v = dec_quad(x, lut, err);
        store_bytes(out + 3 * q, v, 3);
        if (err & kInvalid) atomicMin(err_cell, pack_err(base + 4 * q + first_bad_in_quad(x, lut), kBadChar));
    }

    if (gtid == gthreads - 1) {
        if (is_final && Q > 0) {
            const int64_t q = Q - 1;
            int bad, k;
            uint32_t v;
            const uint32_t kind = final_quad(ld_u8x4(in + 4 * q), lut, tab.pad, tab.lenient, &bad, &k, &v);
            if (kind == kOk) store_bytes(out + 3 * q, v, k);
            else atomicMin(err_cell, pack_err(base + 4 * q + bad, kind));
            if (out_len) *out_len = 3 * q + k;
        } else if (out_len) {
            *out_len = 3 * Q;
        }
        if (join.active) stream_join(join.carry, join.H, join.in, join.m, join.out, lut, join.base, err_cell);
    }
}

// ---------------------------------------------------------------- encode at any input alignment
// enc_fastu_kernel: the encode of a stream whose input is not 8-byte aligned or whose output
// is 4- but not 32-byte aligned (misaligned single calls, shards, and above all the pieces of
// a streaming encode, whose triples start wherever the previous piece left off).  The bulk
// starts at the first triple q0 whose output is 32-byte aligned (q0 = (-out mod 32) / 4 < 8),
// so the chunks' 1024-char outputs go out as in enc_fast_kernel (one lane-linear STG.256 per
// lane).  Lane l's 24 input bytes of chunk c start at in + 3 q0 + 768 c + 24 l: the same
// offset sb within an 8-byte word for EVERY lane and chunk (768 and 24 are multiples of 8),
// so the loads are enc_fast's three LDG.64 at a 24-byte lane stride from the word-aligned
// base plus a fourth when sb != 0, and one warp-uniform funnel shift realigns them.  The < 8
// head triples, the < 256 after the last full chunk and the padded partial triple go one per
// thread.
// EARLY (an overlapped streaming piece, B64_STREAM_OVERLAP): the bulk runs before
// griddepcontrol.wait; after it, the rest and the join with the held bytes (`join`, which
// reads the carry the previous piece writes) by the last thread.
template <int D, bool EARLY>
__global__ void __launch_bounds__(kThreads)
enc_fastu_kernel(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out, EncTab tab, uint32_t pad,
                 int64_t q0, int32_t nchunk, EncJoin join) {
    __shared__ __align__(64) uint32_t s_lut[16];
    griddep_launch_dependents();
    if (!EARLY) griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const uintptr_t ib = reinterpret_cast<uintptr_t>(in) + 3 * uintptr_t(q0);
    const uint32_t sb = uint32_t(ib & 7);
    const bool wsh = sb >= 4;
    const uint32_t sh = (sb & 3) * 8;
    const int32_t C = nchunk, W = int32_t(nwarp), c0i = int32_t(gtid >> 5);
    const int64_t sin = nwarp * 768, sout = nwarp * 1024;
    const uint8_t* pin = reinterpret_cast<const uint8_t*>(ib & ~uintptr_t(7)) + int64_t(c0i) * 768 + lane * 24;
    uint8_t* pout = out + 4 * q0 + int64_t(c0i) * 1024 + lane * 32;
    uint2 xr[D][4];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (c0i + i * W < C) {
            xr[i][0] = ld64_l1(pin);
            xr[i][1] = ld64_l1(pin + 8);
            xr[i][2] = ld64_l1(pin + 16);
            xr[i][3] = sb ? ld64_l1(pin + 24) : make_uint2(0u, 0u);
            pin += sin;
        }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) s_lut[i] = tab.w[i];
    }
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    for (int32_t cb = c0i; cb < C; cb += D * W) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int32_t c = cb + i * W;
            if (c < C) {
                uint2 y[4];
                if (c + D * W < C) {
                    y[0] = ld64_l1(pin);
                    y[1] = ld64_l1(pin + 8);
                    y[2] = ld64_l1(pin + 16);
                    y[3] = sb ? ld64_l1(pin + 24) : make_uint2(0u, 0u);
                    pin += sin;
                }
                const uint32_t v[8] = {xr[i][0].x, xr[i][0].y, xr[i][1].x, xr[i][1].y,
                                       xr[i][2].x, xr[i][2].y, xr[i][3].x, xr[i][3].y};
                uint32_t w[6], o[8];
#pragma unroll
                for (int k = 0; k < 6; ++k) w[k] = __funnelshift_r(wsh ? v[k + 1] : v[k], wsh ? v[k + 2] : v[k + 1], sh);
                enc_lane_compute(w, o, lb);
                st256(pout, o);
                pout += sout;
#pragma unroll
                for (int k = 0; k < 4; ++k) xr[i][k] = y[k];
            }
        }
    }
    if (EARLY) griddep_wait();  // the previous piece done: its carry is written
    // the head triples [0, q0), the triples after the last full chunk and the padded partial
    // triple, one output word per thread (out 4-byte aligned)
    const int64_t T = n / 3, Q = (n + 2) / 3;
    const int64_t qt = q0 + int64_t(C) * 256;
    const int64_t nrest = q0 + (Q - qt);
    for (int64_t t = gtid; t < nrest; t += gthreads) {
        const int64_t q = t < q0 ? t : qt + (t - q0);
        const uint8_t* sp = in + 3 * q;
        uint32_t word;
        if (q < T) {
            word = enc_triple((uint32_t(sp[0]) << 24) | (uint32_t(sp[1]) << 16) | (uint32_t(sp[2]) << 8), lut);
        } else {
            const int r = int(n - 3 * q);
            word = enc_partial(sp[0], r == 2 ? sp[1] : 0u, r, lut, pad);
        }
        *reinterpret_cast<uint32_t*>(out + 4 * q) = word;
    }
    if (EARLY && join.active && gtid == gthreads - 1)
        enc_stream_join(join.carry, join.H, join.in, join.n, join.out, lut);
}

// (D, WS) -> kernel
using DecFastuFn = void (*)(const uint8_t*, int64_t, uint8_t*, DecTab, int64_t, int, unsigned long long*, int64_t*,
                            UnalignedBulk, StreamJoin);
template <int D, bool EARLY = false>
DecFastuFn dec_fastu_pick(int ws) {
    switch (ws) {
        case 0: return dec_fastu_kernel<D, 0, EARLY>;
        case 1: return dec_fastu_kernel<D, 1, EARLY>;
        case 2: return dec_fastu_kernel<D, 2, EARLY>;
        case 3: return dec_fastu_kernel<D, 3, EARLY>;
        case 4: return dec_fastu_kernel<D, 4, EARLY>;
        case 5: return dec_fastu_kernel<D, 5, EARLY>;
        case 6: return dec_fastu_kernel<D, 6, EARLY>;
        default: return dec_fastu_kernel<D, 7, EARLY>;
    }
}

}  // namespace b64
