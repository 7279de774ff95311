// unaligned.cu -- the bulk decode for inputs / outputs at any byte alignment
// (dec_fastu_kernel): misaligned single calls, shards and, above all, the pieces
// of a streaming decode, whose quads start wherever the previous piece left off
// (R15) -- before, all of those took the per-unit generic kernel.
//
// Input.  The quads start at in + 4k, b = in & 3.  An aligned 32-byte block A
// holds the first bytes of exactly 8 quads (those starting at A + b + 4j), the
// last of which runs b bytes into the next block.  So the bulk is cut into
// aligned 1024-byte warp-chunks starting at A0 = align_up(in - b, 32): lane l
// loads its block with ONE LDG.256 exactly as dec_fast_kernel, takes the next
// lane's first word with one SHFL (lane 31 loads it: one extra LDG.32 per
// chunk, only when b != 0) and funnel-shifts the 8 quads out of the 9 words.
// The h < 8 quads before A0 + b, the < 256 after the last full chunk and the
// final quad (R6) are done one per thread with byte loads.
//
// Output.  A chunk's 768 bytes land at out_c = out + 3*(quad index), whose
// alignment os = out_c & 7 is the same for every chunk (768 = 96 * 8).  The
// lanes' 24-byte results are re-laid through the warp's shared buffer shifted
// by os bytes (funnel shifts; each lane's spill word is merged into the next
// lane's first word with one SHFL), so shared byte i is global byte
// (out_c & ~7) + i: the 96 (or 95) whole 8-byte words go out as lane-linear
// STG.64 exactly as in dec_fast_kernel, the two partial boundary words (shared
// with the neighbouring chunks) as aligned 1 / 2 / 4-byte stores.
#include "b64_device.cuh"

namespace b64 {

struct UnalignedBulk {
    const uint8_t* A0;  // first aligned block of the bulk
    uint8_t* out0;      // output of the first bulk quad
    int64_t q0;         // stream quad index of the first bulk quad (= head quads h)
    int32_t nchunk;     // full 256-quad chunks
    uint32_t b;         // in & 3
};

__device__ __forceinline__ uint32_t ld_u8x4(const uint8_t* p) {  // 4 bytes at any alignment
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

// Bytes [lo, hi) of the aligned 8-byte word at g (value wv, little-endian) as aligned
// 1 / 2 / 4-byte stores: the edge words a chunk shares with its neighbours.
__device__ __forceinline__ void partial_store(uint8_t* g, uint2 wv, uint32_t lo, uint32_t hi) {
    const unsigned long long v = (static_cast<unsigned long long>(wv.y) << 32) | wv.x;
    uint32_t t = lo;
    if ((t & 1) && t < hi) { g[t] = uint8_t(v >> (8 * t)); t += 1; }
    if ((t & 2) && t + 2 <= hi) { *reinterpret_cast<uint16_t*>(g + t) = uint16_t(v >> (8 * t)); t += 2; }
    if ((t & 3) == 0 && t + 4 <= hi) { *reinterpret_cast<uint32_t*>(g + t) = uint32_t(v >> (8 * t)); t += 4; }
    if ((t & 1) == 0 && t + 2 <= hi) { *reinterpret_cast<uint16_t*>(g + t) = uint16_t(v >> (8 * t)); t += 2; }
    if (t < hi) g[t] = uint8_t(v >> (8 * t));
}

template <int D>
__global__ void __launch_bounds__(kThreads)
dec_fastu_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab, int64_t base,
                 int is_final, unsigned long long* __restrict__ err_cell, int64_t* __restrict__ out_len,
                 UnalignedBulk ub, StreamJoin join) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][776 / 4];
    griddep_launch_dependents();
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int64_t Q = m >> 2;
    const int64_t Qint = (is_final && Q > 0) ? Q - 1 : Q;
    const uint32_t sbase = smem_u32(&s_stage[threadIdx.x >> 5][0]);
    const uint32_t bsh = ub.b * 8;
    const uint32_t os = uint32_t(reinterpret_cast<uintptr_t>(ub.out0) & 7);
    const uint32_t osr = (os & 3) * 8;

    const int64_t c0 = gtid >> 5;
    const int32_t C = ub.nchunk, W = int32_t(nwarp), c0i = int32_t(c0);
    const int64_t sin = nwarp * 1024, sout = nwarp * 768;
    const uint8_t* pin = ub.A0 + c0 * 1024 + lane * 32;  // next block to load
    int64_t cur = c0;                                    // chunk being decoded
    uint32_t xr[D][8], xe[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (c0i + i * W < C) {
            ld256_stream(pin, xr[i]);
            xe[i] = (bsh && lane == 31) ? ld32(pin + 32) : 0u;
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
                uint32_t y[8], ye = 0;
                if (c + D * W < C) {
                    ld256_stream(pin, y);
                    ye = (bsh && lane == 31) ? ld32(pin + 32) : 0u;
                    pin += sin;
                }
                // the lane's 8 quads: bytes [b, b + 32) of its block and the next one
                uint32_t err = 0, v[8];
                if (bsh) {
                    const uint32_t nx = __shfl_down_sync(kFull, xr[i][0], 1);
                    const uint32_t w8 = lane == 31 ? xe[i] : nx;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        v[q] = dec_quad_s(__funnelshift_r(xr[i][q], q < 7 ? xr[i][q + 1] : w8, bsh), lb, err);
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(xr[i][q], lb, err);
                }
                uint32_t o[6];
                dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
                dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
                // shared byte os + 24 lane + j <- output byte j of this lane (a shift by os)
                uint32_t s[7];
                s[0] = __funnelshift_l(0u, o[0], osr);
#pragma unroll
                for (int k = 1; k < 6; ++k) s[k] = __funnelshift_l(o[k - 1], o[k], osr);
                s[6] = __funnelshift_l(o[5], 0u, osr);
                const uint32_t spill = __shfl_up_sync(kFull, s[6], 1);
                if (lane > 0) s[0] |= spill;
                const uint32_t wa = sbase + (os >> 2) * 4 + lane * 24;
                if (os < 4) {  // 8-byte aligned lane slots: three STS.64 (as dec_fast_kernel)
                    sts64(wa, s[0], s[1]);
                    sts64(wa + 8, s[2], s[3]);
                    sts64(wa + 16, s[4], s[5]);
                } else {
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(wa), "r"(s[0]) : "memory");
                    sts64(wa + 4, s[1], s[2]);
                    sts64(wa + 12, s[3], s[4]);
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(wa + 20), "r"(s[5]) : "memory");
                }
                if (lane == 31) asm volatile("st.shared.u32 [%0], %1;" ::"r"(wa + 24), "r"(s[6]) : "memory");
                __syncwarp();
                // global: word k of the chunk's aligned window = shared bytes [8k, 8k + 8)
                uint8_t* g = ub.out0 + cur * 768 - os;  // 8-byte aligned
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int k = lane + 32 * j;
                    const uint2 wv = lds64(sbase + 8 * k);
                    if (k > 0 || os == 0) st64(g + 8 * k, wv.x, wv.y);
                }
                if (os) {  // the two partial words at the chunk's edges, shared with its neighbours:
                           // bytes [os, 8) of word 0 and [0, os) of word 96, in 1 / 2 / 4-byte stores
                    if (lane == 0) {
                        const uint2 wv = lds64(sbase);
                        partial_store(g, wv, os, 8);
                    } else if (lane == 31) {
                        const uint2 wv = lds64(sbase + 768);
                        partial_store(g + 768, wv, 0, os);
                    }
                }
                __syncwarp();
                const bool bad = (err & kInvalid) != 0;
                if (__any_sync(kFull, bad)) {  // rare: locate the first invalid char of the chunk
                    uint32_t rel = 0xffffffffu;
                    if (bad) {
                        const uint8_t* p = ub.A0 + cur * 1024 + lane * 32 + ub.b;
                        for (int t = 0; t < 32; ++t)
                            if (lut[p[t]] & kInvalid) { rel = uint32_t(lane * 32 + t); break; }
                    }
                    const uint32_t r = __reduce_min_sync(kFull, rel);
                    if (lane == 0) atomicMin(err_cell, pack_err(base + 4 * (ub.q0 + cur * 256) + int64_t(r), kBadChar));
                }
                cur += W;
#pragma unroll
                for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
                xe[i] = ye;
            }
        }
    }

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

}  // namespace b64
