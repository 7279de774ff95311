// decode.cu -- sm_100a validating base64 decode kernels (Sec. 2, 3.2).
//
// dec_fast_kernel<D>: one stream (or one shard of it), d_in 32-byte and d_out
//   16-byte aligned.  Warp-chunk = 1024 chars (256 quads) -> 768 bytes.  Lane l
//   owns chars [32l, 32l+32): ONE lane-linear LDG.256 (whole sectors, fully
//   coalesced); its 24 output bytes go through a per-warp shared buffer so the
//   global stores are three lane-linear STG.64 of whole sectors.  Every lane
//   ORs its translated values into one register (the paper's error register,
//   PAPER.md:305-313); the warp votes once per chunk and only on a set 0x80
//   bit locates the first bad char (__reduce_min_sync + one 64-bit atomicMin
//   of the packed word pos<<3|kind).  Interior quads left over after the
//   chunks go one per thread; the stream's final quad (padding, R6)
//   is done by the grid's last thread -- "a final and separate code path"
//   (PAPER.md:569).
// dec_generic_kernel: any alignment, one stream or a batch of strings.
//   Same byte-range-per-warp split as enc_generic_kernel with 32-char units
//   -> 24 bytes; per string, h < 8 head quads make every unit's output 8-byte
//   aligned (3 STG.64).
// dec_finalize_*: map the packed error word to (err_off, status, out_len).
#include "b64_device.cuh"

namespace b64 {

__device__ __forceinline__ void warp_report(bool bad, uint32_t rel, int64_t pos0, unsigned long long* cell) {
    // rel: position of this lane's first bad char relative to pos0 (only read if bad)
    const uint32_t r = __reduce_min_sync(kFull, bad ? rel : 0xffffffffu);
    if ((threadIdx.x & 31) == 0) atomicMin(cell, pack_err(pos0 + int64_t(r), kBadChar));
}

// Rare path: position (0 .. 4*nquads-1) of the first invalid char of the
// nquads quads at p (4-byte aligned), re-read from global memory, or ~0u.
__device__ __forceinline__ uint32_t scan_first_bad(const uint8_t* p, int nquads, const uint8_t* __restrict__ lut) {
    for (int q = 0; q < nquads; ++q) {
        const int j = first_bad_in_quad(ld32(p + 4 * q), lut);
        if (j < 4) return uint32_t(4 * q + j);
    }
    return 0xffffffffu;
}

// The bulk loop of one stream as seen by one warp of a grouped launch
// (dec_group_kernel): chunks c0, c0 + W, ... of the stream's C warp-chunks
// (1024 chars -> 768 bytes), D of them in flight in registers ahead of the one
// being translated.  prime() issues the first loads
// (before the table is staged); run() is the steady state.  The 24-byte lane
// outputs are re-laid through the warp's shared buffer sb (conflict-free
// STS.64 at a 24 B stride) so the global stores are lane-linear STG.64 writing
// whole sectors.  Positions reported to `cell` are base + char index.  The
// per-lane work is dec_fast_kernel's; that kernel keeps its own copy of the
// loop, whose loop-invariant bounds ptxas keeps in uniform registers (the
// shared struct form measured 3.5 % slower at 1 GiB there, profiles/).
template <int D>
struct DecBulk {
    const uint8_t* pin;   // next chunk to load
    const uint8_t* pcur;  // chunk being decoded (rare error rescan)
    uint8_t* pout;        // its output
    int32_t c0, C, W;
    uint32_t zero;  // 0 at run time, opaque to the compiler (see run())
    int64_t sin, sout;
    uint32_t xr[D][8];

    __device__ __forceinline__ void prime(const uint8_t* in, uint8_t* out, int32_t c0_, int32_t C_, int32_t W_,
                                          int lane, uint32_t zero_) {
        c0 = c0_; C = C_; W = W_; zero = zero_;
        sin = int64_t(W) * 1024;
        sout = int64_t(W) * 768;
        pin = in + int64_t(c0) * 1024 + lane * 32;
        pcur = pin;
        pout = out + int64_t(c0) * 768;
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (c0 + i * W < C) {
                ld256_stream(pin, xr[i]);
                pin += sin;
            }
    }
    __device__ __forceinline__ void run(uint32_t lb, const uint8_t* __restrict__ lut, uint32_t sb, int lane,
                                        int64_t base, unsigned long long* cell) {
        for (int32_t cb = c0; cb < C; cb += D * W) {
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const int32_t c = cb + i * W;
                if (c < C) {
                    uint32_t err = 0, v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(xr[i][q], lb, err);
                    uint32_t o[6];
                    dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
                    dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
                    // The prefetch is issued once xr[i] is consumed: its address carries a
                    // dependency on the translated values (err & zero, zero == 0 at run
                    // time but opaque to ptxas), so it cannot be hoisted above the 32
                    // lookups (hoisted, it keeps 8 more registers live under the
                    // 48-register cap: 2.5 % slower on 6 x 1 GiB groups).
                    uint32_t y[8];
                    if (c + D * W < C) {
                        ld256_stream(pin + (err & zero), y);
                        pin += sin;
                    }
                    sts64(sb + lane * 24, o[0], o[1]);
                    sts64(sb + lane * 24 + 8, o[2], o[3]);
                    sts64(sb + lane * 24 + 16, o[4], o[5]);
                    __syncwarp();
                    uint8_t* dst = pout + lane * 8;
                    const uint2 s0 = lds64(sb + lane * 8), s1 = lds64(sb + 256 + lane * 8),
                                s2 = lds64(sb + 512 + lane * 8);
                    st64(dst, s0.x, s0.y);
                    st64(dst + 256, s1.x, s1.y);
                    st64(dst + 512, s2.x, s2.y);
                    __syncwarp();
                    const bool bad = (err & kInvalid) != 0;
                    if (__any_sync(kFull, bad)) {  // rare: locate the first invalid char of the chunk
                        uint32_t rel = 0xffffffffu;
                        if (bad) {
                            rel = scan_first_bad(pcur, 8, lut);
                            if (rel != 0xffffffffu) rel += lane * 32;
                        }
                        warp_report(bad, rel, base + int64_t(c) * 1024, cell);
                    }
                    pout += sout;
                    pcur += sin;
#pragma unroll
                    for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
                }
            }
        }
    }
};

// The join of a streaming decode (stream.cu, R15), one thread: the held chars
// + the piece's head -> one quad, and the piece's last R chars -> the carry.
__device__ __forceinline__ void stream_join(uint8_t* carry, int H, const uint8_t* in, int64_t m, uint8_t* out,
                                            const uint8_t* lut, int64_t base, unsigned long long* cell) {
    uint8_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = carry[k];
    auto at = [&](int64_t i) -> uint32_t { return i < H ? c[i] : in[i - H]; };
    const int64_t A = H + m;
    if (A == 0) return;
    const int64_t Q = (A - 1) / 4;
    const int R = int(A - 4 * Q);
    if (H > 0 && Q >= 1) {
        const uint32_t x = at(0) | (at(1) << 8) | (at(2) << 16) | (at(3) << 24);
        uint32_t err = 0;
        const uint32_t v = dec_quad(x, lut, err);
        store_bytes(out, v, 3);
        if (err & kInvalid) atomicMin(cell, pack_err(base + first_bad_in_quad(x, lut), kBadChar));
    }
    for (int k = 0; k < R; ++k) carry[k] = uint8_t(at(A - R + k));
}

template <int D, bool EARLY>
__global__ void __launch_bounds__(kThreads)
dec_fast_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab,
                int64_t base, int is_final, unsigned long long* __restrict__ err_cell,
                int64_t* __restrict__ out_len, const int64_t* __restrict__ m_dev, StreamJoin join) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];  // per-warp output staging
    griddep_launch_dependents();
    if (!EARLY) {  // (EARLY: a B64_STREAM_OVERLAP piece -- the bulk runs before the wait)
        griddep_wait();
        // D = 1 (the launches of <= 64 MiB): the laundered m_dev makes the stream's pointers
        // per-thread values, which ptxas schedules better here -- measured 64 MiB pieces 0.51 ->
        // 0.46 ms per GiB; at D = 2 (1 GiB) the uniform-register version is 6 % faster
        // (0.393 vs 0.418 ms).  Either way m_dev is read after the wait (test_pdl_order.py).
        if (D == 1) m_dev = after_wait(m_dev);
    }
    if (m_dev) {  // the compacted text of mime.cu: its length and the kept index its suffix starts at
        const int64_t k0 = m_dev[1];
        m = m_dev[0] - k0;
        in += k0;
        out += 3 * (k0 >> 2);
        base += k0;
    }
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int64_t Q = m >> 2;
    const int64_t Qint = (is_final && Q > 0) ? Q - 1 : Q;
    const int64_t nchunk = Qint >> 8;
    const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);

    // Bulk: grid-stride over warp-chunks (1024 chars -> 768 bytes), so the
    // whole grid sweeps one contiguous window of memory at a time.  Software
    // pipeline: D chunks per warp are in flight ahead of the one being
    // translated (the first ones are issued before the table is staged).  The
    // 24-byte lane outputs are re-laid through a per-warp shared buffer
    // (conflict-free STS.64 at a 24 B stride) so the global stores are
    // lane-linear STG.64 writing whole sectors.
    // int32 chunk indices and pointers advanced by the grid stride.
    const int64_t c0 = gtid >> 5;
    const int32_t C = int32_t(nchunk), W = int32_t(nwarp), c0i = int32_t(c0);
    const int64_t sin = nwarp * 1024, sout = nwarp * 768;
    const uint8_t* pin = in + c0 * 1024 + lane * 32;  // next chunk to load
    const uint8_t* pcur = in + c0 * 1024 + lane * 32; // chunk being decoded (rare error rescan)
    uint8_t* pout = out + c0 * 768;                   // its output
    uint32_t xr[D][8];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (c0i + i * W < C) {
            ld256_stream(pin, xr[i]);
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
                uint32_t y[8];
                if (c + D * W < C) {
                    ld256_stream(pin, y);
                    pin += sin;
                }
                uint32_t err = 0, v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(xr[i][q], lb, err);
                uint32_t o[6];
                dec_pack12(v[0], v[1], v[2], v[3], o[0], o[1], o[2]);
                dec_pack12(v[4], v[5], v[6], v[7], o[3], o[4], o[5]);
                sts64(sb + lane * 24, o[0], o[1]);
                sts64(sb + lane * 24 + 8, o[2], o[3]);
                sts64(sb + lane * 24 + 16, o[4], o[5]);
                __syncwarp();
                uint8_t* dst = pout + lane * 8;
                const uint2 s0 = lds64(sb + lane * 8), s1 = lds64(sb + 256 + lane * 8),
                            s2 = lds64(sb + 512 + lane * 8);
                st64(dst, s0.x, s0.y);
                st64(dst + 256, s1.x, s1.y);
                st64(dst + 512, s2.x, s2.y);
                __syncwarp();
                const bool bad = (err & kInvalid) != 0;
                if (__any_sync(kFull, bad)) {  // rare: locate the first invalid char of the chunk
                    uint32_t rel = 0xffffffffu;
                    if (bad) {
                        rel = scan_first_bad(pcur, 8, lut);
                        if (rel != 0xffffffffu) rel += lane * 32;
                    }
                    if (EARLY) griddep_wait();
                    warp_report(bad, rel, base + int64_t(c) * 1024, err_cell);
                }
                pout += sout;
                pcur += sin;
#pragma unroll
                for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
            }
        }
    }

    if (EARLY) griddep_wait();  // the previous piece done: the rest touches shared state
    // leftover interior quads, one per thread
    for (int64_t q = (nchunk << 8) + gtid; q < Qint; q += gthreads) {
        const uint32_t x = ld32(in + 4 * q);
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
            const uint32_t kind = final_quad(ld32(in + 4 * q), lut, tab.pad, tab.lenient, &bad, &k, &v);
            if (kind == kOk) store_bytes(out + 3 * q, v, k);
            else atomicMin(err_cell, pack_err(base + 4 * q + bad, kind));
            if (out_len) *out_len = 3 * q + k;
        } else if (out_len) {
            *out_len = 3 * Q;
        }
        if (join.active) stream_join(join.carry, join.H, join.in, join.m, join.out, lut, join.base, err_cell);
    }
}


// ---------------------------------------------------------------- generic / batch

// A short string decoded whole by one lane (dec_generic_kernel): interior
// quads, then the final quad when `fin` (R6 / R16); the first error
// is reported and ends the string.  Chars are read as naturally aligned
// 4-byte words + funnel shifts (src has any alignment); output bytes are
// gathered in a 64-bit register and written as aligned 4-byte words (one
// store per 4 bytes instead of 3 byte stores per quad), the unaligned head
// and tail byte by byte.
#ifndef B64_SHORT_DEC
#define B64_SHORT_DEC 128
#endif
constexpr int64_t kShortDec = B64_SHORT_DEC;  // chars
__device__ __forceinline__ void dec_short_lane(const uint8_t* __restrict__ src, int64_t L, uint8_t* __restrict__ o,
                                               const uint8_t* __restrict__ lut, uint32_t pad, uint32_t lenient,
                                               bool fin, int64_t pbase, unsigned long long* cell) {
    const int64_t Qs = L >> 2;
    const uintptr_t su = reinterpret_cast<uintptr_t>(src);
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(su & ~uintptr_t(3));
    const uint32_t sh = uint32_t(su & 3) * 8;
    uint32_t w0 = ld32(sw);
    // output: bytes before the first 4-byte boundary go one by one
    int64_t pos = 0;                                            // output bytes emitted
    const int head = int((4 - (reinterpret_cast<uintptr_t>(o) & 3)) & 3);
    unsigned long long acc = 0;                                 // pending bytes, little-endian
    int nacc = 0;
    auto emit = [&](uint32_t v, int k) {                        // k bytes of v in stream order (v>>16, v>>8, v)
        for (int b = 0; b < k; ++b) {
            const uint32_t byte = (v >> (16 - 8 * b)) & 0xffu;
            if (pos < head) {
                o[pos++] = uint8_t(byte);
            } else {
                acc |= (unsigned long long)byte << (8 * nacc);
                if (++nacc == 4) {
                    *reinterpret_cast<uint32_t*>(o + pos) = uint32_t(acc);
                    pos += 4;
                    acc = 0;
                    nacc = 0;
                }
            }
        }
    };
    int64_t q = 0;
    for (; q < Qs; ++q) {
        const uint32_t w1 = (sh || q + 1 < Qs) ? ld32(sw + q + 1) : 0u;  // never past the string's last word
        const uint32_t x = sh ? __funnelshift_r(w0, w1, sh) : w0;
        w0 = w1;
        if (fin && q == Qs - 1) {
            int bad, k;
            uint32_t v;
            const uint32_t kind = final_quad(x, lut, pad, lenient, &bad, &k, &v);
            if (kind == kOk) emit(v, k);
            else atomicMin(cell, pack_err(pbase + 4 * q + bad, kind));
            break;
        }
        uint32_t err = 0;
        const uint32_t v = dec_quad(x, lut, err);
        if (err & kInvalid) {
            atomicMin(cell, pack_err(pbase + 4 * q + first_bad_in_quad(x, lut), kBadChar));
            break;
        }
        emit(v, 3);
    }
    for (int b = 0; b < nacc; ++b) o[pos + b] = uint8_t(acc >> (8 * b));  // tail bytes
}

// Batch: err cell per string, positions relative to the string start.
// Single: one cell, positions base + offset; is_final as given.
#ifndef B64_GEN_MINB
#define B64_GEN_MINB 5
#endif
__global__ void __launch_bounds__(kThreads, B64_GEN_MINB)
dec_generic_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, Offsets off, DecTab tab,
                   int64_t base, int is_final_single, unsigned long long* __restrict__ err_cells,
                   int64_t* __restrict__ out_len_single, const BatchCtx* gate) {
    __shared__ __align__(256) uint32_t s_lut[64];
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    const bool batch = off.in_off != nullptr;
    griddep_wait();
    if (gate && !gate->generic) return;  // the batch's concatenation path did it all (batch.cu)

    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;

    if (!batch && out_len_single && w == 0 && lane == 0) {
        // bytes written assuming the chunk is valid
        const int64_t Q = off.n >> 2;
        int64_t ol = 3 * Q;
        if (is_final_single && Q > 0) {
            const uint8_t c2 = in[off.n - 2], c3 = in[off.n - 1];
            ol -= (c2 == tab.pad) ? 2 : (c3 == tab.pad ? 1 : 0);
        }
        *out_len_single = ol;
    }

    const int64_t first = off.in(0);
    const int64_t total = off.in(off.count) - first;
    if (total <= 0) return;
    const int64_t lo = first + (total * w) / W;
    const int64_t hi = first + (total * (w + 1)) / W;
    if (lo >= hi) return;

    // Strings are visited 32 at a time (lane i holds string s0 + i's offsets): a short string
    // (<= kShortDec chars) is decoded whole by its own lane -- by the warp whose range holds
    // its first char -- and the longer ones one after the other by the whole warp (every
    // unit whose first char lies in [lo, hi)).  Empty strings and len % 4 != 0 (LENGTH) are
    // settled by the finalize kernel.
    const bool fin = batch ? true : (is_final_single != 0);
    const int64_t pbase = batch ? 0 : base;  // reported position = pbase + (char index in string)
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
      const bool ok_len = Li > 0 && (Li & 3) == 0;
      if (started && ok_len && Li <= kShortDec && ai >= lo)
          dec_short_lane(in + ai, Li, out + obi, lut, tab.pad, tab.lenient, fin, pbase,
                         batch ? err_cells + si : err_cells);
      for (uint32_t longs = __ballot_sync(kFull, started && ok_len && Li > kShortDec); longs; longs &= longs - 1) {
        const int jl = __ffs(longs) - 1;
        const int64_t s = s0 + jl;
        const int64_t a = __shfl_sync(kFull, ai, jl);
        const int64_t L = __shfl_sync(kFull, Li, jl);
        const int64_t ob = __shfl_sync(kFull, obi, jl);
        uint8_t* o = out + ob;
        unsigned long long* cell = batch ? err_cells + s : err_cells;
        const int64_t Qs = L >> 2;
        const int64_t Qint = fin ? Qs - 1 : Qs;
        // h head quads make the unit outputs 8-byte aligned: 3h == -o (mod 8), 3^-1 == 3 (mod 8)
        const int64_t h = min(int64_t(((8 - (reinterpret_cast<uintptr_t>(o) & 7)) * 3) & 7), Qint);
        const int64_t U = (Qint - h) >> 3;       // full 8-quad units (32 chars -> 24 bytes)
        const int64_t ua = a + 4 * h;             // first char of unit 0
        const int64_t kb = lo > ua ? (lo - ua + 31) / 32 : 0;
        const int64_t ke = min(U, (hi - ua + 31) / 32);
        for (int64_t k0 = kb; k0 < ke; k0 += 32) {
            const int64_t k = k0 + lane;
            const bool act = k < ke;
            uint32_t err = 0;
            if (act) {
                uint32_t x[8], v[8], ov[6];
                ld32_unaligned128(in + ua + 32 * k, x);
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(x[q], lb, err);
                dec_pack12(v[0], v[1], v[2], v[3], ov[0], ov[1], ov[2]);
                dec_pack12(v[4], v[5], v[6], v[7], ov[3], ov[4], ov[5]);
                uint8_t* dst = o + 3 * h + 24 * k;
                st64(dst, ov[0], ov[1]);
                st64(dst + 8, ov[2], ov[3]);
                st64(dst + 16, ov[4], ov[5]);
            }
            const bool bad = act && (err & kInvalid);
            if (__any_sync(kFull, bad)) {
                uint32_t rel = 0xffffffffu;
                if (bad) {
                    const uint8_t* src = in + ua + 32 * k;
                    for (int c = 0; c < 32; ++c) {
                        if (lut[src[c]] & kInvalid) { rel = uint32_t(lane * 32 + c); break; }
                    }
                }
                warp_report(bad, rel, pbase + (ua - a) + 32 * k0, cell);
            }
        }
        // quads outside full units: head [0,h), tail [h+8U, Qint), final Qs-1 (at most 15)
        const int64_t t0 = h + 8 * U;
        const int64_t ntail = Qint - t0;
        const int nsc = int(h + ntail + (fin ? 1 : 0));
        if (lane < nsc) {
            int64_t j;
            if (lane < h) j = lane;
            else if (lane < h + ntail) j = t0 + (lane - h);
            else j = Qs - 1;
            const int64_t p = a + 4 * j;
            if (p >= lo && p < hi) {
                const uint8_t* src = in + p;
                const uint32_t x = uint32_t(src[0]) | (uint32_t(src[1]) << 8) | (uint32_t(src[2]) << 16) |
                                   (uint32_t(src[3]) << 24);
                if (fin && j == Qs - 1) {
                    int badj, kk;
                    uint32_t v;
                    const uint32_t kind = final_quad(x, lut, tab.pad, tab.lenient, &badj, &kk, &v);
                    if (kind == kOk) store_bytes(o + 3 * j, v, kk);
                    else atomicMin(cell, pack_err(pbase + 4 * j + badj, kind));
                } else {
                    uint32_t err = 0;
                    const uint32_t v = dec_quad(x, lut, err);
                    store_bytes(o + 3 * j, v, 3);
                    if (err & kInvalid) atomicMin(cell, pack_err(pbase + 4 * j + first_bad_in_quad(x, lut), kBadChar));
                }
            }
        }
      }
      if (__any_sync(kFull, !started)) break;  // a string at or after hi (or the end): done
    }
}

// ---------------------------------------------------------------- finalize

// Single stream: the cell IS *err_off (initialised to kErrNone by memset).
__global__ void dec_finalize_single_kernel(int64_t* err_off, int32_t* status, int64_t* out_len,
                                           const uint8_t* __restrict__ in, int64_t m, uint32_t pad) {
    griddep_wait();
    const unsigned long long wv = *reinterpret_cast<unsigned long long*>(err_off);
    if (wv >= kErrNone) {
        *err_off = -1;
        if (status) *status = kOk;
        if (out_len) {
            int64_t ol = 3 * (m >> 2);
            if (m >= 4) ol -= (in[m - 2] == pad) ? 2 : (in[m - 1] == pad ? 1 : 0);
            *out_len = ol;
        }
    } else {
        const int64_t pos = int64_t(wv >> 3);
        *err_off = pos;
        if (status) *status = int32_t(wv & 7);
        if (out_len) *out_len = 3 * (pos >> 2);
    }
}

// Padding-optional decode (R13), m % 4 in {2, 3}: the 4*floor(m/4)
// full quads were decoded as interior quads into the cell; this one thread
// checks the trailing 2-3 char group (alphabet chars, zero dropped bits),
// decodes it to 1-2 bytes and writes the API results.
__global__ void dec_finalize_unpadded_kernel(int64_t* err_off, int32_t* status, int64_t* out_len,
                                             const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out,
                                             DecTab tab) {
    griddep_wait();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(tab.w);
    const int r = int(m & 3);
    const int64_t p = m - r;
    unsigned long long wv = *reinterpret_cast<unsigned long long*>(err_off);
    const uint32_t a = lut[in[p]], b = lut[in[p + 1]], c = (r == 3) ? lut[in[p + 2]] : 0u;
    unsigned long long pw = kErrNone;
    if (a & kInvalid) pw = pack_err(p, kBadChar);
    else if (b & kInvalid) pw = pack_err(p + 1, kBadChar);
    else if (r == 3 && (c & kInvalid)) pw = pack_err(p + 2, kBadChar);
    else if (!tab.lenient && ((r == 2 && (b & 15u)) || (r == 3 && (c & 3u)))) pw = pack_err(m - 1, kNonCanon);
    if (pw == kErrNone) {
        out[3 * (p >> 2)] = uint8_t((a << 2) | (b >> 4));
        if (r == 3) out[3 * (p >> 2) + 1] = uint8_t(((b & 15u) << 4) | (c >> 2));
    }
    wv = pw < wv ? pw : wv;
    if (wv >= kErrNone) {
        *err_off = -1;
        if (status) *status = kOk;
        if (out_len) *out_len = 3 * (p >> 2) + (r - 1);
    } else {
        const int64_t pos = int64_t(wv >> 3);
        *err_off = pos;
        if (status) *status = int32_t(wv & 7);
        if (out_len) *out_len = 3 * (pos >> 2);
    }
}

// Chunk / multi-GPU: packed word -> (err_off, status).
__global__ void dec_finalize_packed_kernel(const int64_t* cell, int64_t* err_off, int32_t* status) {
    griddep_wait();
    const unsigned long long wv = *reinterpret_cast<const unsigned long long*>(cell);
    if (wv >= kErrNone) {
        *err_off = -1;
        if (status) *status = kOk;
    } else {
        *err_off = int64_t(wv >> 3);
        if (status) *status = int32_t(wv & 7);
    }
}

// Host pipeline (b64_decode_host): packed word -> (err_off, status) and the exact output
// length: *out_len holds the final chunk's valid length (b64_decode_chunk), out_base the
// bytes of the chunks before it; on an error only 3*floor(err/4) bytes are exact.
__global__ void dec_finalize_len_kernel(const int64_t* cell, int64_t* err_off, int32_t* status, int64_t* out_len,
                                        int64_t out_base) {
    griddep_wait();
    const unsigned long long wv = *reinterpret_cast<const unsigned long long*>(cell);
    if (wv >= kErrNone) {
        *err_off = -1;
        if (status) *status = kOk;
        if (out_len) *out_len += out_base;
    } else {
        const int64_t pos = int64_t(wv >> 3);
        *err_off = pos;
        if (status) *status = int32_t(wv & 7);
        if (out_len) *out_len = 3 * (pos >> 2);
    }
}

__global__ void dec_batch_init_kernel(int64_t* err, int64_t count, const BatchCtx* gate) {
    griddep_wait();
    if (gate && !gate->generic) return;  // the concatenation path finished the batch (batch.cu)
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        err[i] = int64_t(kErrNone);
}

__global__ void dec_batch_finalize_kernel(const uint8_t* __restrict__ in, const int64_t* __restrict__ in_off,
                                          int64_t count, uint32_t pad, int32_t* status, int64_t* err,
                                          int64_t* out_len, int64_t index_base, unsigned long long* first_bad,
                                          BatchCtx* ctx) {
    griddep_wait();
    if (ctx) {  // gated (batch.cu): only after the generic kernel ran; the last CTA resets the context
        __shared__ bool s_last;
        const bool run = ctx->generic != 0;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&ctx->reserved[0], 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last && threadIdx.x < sizeof(BatchCtx) / 4) reinterpret_cast<uint32_t*>(ctx)[threadIdx.x] = 0;
        if (!run) return;
    }
    int64_t bad = INT64_MAX;  // this thread's first failing string (index_base + i)
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = in_off[i], L = in_off[i + 1] - a;
        const unsigned long long wv = static_cast<unsigned long long>(err[i]);
        int32_t st;
        int64_t e, ol;
        if (L & 3) {
            st = kLength; e = L - (L & 3); ol = 0;
        } else if (wv >= kErrNone) {
            st = kOk; e = -1; ol = 3 * (L >> 2);
            if (L >= 4) ol -= (in[a + L - 2] == pad) ? 2 : (in[a + L - 1] == pad ? 1 : 0);
        } else {
            e = int64_t(wv >> 3); st = int32_t(wv & 7); ol = 3 * (e >> 2);
        }
        err[i] = e;
        if (status) status[i] = st;
        if (out_len) out_len[i] = ol;
        if (st != kOk && bad == INT64_MAX) bad = index_base + i;  // i only grows per thread
    }
    if (first_bad) {  // the batch's first failing string: warp MIN, one atomic per warp
        const unsigned long long b = static_cast<unsigned long long>(bad);
        const unsigned hi = __reduce_min_sync(kFull, unsigned(b >> 32));
        const unsigned lo_min = __reduce_min_sync(kFull, unsigned(b >> 32) == hi ? unsigned(b) : ~0u);
        if ((threadIdx.x & 31) == 0 && hi != 0x7FFFFFFFu) atomicMin(first_bad, (static_cast<unsigned long long>(hi) << 32) | lo_min);
    }
}

}  // namespace b64
