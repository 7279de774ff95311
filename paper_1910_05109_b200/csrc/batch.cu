// batch.cu -- the batched decode's concatenation path (BASELINE.json configs[3];
// b64_decode_batch_fast).
//
// When every string length is a multiple of 4 and the output offsets are the
// scan of 3*len/4 (the layout b64_decode_batch_offsets produces), the batch's
// output is laid out exactly like the decode of the concatenated text: quad q
// of the concatenation lands at out + 3q whatever string it belongs to
// (every quad decodes on its own).  So the bulk of the batch
// runs the single-stream dec_fast loop (one LDG.256 per lane, shared-memory
// re-layout, lane-linear stores) over the concatenation, and only the strings'
// final quads -- the one place padding may appear (DESIGN.md
// R6) -- get a per-string pass.  Six launches, three of them gated:
//   1. dec_batch_prep_kernel   err[i] = none; checks the layout (len % 4, the
//                              offsets, alignment) -> ctx->generic = 1 if not.
//   2. dec_batch_bulk_kernel   the concatenation, every quad as interior, with
//                              the pad char classified as 0x40 (a "deferred pad
//                              candidate", PAPER.md:305-313's deferred check):
//                              0x80 chars are reported per string, the '='
//                              seen are counted.
//   3. dec_batch_strfinal_kernel  per string: the final quad under R6 / R16
//                              (bytes rewritten), then status / err_off /
//                              out_len / first failing string in final form;
//                              and the count of '=' at len-2 / len-1.  The
//                              last CTA compares: more '=' seen than at final
//                              positions -> a pad is misplaced somewhere ->
//                              ctx->generic = 1 and the results are redone:
//   4-6. dec_batch_init / dec_generic / dec_batch_finalize, each gated on
//                              ctx->generic (they return at once otherwise):
//                              the exact per-string decode of
//                              b64_decode_batch_ex.  The finalize's last CTA
//                              resets the context for the next call.
// Every position reported in steps 2-3 is a genuinely bad position under the
// rules, so the per-string MIN is the first error.
#include "b64_device.cuh"

namespace b64 {

constexpr uint32_t kPadCand = 0x40u;  // table value of the pad char in the bulk pass
constexpr uint32_t kBadSlots = 64;    // per warp: 32-char windows with a bad char noted for after the loop

__global__ void __launch_bounds__(kThreads)
dec_batch_prep_kernel(const uint8_t* __restrict__ in, const int64_t* __restrict__ in_off, const uint8_t* out,
                      const int64_t* __restrict__ out_off, int64_t count, int64_t* __restrict__ err, BatchCtx* ctx) {
    griddep_launch_dependents();
    griddep_wait();
    in_off = after_wait(in_off);  // the offsets may come from the kernel before (batch_offsets)
    out_off = after_wait(out_off);
    const int64_t g0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, gs = int64_t(gridDim.x) * blockDim.x;
    const int64_t a0 = in_off[0], o0 = out_off[0];
    bool bad = g0 == 0 && (((reinterpret_cast<uintptr_t>(in + a0) & 31) != 0) ||
                           ((reinterpret_cast<uintptr_t>(out + o0) & 15) != 0));
    // 4 consecutive strings per thread per step, every load of a step issued before its checks
    for (int64_t i0 = 4 * g0; i0 < count; i0 += 4 * gs) {
        int64_t a[5], o[4];
#pragma unroll
        for (int j = 0; j < 5; ++j) a[j] = i0 + j <= count ? in_off[i0 + j] : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = i0 + j < count ? out_off[i0 + j] : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i0 + j < count) {
                err[i0 + j] = int64_t(kErrNone);
                const int64_t L = a[j + 1] - a[j];
                bad |= (L & 3) != 0 || L < 0 || o[j] - o0 != 3 * ((a[j] - a0) >> 2);
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) ctx->generic = 1u;
}

// First string s with in_off[s + 1] > pos (pos absolute, in the concatenated input).
__device__ __forceinline__ int64_t string_of(const int64_t* __restrict__ in_off, int64_t count, int64_t pos) {
    int64_t lo = 0, hi = count - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (in_off[mid + 1] > pos) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// Rare path: every string with a non-alphabet char among the nchar chars at p (absolute
// input position P) gets its first such char (within the window) reported, relative to
// the string's start.  The pad char is not reported here (step 3 / 4 decide it).
__device__ __forceinline__ void report_window(const uint8_t* p, int64_t P, int nchar, const uint8_t* __restrict__ lut,
                                           const int64_t* __restrict__ in_off, int64_t count,
                                           unsigned long long* __restrict__ cells) {
    int64_t send = INT64_MIN;
    for (int c = 0; c < nchar; ++c) {
        if (!(lut[p[c]] & kInvalid)) continue;
        const int64_t pos = P + c;
        if (pos < send) continue;  // a later bad char of a string already reported
        const int64_t s = string_of(in_off, count, pos);
        const int64_t a = in_off[s];
        send = in_off[s + 1];
        atomicMin(&cells[s], pack_err(pos - a, kBadChar));
    }
}

__device__ __forceinline__ uint32_t count_pads(const uint32_t (&x)[8], uint32_t pad4) {
    uint32_t k = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) k += __popc(__vcmpeq4(x[q], pad4));
    return k >> 3;
}

template <int D>
__global__ void __launch_bounds__(kThreads, kBulkCtasPerSm)
dec_batch_bulk_kernel(const uint8_t* __restrict__ in_base, const int64_t* __restrict__ in_off,
                      uint8_t* __restrict__ out_base, const int64_t* __restrict__ out_off, int64_t count, DecTab tab,
                      unsigned long long* __restrict__ cells, BatchCtx* ctx) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];
    __shared__ unsigned long long s_badw[kThreads / 32][kBadSlots];  // windows with a bad char: chunk << 5 | lane
    __shared__ uint32_t s_nbad[kThreads / 32];
    griddep_launch_dependents();
    if (threadIdx.x < kThreads / 32) s_nbad[threadIdx.x] = 0;
    griddep_wait();
    if (ctx->generic) return;  // the layout is not the concatenation's: step 4 does it all
    const int lane = threadIdx.x & 31;
    const int64_t a0 = in_off[0];
    const int64_t m = in_off[count] - a0;
    const uint8_t* in = in_base + a0;
    uint8_t* out = out_base + out_off[0];
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t nwarp = gthreads >> 5;
    const int64_t Q = m >> 2;
    const int64_t nchunk = Q >> 8;
    const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);
    const uint32_t pad4 = tab.pad * 0x01010101u;

    // the dec_fast_kernel loop (decode.cu) over the concatenation, every quad interior
    const int64_t c0 = gtid >> 5;
    const int32_t C = int32_t(nchunk), W = int32_t(nwarp), c0i = int32_t(c0);
    const int64_t sin = nwarp * 1024, sout = nwarp * 768;
    const uint8_t* pin = in + c0 * 1024 + lane * 32;
    const uint8_t* pcur = pin;
    uint8_t* pout = out + c0 * 768;
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
    uint32_t npad = 0;
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
                if (err & (kInvalid | kPadCand)) {  // rare: a bad char or a pad candidate in my 32 chars
                    if (err & kPadCand) npad += count_pads(xr[i], pad4);
                    if (err & kInvalid) {  // noted here, reported after the loop (keeps the loop's registers few)
                        const uint32_t slot = atomicAdd(&s_nbad[threadIdx.x >> 5], 1u);
                        if (slot < kBadSlots)
                            s_badw[threadIdx.x >> 5][slot] = (static_cast<unsigned long long>(c) << 5) | lane;
                    }
                }
                pout += sout;
                pcur += sin;
#pragma unroll
                for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
            }
        }
    }
    // leftover quads, one per thread
    for (int64_t q = (nchunk << 8) + gtid; q < Q; q += gthreads) {
        const uint32_t x = ld32(in + 4 * q);
        uint32_t err = 0;
        const uint32_t v = dec_quad(x, lut, err);
        store_bytes(out + 3 * q, v, 3);
        if (err & kPadCand) npad += __popc(__vcmpeq4(x, pad4)) >> 3;
        if (err & kInvalid) report_window(in + 4 * q, a0 + 4 * q, 4, lut, in_off, count, cells);
    }
    npad = __reduce_add_sync(kFull, npad);
    if (lane == 0 && npad) atomicAdd(&ctx->eq, static_cast<unsigned long long>(npad));
    // the noted windows: every string with a non-alphabet char there gets its first one
    __syncwarp();
    const uint32_t nb = s_nbad[threadIdx.x >> 5];
    if (nb > kBadSlots) {  // more than the notes hold: the per-string fallback redoes the batch exactly
        if (lane == 0) ctx->generic = 1u;
    } else {
        for (uint32_t k = lane; k < nb; k += 32) {
            const unsigned long long wv = s_badw[threadIdx.x >> 5][k];
            const int64_t p = int64_t(wv >> 5) * 1024 + int64_t(wv & 31) * 32;
            report_window(in + p, a0 + p, 32, lut, in_off, count, cells);
        }
    }
}

// Step 3: one thread per string.  The final quad under R6 / R16 (lenient: its 1-3 bytes
// rewritten -- the bulk pass decoded it with the pad as a candidate value), then the
// string's results in their final form: the first error is the MIN of what the bulk pass
// reported and the final quad's verdict, out_len follows (b64_decode_ex rules), and the
// batch's first failing string is folded in.  The last CTA compares the pad counts: a pad
// anywhere but the last two chars of its string makes all of this provisional, and the
// gated kernels after this one redo the batch per string.
__global__ void __launch_bounds__(kThreads)
dec_batch_strfinal_kernel(const uint8_t* __restrict__ in, const int64_t* __restrict__ in_off, uint8_t* __restrict__ out,
                          const int64_t* __restrict__ out_off, int64_t count, DecTab tab, int64_t* __restrict__ err,
                          int32_t* __restrict__ status, int64_t* __restrict__ out_len, int64_t index_base,
                          unsigned long long* first_bad, BatchCtx* ctx) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ unsigned long long s_sum[kThreads / 32];
    __shared__ bool s_last;
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    __syncthreads();
    griddep_wait();
    if (ctx->generic) return;  // not eligible: the gated kernels do the batch
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    uint32_t legit = 0;
    int64_t bad_idx = INT64_MAX;
    // 4 consecutive strings per thread per step: their offsets and words, then their final
    // quads, are loaded together (two dependent DRAM round trips per step, not per string)
    const int64_t gs = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i0 = 4 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x); i0 < count; i0 += 4 * gs) {
        int64_t a[5];
        unsigned long long wv[4];
        uint32_t x[4];
#pragma unroll
        for (int j = 0; j < 5; ++j) a[j] = i0 + j <= count ? in_off[i0 + j] : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) wv[j] = i0 + j < count ? static_cast<unsigned long long>(err[i0 + j]) : kErrNone;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t L = a[j + 1] - a[j];
            x[j] = (i0 + j < count && L >= 4) ? ld32(in + a[j] + L - 4) : 0u;  // 4-byte aligned: layout checked
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = i0 + j;
            if (i >= count) break;
            const int64_t L = a[j + 1] - a[j];
            unsigned long long w = wv[j];  // the bulk pass's packed word
            int64_t ol = 0;
            if (L >= 4) {
                legit += uint32_t(((x[j] >> 16) & 0xffu) == tab.pad) + uint32_t((x[j] >> 24) == tab.pad);
                int bad, k;
                uint32_t v;
                const uint32_t kind = final_quad(x[j], lut, tab.pad, tab.lenient, &bad, &k, &v);
                if (kind == kOk) {
                    // strict: the bulk pass already wrote the exact bytes -- a canonical final quad's
                    // dropped bits are zero, so the pad candidate (0x40 = 1 << 6) only sets a bit of
                    // a discarded byte; lenient: non-zero dropped bits can carry into a kept byte
                    if (tab.lenient) store_bytes(out + out_off[i] + 3 * ((L >> 2) - 1), v, k);
                    ol = 3 * ((L >> 2) - 1) + k;
                } else {
                    const unsigned long long fw = pack_err(L - 4 + bad, kind);
                    w = fw < w ? fw : w;
                }
            }
            int32_t st;
            int64_t e;
            if (w >= kErrNone) {
                st = kOk; e = -1;
            } else {
                e = int64_t(w >> 3); st = int32_t(w & 7); ol = 3 * (e >> 2);
                if (bad_idx == INT64_MAX) bad_idx = index_base + i;  // i only grows per thread
            }
            err[i] = e;
            if (status) status[i] = st;
            if (out_len) out_len[i] = ol;
        }
    }
    if (first_bad) {  // the batch's first failing string: warp MIN, one atomic per warp
        const unsigned long long b = static_cast<unsigned long long>(bad_idx);
        const unsigned hi = __reduce_min_sync(kFull, unsigned(b >> 32));
        const unsigned lo_min = __reduce_min_sync(kFull, unsigned(b >> 32) == hi ? unsigned(b) : ~0u);
        if ((threadIdx.x & 31) == 0 && hi != 0x7FFFFFFFu)
            atomicMin(first_bad, (static_cast<unsigned long long>(hi) << 32) | lo_min);
    }
    legit = __reduce_add_sync(kFull, legit);  // < 2^32 per warp
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = legit;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b = 0;
        for (int w = 0; w < kThreads / 32; ++w) b += s_sum[w];
        if (b) atomicAdd(&ctx->legit, b);
        __threadfence();
        s_last = atomicAdd(&ctx->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long eq = atomicAdd(&ctx->eq, 0ull), lg = atomicAdd(&ctx->legit, 0ull);
        if (eq != lg) ctx->generic = 1u;  // a pad char outside the final two positions of its string
    }
}

}  // namespace b64
