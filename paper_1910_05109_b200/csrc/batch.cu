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
// R6) -- get a per-string pass.  Two cooperative launches (every CTA resident,
// phases separated by grid barriers instead of kernel boundaries):
//   dec_batch_main_kernel
//     A. per string: err[i] = none; the layout check (len % 4, the offsets,
//        alignment) -> ctx->generic = 1 if it fails;
//     B. the concatenation, every quad as interior, with the pad char
//        classified as 0x40 (a "deferred pad candidate", PAPER.md:305-313's
//        deferred check): 0x80 chars are reported per string, the '=' seen
//        are counted;
//     C. per string: the final quad under R6 / R16, then status / err_off /
//        out_len / first failing string in final form, and the count of '='
//        at len-2 / len-1.  The last CTA compares: more '=' seen than at final
//        positions -> a pad is misplaced somewhere -> ctx->generic = 1 and C's
//        results are provisional:
//   dec_batch_fallback_kernel   returns at once unless ctx->generic; else the
//        per-string path of b64_decode_batch_ex (init, dec_generic_body,
//        finalize), grid barriers between.  Its last CTA resets the context.
// Every position reported in B and C is a genuinely bad position under the
// rules, so the per-string MIN is the first error.
#include "b64_device.cuh"

#include <cooperative_groups.h>

namespace b64 {

constexpr uint32_t kPadCand = 0x40u;  // table value of the pad char in the bulk pass

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

// Last-CTA ticket on `t`: true in exactly one thread (thread 0 of the last CTA to arrive).
__device__ __forceinline__ bool last_cta(uint32_t* t) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(t, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    return s_last && threadIdx.x == 0;
}

template <int D>
__global__ void __launch_bounds__(kThreads, kBulkCtasPerSm)
dec_batch_main_kernel(const uint8_t* __restrict__ in_base, const int64_t* __restrict__ in_off,
                      uint8_t* __restrict__ out_base, const int64_t* __restrict__ out_off, int64_t count,
                      DecTab btab /* pad -> kPadCand */, DecTab tab, int64_t* __restrict__ err,
                      int32_t* __restrict__ status, int64_t* __restrict__ out_len, int64_t index_base,
                      unsigned long long* first_bad, BatchCtx* ctx) {
    __shared__ __align__(256) uint32_t s_lut[64];   // bulk table (pad = candidate)
    __shared__ __align__(256) uint32_t s_lut2[64];  // strict table (final quads)
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];
    __shared__ unsigned long long s_sum[kThreads / 32];
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    griddep_launch_dependents();
    if (threadIdx.x < 64) {
        s_lut[threadIdx.x] = btab.w[threadIdx.x];
        s_lut2[threadIdx.x] = tab.w[threadIdx.x];
    }
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    unsigned long long* cells = reinterpret_cast<unsigned long long*>(err);
    const int64_t a0 = in_off[0], o0 = out_off[0];

    // ---- A: error cells, layout check
    {
        bool bad = gtid == 0 && (((reinterpret_cast<uintptr_t>(in_base + a0) & 31) != 0) ||
                                 ((reinterpret_cast<uintptr_t>(out_base + o0) & 15) != 0));
        for (int64_t i = gtid; i < count; i += gthreads) {
            err[i] = int64_t(kErrNone);
            const int64_t a = in_off[i], L = in_off[i + 1] - a;
            bad |= (L & 3) != 0 || L < 0 || out_off[i] - o0 != 3 * ((a - a0) >> 2);
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0) ctx->generic = 1u;
    }
    grid.sync();
    if (ctx->generic) return;  // not the concatenation's layout: the fallback kernel does the batch

    // ---- B: the dec_fast_kernel loop (decode.cu) over the concatenation, every quad interior
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    {
        const int64_t m = in_off[count] - a0;
        const uint8_t* in = in_base + a0;
        uint8_t* out = out_base + o0;
        const int64_t nwarp = gthreads >> 5;
        const int64_t Q = m >> 2;
        const int64_t nchunk = Q >> 8;
        const uint32_t sb = smem_u32(&s_stage[threadIdx.x >> 5][0]);
        const uint32_t pad4 = btab.pad * 0x01010101u;
        const int64_t c0 = gtid >> 5;
        const int32_t C = int32_t(nchunk), W = int32_t(nwarp), c0i = int32_t(c0);
        const int64_t sin = nwarp * 1024, sout = nwarp * 768;
        const uint8_t* pin = in + c0 * 1024 + lane * 32;
        const uint8_t* pcur = pin;
        uint8_t* pout = out + c0 * 768;
        const uint32_t lb = smem_u32(s_lut);
        uint32_t xr[D][8];
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (c0i + i * W < C) {
                ld256_stream(pin, xr[i]);
                pin += sin;
            }
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
                    uint32_t e = 0, v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(xr[i][q], lb, e);
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
                    if (e & (kInvalid | kPadCand)) {  // rare: a bad char or a pad candidate in my 32 chars
                        if (e & kPadCand) npad += count_pads(xr[i], pad4);
                        if (e & kInvalid)
                            report_window(pcur, a0 + int64_t(c) * 1024 + lane * 32, 32, lut, in_off, count, cells);
                    }
                    pout += sout;
                    pcur += sin;
#pragma unroll
                    for (int j = 0; j < 8; ++j) xr[i][j] = y[j];
                }
            }
        }
        for (int64_t q = (nchunk << 8) + gtid; q < Q; q += gthreads) {  // leftover quads
            const uint32_t x = ld32(in + 4 * q);
            uint32_t e = 0;
            const uint32_t v = dec_quad(x, lut, e);
            store_bytes(out + 3 * q, v, 3);
            if (e & kPadCand) npad += __popc(__vcmpeq4(x, pad4)) >> 3;
            if (e & kInvalid) report_window(in + 4 * q, a0 + 4 * q, 4, lut, in_off, count, cells);
        }
        npad = __reduce_add_sync(kFull, npad);
        if (lane == 0 && npad) atomicAdd(&ctx->eq, static_cast<unsigned long long>(npad));
    }
    grid.sync();

    // ---- C: final quads and the strings' results
    {
        const uint8_t* lut2 = reinterpret_cast<const uint8_t*>(s_lut2);
        uint32_t legit = 0;
        int64_t bad_idx = INT64_MAX;
        for (int64_t i = gtid; i < count; i += gthreads) {
            const int64_t a = in_off[i], L = in_off[i + 1] - a;
            unsigned long long w = cells[i];  // B's packed word
            int64_t ol = 0;
            if (L >= 4) {
                const uint32_t x = ld32(in_base + a + L - 4);  // 4-byte aligned: the layout check passed
                legit += uint32_t(((x >> 16) & 0xffu) == tab.pad) + uint32_t((x >> 24) == tab.pad);
                int bd, k;
                uint32_t v;
                const uint32_t kind = final_quad(x, lut2, tab.pad, tab.lenient, &bd, &k, &v);
                if (kind == kOk) {
                    // strict: B already wrote the exact bytes -- a canonical final quad's dropped bits
                    // are zero, so the pad candidate (0x40 = 1 << 6) only sets a bit of a discarded
                    // byte; lenient: non-zero dropped bits can carry into a kept byte
                    if (tab.lenient) store_bytes(out_base + out_off[i] + 3 * ((L >> 2) - 1), v, k);
                    ol = 3 * ((L >> 2) - 1) + k;
                } else {
                    const unsigned long long fw = pack_err(L - 4 + bd, kind);
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
        if (first_bad) {  // the batch's first failing string: warp MIN, one atomic per warp
            const unsigned long long b = static_cast<unsigned long long>(bad_idx);
            const unsigned hi = __reduce_min_sync(kFull, unsigned(b >> 32));
            const unsigned lo_min = __reduce_min_sync(kFull, unsigned(b >> 32) == hi ? unsigned(b) : ~0u);
            if (lane == 0 && hi != 0x7FFFFFFFu) atomicMin(first_bad, (static_cast<unsigned long long>(hi) << 32) | lo_min);
        }
        legit = __reduce_add_sync(kFull, legit);  // < 2^32 per warp
        if (lane == 0) s_sum[threadIdx.x >> 5] = legit;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long b = 0;
            for (int w = 0; w < kThreads / 32; ++w) b += s_sum[w];
            if (b) atomicAdd(&ctx->legit, b);
        }
        if (last_cta(&ctx->ticket)) {
            __threadfence();
            const unsigned long long eq = atomicAdd(&ctx->eq, 0ull), lg = atomicAdd(&ctx->legit, 0ull);
            if (eq != lg) ctx->generic = 1u;  // a pad char outside the final two positions of its string
        }
    }
}

// The per-string path (b64_decode_batch_ex) when the main kernel flagged the batch; a no-op
// otherwise.  Either way its last CTA leaves the context zeroed for the next call.
__global__ void __launch_bounds__(kThreads, B64_GEN_MINB)
dec_batch_fallback_kernel(const uint8_t* __restrict__ in, const int64_t* __restrict__ in_off,
                          uint8_t* __restrict__ out, const int64_t* __restrict__ out_off, int64_t count, DecTab tab,
                          int64_t* __restrict__ err, int32_t* __restrict__ status, int64_t* __restrict__ out_len,
                          int64_t index_base, unsigned long long* first_bad, BatchCtx* ctx) {
    __shared__ __align__(256) uint32_t s_lut[64];
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    griddep_wait();
    const bool run = ctx->generic != 0;
    if (run) {
        const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
        const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
        for (int64_t i = gtid; i < count; i += gthreads) err[i] = int64_t(kErrNone);
        grid.sync();  // (also orders the table stores before the generic body's look-ups)
        Offsets off{in_off, out_off, count, 0};
        dec_generic_body(in, out, off, tab, reinterpret_cast<const uint8_t*>(s_lut), smem_u32(s_lut), 0, 1,
                         reinterpret_cast<unsigned long long*>(err), nullptr, gtid >> 5, gthreads >> 5);
        grid.sync();
        dec_batch_finalize_body(in, in_off, count, tab.pad, status, err, out_len, index_base, first_bad, gtid,
                                gthreads);
    }
    if (last_cta(&ctx->reserved[0])) {
        for (int k = 0; k < int(sizeof(BatchCtx) / 4); ++k) reinterpret_cast<uint32_t*>(ctx)[k] = 0;
    }
}

}  // namespace b64
