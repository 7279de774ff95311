// mime.cu -- whitespace-skipping validating decode (reading R14;
// SURVEY.md Sec. 8(f) f2; MIME line-wrapped base64 is the paper's motivating
// use).
//
// The bytes 0x09-0x0D and 0x20 that are not alphabet chars are removed and the
// rest is decoded under the strict rules; errors are reported at their
// position in the ORIGINAL text.  Stream compaction on the GPU, four kernels:
//   1. ws_count_kernel    per 4 KiB chunk: number of kept chars; per CTA total
//                         (CTA b owns the K consecutive chunks [bK, bK + K));
//                         a warp loads its whole chunk at once (8 lane-linear
//                         LDG.128 per lane) before the table look-ups;
//   2. ws_scan_kernel     one CTA: exclusive scan of the <= 1024 CTA totals and
//                         the compacted length m';
//   3. ws_compact_kernel  each CTA scans its own K chunk counts in shared
//                         memory; a warp loads its whole chunk (8 x LDG.128
//                         per lane), compacts it through a per-warp shared
//                         buffer (16-bit keep mask per lane, one warp prefix
//                         sum per 512 B) and writes it with 4-byte stores
//                         (funnel-shifted from aligned shared words) into the
//                         workspace (byte-at-a-time paths for an unaligned
//                         input and the last chunk);
//   4. dec_fast_kernel    strict decode of the compacted text (its length m'
//                         read from device memory);
//   5. ws_finalize_kernel one warp maps the compacted error position (or the
//                         LENGTH position m' - m' % 4) back to the original
//                         text: CTA (binary search) -> chunk -> byte.
// Traffic: read m (count) + read m, write m' (compact) + read m', write 3m'/4
// (decode), i.e. ~4.75 B per char against 1.75 for the strict decode.
// Measured (1 GiB of data as MIME lines of 76 chars + CRLF): 1.67 ms in all;
// per 256 MiB (ncu): count 72 us, compact 238 us, decode ~100 us.  The
// compaction (shared byte store per char) is issue-bound; with an alphabet
// that has no whitespace chars the keep masks come from an arithmetic
// per-byte test (ws_bits) instead of table look-ups (count 88 -> 72 us,
// compact 285 -> 238 us).  The byte-at-a-time first version took 3.7 ms.
#include "b64_device.cuh"

namespace b64 {

constexpr int kWsChunk = 4096;     // bytes per chunk (one warp at a time)
constexpr int kWsMaxCtas = 1024;   // the scan kernel scans the CTA totals in one CTA
constexpr uint8_t kSkip = 0x40;    // class value of a skipped byte in the ws table

struct WsTab { uint32_t w[64]; };  // 256 entries: 6-bit value, kInvalid, or kSkip

__device__ __forceinline__ bool ws_keep(const uint8_t* lut, uint32_t c) { return lut[c] != kSkip; }

// keep-mask of the 4 bytes of x (bit b = byte b kept)
__device__ __forceinline__ uint32_t ws_keep4(const uint8_t* lut, uint32_t x) {
    uint32_t mask = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) mask |= ws_keep(lut, (x >> (8 * b)) & 0xffu) ? (1u << b) : 0u;
    return mask;
}

// Arithmetic whitespace test for alphabets without whitespace chars (host
// checked; the table path handles the others): 0x80 in every byte of x that is
// 0x09-0x0D or 0x20, exact per byte (no carries: each byte is masked to 7 bits
// first), ~7 instructions per 4 bytes instead of 4 table look-ups.
__device__ __forceinline__ uint32_t ws_bits(uint32_t x) {
    const uint32_t y = x & 0x7F7F7F7Fu;
    const uint32_t z = y ^ 0x20202020u;
    const uint32_t nz = (z + 0x7F7F7F7Fu) | z;   // bit 7: byte != 0x20
    const uint32_t ge9 = y + 0x77777777u;        // bit 7: byte >= 0x09
    const uint32_t ge14 = y + 0x72727272u;       // bit 7: byte >= 0x0E
    return (~nz | (ge9 & ~ge14)) & ~x & 0x80808080u;
}

// keep-mask of the 4 bytes of x (bit b = byte b kept), either way
template <bool SW>
__device__ __forceinline__ uint32_t keep4(const uint8_t* lut, uint32_t x) {
    if (SW) {
        const uint32_t k = ~ws_bits(x) & 0x80808080u;
        return ((k >> 7) | (k >> 14) | (k >> 21) | (k >> 28)) & 0xFu;
    }
    return ws_keep4(lut, x);
}

template <bool SW>
__global__ void __launch_bounds__(kThreads)
ws_count_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, int64_t K, int32_t* __restrict__ counts,
                int64_t* __restrict__ cta_tot) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ unsigned long long s_tot;
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    if (threadIdx.x == 0) s_tot = 0;
    griddep_wait();
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nch = (m + kWsChunk - 1) / kWsChunk;
    const int64_t c_lo = int64_t(blockIdx.x) * K, c_hi = min(c_lo + K, nch);
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    uint32_t mine = 0;
    for (int64_t c = c_lo + wib; c < c_hi; c += kThreads / 32) {
        const int64_t b0 = c * kWsChunk;
        const int64_t len = min(int64_t(kWsChunk), m - b0);
        uint32_t cnt = 0;
        if (vec && len == kWsChunk) {
            // 8 x 16 B per lane, lane-linear (whole sectors), all in flight before the look-ups
            uint4 v[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) v[it] = ld128_nc(in + b0 + it * 512 + lane * 16);
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const uint32_t wv[4] = {v[it].x, v[it].y, v[it].z, v[it].w};
                if (SW) {  // the 16 whitespace flags at distinct bits, one popcount
                    const uint32_t f = (ws_bits(wv[0]) >> 7) | (ws_bits(wv[1]) >> 6) | (ws_bits(wv[2]) >> 5) |
                                       (ws_bits(wv[3]) >> 4);
                    cnt += 16u - __popc(f);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int b = 0; b < 4; ++b) cnt += ws_keep(lut, (wv[q] >> (8 * b)) & 0xffu) ? 1u : 0u;
                }
            }
        } else {
            for (int64_t i = lane; i < len; i += 32) cnt += ws_keep(lut, in[b0 + i]) ? 1u : 0u;
        }
        cnt = __reduce_add_sync(kFull, cnt);
        if (lane == 0) {
            counts[c] = int32_t(cnt);
            mine += cnt;
        }
    }
    if (lane == 0) atomicAdd(&s_tot, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0) cta_tot[blockIdx.x] = int64_t(s_tot);
}

// One CTA: exclusive scan of n (<= 1024) CTA totals -> cta_base; *m_out = sum.
__global__ void __launch_bounds__(1024) ws_scan_kernel(const int64_t* __restrict__ cta_tot, int n,
                                                       int64_t* __restrict__ cta_base, int64_t* __restrict__ m_out) {
    __shared__ int64_t s_warp[32];
    griddep_launch_dependents();
    griddep_wait();
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t v = t < n ? cta_tot[t] : 0;
    int64_t x = v;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = s_warp[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, s, d);
            if (lane >= d) s += y;
        }
        s_warp[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = (w ? s_warp[w - 1] : 0) + x - v;
    if (t < n) cta_base[t] = before;
    if (t == 0) *m_out = s_warp[31];
}

template <bool SW>
__global__ void __launch_bounds__(kThreads)
ws_compact_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, int64_t K, const int32_t* __restrict__ counts,
                  const int64_t* __restrict__ cta_base, uint8_t* __restrict__ dst) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(16) uint8_t s_buf[kThreads / 32][kWsChunk + 16];
    __shared__ int64_t s_pref[kThreads];   // per-thread partial sums of the CTA's chunk counts
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    griddep_wait();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nch = (m + kWsChunk - 1) / kWsChunk;
    const int64_t c_lo = int64_t(blockIdx.x) * K, c_hi = min(c_lo + K, nch);
    const int64_t nloc = c_hi > c_lo ? c_hi - c_lo : 0;
    // exclusive prefix of the CTA's chunk counts: thread t sums the chunks
    // [t*per, (t+1)*per); s_pref[t] becomes the exclusive prefix of those sums
    const int64_t per = (nloc + kThreads - 1) / kThreads;
    int64_t part = 0;
    for (int64_t j = threadIdx.x * per; j < min(nloc, int64_t(threadIdx.x + 1) * per); ++j) part += counts[c_lo + j];
    s_pref[threadIdx.x] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = cta_base[blockIdx.x];
        for (int t = 0; t < kThreads; ++t) {
            const int64_t v = s_pref[t];
            s_pref[t] = run;
            run += v;
        }
    }
    __syncthreads();
    uint8_t* buf = &s_buf[wib][0];
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    for (int64_t j = wib; j < nloc; j += kThreads / 32) {
        // output offset of chunk c_lo + j: the prefix of its segment plus the
        // counts of the segment's chunks before it (fewer than `per`)
        const int64_t seg = j / per;
        int64_t mine = 0;
        for (int64_t i = seg * per + lane; i < j; i += 32) mine += counts[c_lo + i];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(kFull, mine, d);
        const int64_t off = s_pref[seg] + mine;

        const int64_t b0 = (c_lo + j) * kWsChunk;
        const int len = int(min(int64_t(kWsChunk), m - b0));
        int n_kept = 0;
        if (vec && len == kWsChunk) {
            // the whole 4 KiB chunk in flight at once (8 x lane-linear LDG.128 per lane), then per
            // 512 B: a 16-bit keep mask per lane (table look-ups), ONE warp prefix sum of the
            // per-lane counts, and the kept bytes stored at their compacted positions
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ld128_nc(in + b0 + u * 512 + lane * 16);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                uint32_t mask = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) mask |= keep4<SW>(lut, wv[q]) << (4 * q);
                const int cnt = __popc(mask);
                int incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(kFull, incl, d);
                    if (lane >= d) incl += y;
                }
                int pos = n_kept + incl - cnt;
                if (mask == 0xffffu) {  // nothing skipped in this lane's 16 bytes
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int b = 0; b < 4; ++b) buf[pos + 4 * q + b] = uint8_t(wv[q] >> (8 * b));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if (mask & (1u << (4 * q + b))) buf[pos++] = uint8_t(wv[q] >> (8 * b));
                }
                n_kept += __shfl_sync(kFull, incl, 31);
            }
        } else {
            for (int i0 = 0; i0 < len; i0 += 32) {
                const int i = i0 + lane;
                const uint32_t c = i < len ? in[b0 + i] : 0u;
                const bool keep = i < len && ws_keep(lut, c);
                const uint32_t bal = __ballot_sync(kFull, keep);
                if (keep) buf[n_kept + __popc(bal & ((1u << lane) - 1u))] = uint8_t(c);
                n_kept += __popc(bal);
            }
        }
        __syncwarp();
        // copy the compacted chunk to dst + off: byte head up to 4-alignment, words, byte tail
        uint8_t* d = dst + off;
        const int head = int((4 - (reinterpret_cast<uintptr_t>(d) & 3)) & 3);
        const int h = head < n_kept ? head : n_kept;
        if (lane < h) d[lane] = buf[lane];
        const int nw = (n_kept - h) >> 2;
        // word t of the output = buffer bytes [h + 4t, h + 4t + 4): two aligned shared words + a
        // funnel shift (h < 4 is uniform; the second word may lie past the kept bytes -- unused)
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(buf);
        const uint32_t fsh = uint32_t(h) * 8;
        for (int t = lane; t < nw; t += 32) {
            const uint32_t v = __funnelshift_r(bw[t], bw[t + 1], fsh);
            *reinterpret_cast<uint32_t*>(d + h + 4 * t) = v;
        }
        const int tail0 = h + 4 * nw;
        if (lane < n_kept - tail0) d[tail0 + lane] = buf[tail0 + lane];
        __syncwarp();
    }
}

// One warp.  Finalises a whitespace-skipping decode: the strict decode of the
// compacted text wrote its packed first error into *err_off (initialised to
// kErrNone); *m_c is the compacted length.  Maps the compacted position back
// to the original text and writes err_off / status / out_len.
__global__ void __launch_bounds__(32)
ws_finalize_kernel(int64_t* err_off, int32_t* status, int64_t* out_len, const int64_t* __restrict__ m_c,
                   const uint8_t* __restrict__ in, int64_t m, const uint8_t* __restrict__ comp, WsTab tab, uint32_t pad,
                   int64_t K, int ncta, const int32_t* __restrict__ counts, const int64_t* __restrict__ cta_base) {
    __shared__ __align__(256) uint32_t s_lut[64];
    griddep_wait();
    const int lane = threadIdx.x;
    s_lut[lane] = tab.w[lane];
    s_lut[lane + 32] = tab.w[lane + 32];
    __syncwarp();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int64_t mc = *m_c;
    const unsigned long long wv = *reinterpret_cast<unsigned long long*>(err_off);
    int64_t e = -1;
    int32_t kind = kOk;
    if (mc & 3) {
        e = mc - (mc & 3);
        kind = kLength;
    } else if (wv < kErrNone) {
        e = int64_t(wv >> 3);
        kind = int32_t(wv & 7);
    }
    if (e < 0) {
        if (lane == 0) {
            *err_off = -1;
            if (status) *status = kOk;
            if (out_len) {
                int64_t ol = 3 * (mc >> 2);
                if (mc >= 4) ol -= (comp[mc - 2] == pad) ? 2 : (comp[mc - 1] == pad ? 1 : 0);
                *out_len = ol;
            }
        }
        return;
    }
    // CTA holding compacted index e: the last b with cta_base[b] <= e
    int lo = 0, hi = ncta - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cta_base[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const int64_t nch = (m + kWsChunk - 1) / kWsChunk;
    int64_t run = cta_base[lo];
    int64_t c = int64_t(lo) * K;
    const int64_t c_end = min(c + K, nch);
    // chunk: walk the CTA's counts 32 at a time
    for (;;) {
        const int64_t ci = c + lane;
        const int64_t v = ci < c_end ? counts[ci] : 0;
        int64_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const bool past = ci < c_end && run + incl > e;
        const uint32_t bal = __ballot_sync(kFull, past);
        if (bal) {
            const int l = __ffs(bal) - 1;
            const int64_t before = __shfl_sync(kFull, incl - v, l);
            run += before;
            c += l;
            break;
        }
        run += __shfl_sync(kFull, incl, 31);
        c += 32;
    }
    // byte inside chunk c: the (e - run)-th kept byte
    const int64_t b0 = c * kWsChunk;
    const int len = int(min(int64_t(kWsChunk), m - b0));
    int64_t want = e - run;
    int64_t pos = -1;
    for (int i0 = 0; i0 < len && pos < 0; i0 += 32) {
        const int i = i0 + lane;
        const bool keep = i < len && ws_keep(lut, in[b0 + i]);
        const uint32_t bal = __ballot_sync(kFull, keep);
        const int k = __popc(bal);
        if (want < k) {
            uint32_t b = bal;
            for (int64_t t = 0; t < want; ++t) b &= b - 1;  // drop the lowest `want` set bits
            pos = b0 + i0 + (__ffs(b) - 1);
        } else {
            want -= k;
        }
    }
    if (lane == 0) {
        *err_off = pos;
        if (status) *status = kind;
        if (out_len) *out_len = kind == kLength ? 0 : 3 * (e >> 2);  // LENGTH: nothing decoded (R6)
    }
}

}  // namespace b64
