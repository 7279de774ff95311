// mime.cu -- whitespace-skipping validating decode (reading R14;
// SURVEY.md Sec. 8(f) f2; MIME line-wrapped base64 is the paper's motivating
// use).
//
// The bytes 0x09-0x0D and 0x20 that are not alphabet chars are removed and the
// rest is decoded under the strict rules; errors are reported at their
// position in the ORIGINAL text.  Stream compaction on the GPU, four kernels:
//   1. ws_count_kernel    per 4 KiB chunk: number of kept chars; per group
//                         total (group b = the K consecutive chunks [bK, bK +
//                         K); 1024 groups, or 4096 from 256 MiB of text on,
//                         taken from a counter by a resident grid); a warp
//                         loads its whole chunk at once (8 lane-linear LDG.128
//                         per lane) before the table look-ups;
//   2. ws_scan_kernel     one CTA: exclusive scan of the <= 4096 group totals
//                         and the compacted length m';
//   3. ws_compact_kernel  groups from a counter again; each scans its own K
//                         chunk counts (block scan); a warp compacts its chunk
//                         (rows of lane-linear LDG.32) through a per-warp shared
//                         buffer (16-bit keep mask per lane, one warp prefix
//                         sum per 512 B) and writes it with 8-byte stores
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
// Texts up to 512 KiB take ONE cluster launch instead (ws_small_kernel: the
// same steps separated by cluster barriers).
// Line-structured text (MIME / PEM: every line L >= 32 chars, L % 4 == 0,
// then the same 1-2 whitespace bytes) skips all of that: ws_line_probe_kernel
// guesses the layout, ws_line_kernel decodes straight from the text in one
// pass and verifies every byte; the general kernels above then return at once
// (they run when the layout does not hold).  Measured (1 GiB of data as MIME
// lines of 76 chars + CRLF): 0.60 ms (line kernel ~149 us per 256 MiB with the
// bulk-copy staging, issue-bound); the general path 1.50 ms on a random layout
// (per 256 MiB: count ~70 us, compact ~199 us, decode ~100 us; the compaction
// is issue-bound; alphabets without whitespace chars use an arithmetic
// per-byte test for the keep masks).  The byte-at-a-time first version took
// 3.7 ms.
#include "b64_device.cuh"

namespace b64 {

// ws_compact_kernel's byte stores: 1 = all four byte positions, highest first, __syncwarp between
// (branch-free, the default); 0 = the earlier per-count tests (A/B only).  The __syncwarps are
// required: without them ptxas reorders a lane's four stores and the overwrite order is lost.
#ifndef B64_WS_STORE_ALL
#define B64_WS_STORE_ALL 1
#endif
#define B64_WS_SYNC() __syncwarp()
constexpr int kWsChunk = 4096;     // bytes per chunk (one warp at a time)
#ifndef B64_WS_MAX_CTAS
#define B64_WS_MAX_CTAS 4096
#endif
constexpr int kWsMaxCtas = B64_WS_MAX_CTAS;  // the scan kernel scans the CTA totals in one CTA (4 per thread)
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

// PTX prmt with the selector used as given (__byte_perm masks it with 0x7777 first: one LOP3)
__device__ __forceinline__ uint32_t prmt_raw(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// keep-mask of the 4 bytes of x (bit b = byte b kept), either way
template <bool SW>
__device__ __forceinline__ uint32_t keep4(const uint8_t* lut, uint32_t x) {
    if (SW) {
        // the kept flags (bit 7 of each byte: ws_bits inverted, folded by ptxas into its LOP3s),
        // gathered by one multiply: bits 7 / 15 / 23 / 31 land on 28 / 29 / 30 / 31 and every
        // cross product on a distinct lower bit (7, 14, 15, 21, 22, 23: no carries into the top)
        const uint32_t y = x & 0x7F7F7F7Fu;
        const uint32_t z = y ^ 0x20202020u;
        const uint32_t nz = (z + 0x7F7F7F7Fu) | z;   // bit 7: byte != 0x20
        const uint32_t ge9 = y + 0x77777777u;        // bit 7: byte >= 0x09
        const uint32_t ge14 = y + 0x72727272u;       // bit 7: byte >= 0x0E
        const uint32_t k = ((nz & ~(ge9 & ~ge14)) | x) & 0x80808080u;
        return (k * 0x00204081u) >> 28;
    }
    return ws_keep4(lut, x);
}

// ---------------------------------------------------------------- line-structured text
// MIME / PEM text is lines of L chars (L % 4 == 0) each followed by the same
// 1-2 whitespace bytes, the last line possibly shorter (and any whitespace
// after it, e.g. blank lines at the end of a mail part).  Then kept char e sits
// at orig(e) = (e / L) * P + e % L (P = L + s): no compaction is needed.  A
// one-warp probe guesses (L, s, separator) from the first whitespace byte and
// the text's end; ws_line_kernel decodes straight from the text AND verifies
// every byte (chars non-whitespace, separators exact); any deviation clears
// `mode` and the general path (count / scan / compact / decode, which exit
// at once in line mode) runs instead.  Traffic: read m + write 3m'/4, one pass.
struct WsLine {
    int32_t mode;             // 1: a line segment is active (ws_line_kernel decodes it); 2: line segments
                              // decoded the whole text; 0: the general path decodes the suffix that
                              // starts at text position `off`, kept index k0
    int32_t L, s, sep;        // chars per full line, separator bytes (0-2) and their values (LE)
    int32_t v0;               // chars the segment's first line lacks (it may start mid-line): kept char e
                              // of the segment sits at off + line_orig(e + v0) -- lines counted virtually
    int64_t nfull, r, mc;     // the segment's full (virtual) lines, chars of its last line, kept chars
    unsigned long long cell;  // the segment's first interior error, packed (GLOBAL kept index << 3 | kind)
    int64_t off;              // modes 1 / 2: the segment's virtual text base (its first kept char is at
                              // off + v0); mode 0: where the general path's suffix starts
    int64_t k0;               // kept index of the segment's first char (a multiple of kLineBlk)
    long long fail;           // first block of the segment whose layout check failed (LLONG_MAX: none)
    unsigned long long errk;  // first error of the finished segments, packed (kept index << 3 | kind)
    int64_t errt;             // its text position
};
constexpr int64_t kLineProbe = 65536;  // bytes searched for the first whitespace byte
constexpr int kLineSegs = 3;           // line segments per call (b64_decode_ws): 2 layout breaks at line speed
#ifndef B64_LINE_BLK
#define B64_LINE_BLK 4096
#endif
#ifndef B64_LINE_THREADS
#define B64_LINE_THREADS 128
#endif
constexpr int kLineThreads = B64_LINE_THREADS;
constexpr int kLineBlk = B64_LINE_BLK;  // kept chars per warp step (kLineBlk / 1024 units per lane)
constexpr int kLineStage = kLineBlk + kLineBlk / 16 + 80;  // + separators (L >= 32: <= 2 per 32) + slop

__device__ __forceinline__ int64_t line_orig(int64_t e, int64_t L, int64_t P) { return (e / L) * P + e % L; }

// The layout of the text [start, m) (lane 0's w; w.mode 1 = line-structured, 0 = not).
// Trailing whitespace (a final line break, blank lines, blanks) is skipped: the layout is
// read on [ms, me), me = one past the last non-whitespace byte (searched in the last
// kLineProbe bytes), ms = the first non-whitespace byte at or after start (searched in
// kLineProbe bytes); p = the first whitespace byte after ms gives the line length.
__device__ void probe_layout(const uint8_t* __restrict__ in, int64_t start, int64_t m, const uint8_t* lut,
                             int lane, WsLine& w, bool& early_fail) {
    early_fail = false;
    int64_t me = -1;
    for (int64_t j0 = m; j0 > start && m - j0 < kLineProbe && me < 0; j0 -= 32) {
        const int64_t i = j0 - 1 - lane;
        const uint32_t bal = __ballot_sync(kFull, i >= start && lut[in[i]] != kSkip);
        if (bal) me = j0 - (__ffs(bal) - 1);
    }
    int64_t ms = -1;
    for (int64_t i0 = start; i0 < min(me, start + kLineProbe) && ms < 0; i0 += 32) {
        const int64_t i = i0 + lane;
        const uint32_t bal = __ballot_sync(kFull, i < me && lut[in[i]] != kSkip);
        if (bal) ms = i0 + __ffs(bal) - 1;
    }
    const int64_t lim = ms < 0 ? 0 : min(me, ms + kLineProbe);
    int64_t p = -1;  // the first whitespace byte after ms: the end of the (maybe partial) first line
    for (int64_t i0 = ms; i0 >= 0 && i0 < lim && p < 0; i0 += 32) {
        const int64_t i = i0 + lane;
        const uint32_t bal = __ballot_sync(kFull, i < lim && lut[in[i]] == kSkip);
        if (bal) p = i0 + __ffs(bal) - 1;
    }
    int s = 0;  // separator bytes after it
    if (p >= 0)
        while (s < 3 && p + s < me && lut[in[p + s]] == kSkip) ++s;
    const int64_t q = p + s;  // the second line's first char
    const int64_t lim2 = (p >= 0 && s <= 2) ? min(me, q + kLineProbe) : 0;
    int64_t p2 = -1;  // the end of the second line
    for (int64_t i0 = q; p >= 0 && s <= 2 && i0 < lim2 && p2 < 0; i0 += 32) {
        const int64_t i = i0 + lane;
        const uint32_t bal = __ballot_sync(kFull, i < lim2 && lut[in[i]] == kSkip);
        if (bal) p2 = i0 + __ffs(bal) - 1;
    }
    w.mode = 0; w.L = 0; w.s = 0; w.sep = 0; w.v0 = 0; w.nfull = 0; w.r = 0; w.mc = 0; w.off = start;
    if (me <= start || ms < 0) {
        // whitespace only, or a leading / trailing run longer than the probe: the general path
    } else if (p < 0) {  // no whitespace between ms and the trailing run (probe window): one line
        const int64_t n1 = me - ms;
        w.mode = 1; w.r = n1; w.mc = n1; w.off = ms;
        w.L = int32_t(min(int64_t(1) << 30, (n1 + 4) & ~int64_t(3)));  // any multiple of 4 above n1
    } else if (s >= 1 && s <= 2) {
        // lines of L chars each followed by the separator; the first may be partial (L0 chars,
        // the segment starting mid-line), the last has 1..L chars
        // L = the second line's length when it is at least the first's (the first is then
        // partial: a segment starting mid-line), else the first's (the second is the last line,
        // or holds the irregularity the line kernel will find)
        const int64_t L0 = p - ms;
        const int64_t L = (p2 >= 0 && p2 - q >= L0) ? p2 - q : L0;
        if (L >= 32 && (L & 3) == 0 && L < (int64_t(1) << 30) && L0 >= 1 && L0 <= L && (L0 & 3) == 0) {
            const int64_t v0 = L - L0, P = L + s, n1 = me - ms + v0;
            const int64_t nfull = (n1 - 1) / P, r = n1 - nfull * P;
            if (r >= 1 && r <= L) {
                w.mode = 1; w.L = int32_t(L); w.s = s; w.v0 = int32_t(v0); w.nfull = nfull; w.r = r;
                w.mc = nfull * L + r - v0; w.off = ms - v0;
                w.sep = int32_t(in[p]) | int32_t(s > 1 ? in[p + 1] : 0) << 8;
                // the separators of the first block's first 32 lines, one per lane: a layout that
                // breaks there is known broken before the line kernel runs (w.fail = 0: its grid
                // exits at once and the reprobe patches block 0) -- a failed attempt costs three
                // small launches instead of one wave of line-kernel blocks
                const int64_t j = lane;
                bool broke = false;
                if (j < nfull && (j + 1) * L - v0 <= kLineBlk) {
                    const int64_t sp = w.off + j * P + L;
                    broke = in[sp] != in[p] || (s > 1 && in[sp + 1] != in[p + 1]);
                }
                early_fail = __any_sync(kFull, broke);
            }
        }
    }
}

__global__ void __launch_bounds__(32)
ws_line_probe_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, WsLine* __restrict__ li,
                     int64_t* __restrict__ mc_general) {
    __shared__ __align__(256) uint32_t s_lut[64];
    griddep_launch_dependents();
    const int lane = threadIdx.x;
    s_lut[lane] = tab.w[lane];
    s_lut[lane + 32] = tab.w[lane + 32];
    griddep_wait();
    __syncwarp();
    WsLine w;
    bool early_fail;
    probe_layout(in, 0, m, reinterpret_cast<const uint8_t*>(s_lut), lane, w, early_fail);
    if (lane) return;
    w.cell = kErrNone; w.k0 = 0; w.fail = early_fail ? 0 : LLONG_MAX; w.errk = kErrNone; w.errt = -1;
    mc_general[0] = 0;  // the general path's decode does nothing unless its scan runs
    mc_general[1] = 0;
    mc_general[2] = 0;  // the count / compaction kernels' group counters
    mc_general[3] = 0;
    *li = w;
}

// After a line segment: if its layout held everywhere, the line path is done (mode 2).
// Otherwise the blocks before the first failing one are verified and decoded: their first
// error (if any) is kept with its text position (errk / errt).  The failing block itself --
// its first kLineBlk kept chars, wherever the irregularity sits among them -- is decoded
// here by one CTA (stage ~8 KiB of text in shared memory, compact the kept chars with a
// block-wide prefix sum, decode the 1024 interior quads), and the rest of the text after its
// last kept char becomes the next segment: probed again (mode 1, the next line kernel) or,
// without a line layout, left to the general path (mode 0: suffix [off, m) from kept index
// k0).  After the last segment (`last`) the general path takes the rest from the failing
// block on.  So a stray byte in MIME text costs one probe, one 4 KiB block and the line pass
// over the rest -- not the general path over everything.
constexpr int kPatchThreads = 256;
constexpr int kPatchWin = 8192;  // text bytes staged: the block's 4096 kept chars and at least one more
// the patch CTA decodes a whole block with 4 quads per thread (B64_LINE_BLK is not free: 2048
// measured slower on the line path anyway, 0.74 vs 0.64 ms per GiB)
static_assert(kLineBlk == 16 * kPatchThreads && kLineBlk <= kPatchWin / 2, "reprobe block geometry");

__global__ void __launch_bounds__(kPatchThreads)
ws_line_reprobe_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, WsLine* __restrict__ li,
                       uint8_t* __restrict__ out, int last) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(16) uint8_t s_win[kPatchWin];
    __shared__ __align__(16) uint8_t s_comp[kLineBlk];
    __shared__ int32_t s_wsum[kPatchThreads / 32];
    __shared__ int32_t s_plan, s_end, s_bad, s_badpos;
    __shared__ int64_t s_p0, s_k0;
    __shared__ unsigned long long s_errk;
    __shared__ int64_t s_errt;
    griddep_launch_dependents();
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t < 64) s_lut[t] = tab.w[t];
    griddep_wait();
    __syncthreads();
    if (__ldcg(&li->mode) != 1) return;
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    if (t == 0) {
        const WsLine cur = *li;
        s_plan = 0;
        if (cur.fail == LLONG_MAX) {
            li->mode = 2;  // the whole segment verified: the line path decoded everything
        } else {
            const int64_t L = cur.L, P = L + cur.s;
            const int64_t kb = int64_t(cur.fail) * kLineBlk;  // segment-relative kept index of the failing block
            unsigned long long errk = cur.errk;
            int64_t errt = cur.errt;
            if (cur.cell < kErrNone && int64_t(cur.cell >> 3) - cur.k0 < kb && cur.cell < errk) {
                errk = cur.cell;  // a verified block's error: keep it, with its text position
                errt = cur.off + line_orig(int64_t(cur.cell >> 3) - cur.k0 + cur.v0, L, P);
            }
            s_p0 = cur.off + line_orig(kb + cur.v0, L, P);
            s_k0 = cur.k0 + kb;
            s_errk = errk;
            s_errt = errt;
            s_plan = last ? 2 : 1;
        }
        s_bad = INT32_MAX;
    }
    __syncthreads();
    if (s_plan == 0) return;
    const int64_t p0 = s_p0, k0 = s_k0;
    int32_t general = s_plan == 2;
    int64_t p1 = -1;
    if (!general) {
        // ---- stage the text from p0 (16-byte aligned loads when the address allows)
        int64_t A = p0 - int64_t((reinterpret_cast<uintptr_t>(in) + p0) & 15);
        if (A < 0) A = 0;
        const int skip = int(p0 - A);
        const int nb = int(min(int64_t(kPatchWin), m - A));
        if (((reinterpret_cast<uintptr_t>(in) + A) & 15) == 0) {
            for (int c = t; c < nb / 16; c += kPatchThreads)
                *reinterpret_cast<uint4*>(s_win + 16 * c) = ld128_nc(in + A + 16 * c);
            for (int i = (nb / 16) * 16 + t; i < nb; i += kPatchThreads) s_win[i] = in[A + i];
        } else {
            for (int i = t; i < nb; i += kPatchThreads) s_win[i] = in[A + i];
        }
        __syncthreads();
        // ---- keep flags of this thread's 32 window bytes, block-wide exclusive prefix
        uint32_t mask = 0;
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const int i = 32 * t + j;
            if (i >= skip && i < nb && lut[s_win[i]] != kSkip) mask |= 1u << j;
        }
        const int cnt = __popc(mask);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_wsum[wid] = incl;
        __syncthreads();
        int wpre = 0, total = 0;
        for (int w = 0; w < kPatchThreads / 32; ++w) {
            if (w < wid) wpre += s_wsum[w];
            total += s_wsum[w];
        }
        const int pre = wpre + incl - cnt;
        // the block's kLineBlk kept chars must all be interior: at least one more kept char
        // must follow in the window (else: the general path takes the rest, it is short or
        // whitespace-heavy)
        general = total <= kLineBlk;
        if (!general) {
            int k = pre;
            for (uint32_t mm = mask; mm; mm &= mm - 1) {
                const int j = __ffs(mm) - 1;
                if (k < kLineBlk) s_comp[k] = s_win[32 * t + j];
                if (k == kLineBlk - 1) s_end = 32 * t + j;
                ++k;
            }
            __syncthreads();
            // ---- decode the 1024 interior quads: thread t -> quads 4t .. 4t+3 (12 bytes)
            const uint4 xv = *reinterpret_cast<const uint4*>(s_comp + 16 * t);
            const uint32_t x[4] = {xv.x, xv.y, xv.z, xv.w};
            uint32_t err = 0, v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = dec_quad(x[q], lut, err);
            if (err & (kInvalid | kSkip)) {
                for (int q = 0; q < 4; ++q) {
                    const int jb = first_bad_in_quad(x[q], lut);
                    if (jb < 4) { atomicMin(&s_bad, 16 * t + 4 * q + jb); break; }
                }
            }
            uint32_t o0, o1, o2;
            dec_pack12(v[0], v[1], v[2], v[3], o0, o1, o2);
            uint32_t* ow = reinterpret_cast<uint32_t*>(out + 3 * (k0 >> 2) + 12 * t);  // 4-byte aligned
            ow[0] = o0;
            ow[1] = o1;
            ow[2] = o2;
            __syncthreads();
            // ---- the first bad char's text position (the thread whose window bytes hold it)
            const int bad = s_bad;
            if (bad != INT32_MAX && bad >= pre && bad < pre + cnt) {
                uint32_t mm = mask;
                for (int r = bad - pre; r > 0; --r) mm &= mm - 1;
                s_badpos = 32 * t + __ffs(mm) - 1;
            }
            __syncthreads();
            if (t == 0) {
                if (bad != INT32_MAX && pack_err(k0 + bad, kBadChar) < s_errk) {
                    s_errk = pack_err(k0 + bad, kBadChar);
                    s_errt = A + s_badpos;
                }
                s_p0 = A + s_end + 1;  // the next segment starts after the block's last kept char
            }
            __syncthreads();
            p1 = s_p0;
        }
    }
    // ---- the next segment: probe the rest (warp 0) or hand it to the general path
    if (wid) return;
    WsLine w;
    bool early_fail = false;
    if (!general) {
        probe_layout(in, p1, m, lut, lane, w, early_fail);
        // a layout that breaks again within the first block after a break is not line-structured
        // here (lines of varying length): the general path takes the rest now, not after two
        // more segment attempts that would each fail at their first block
        if (early_fail) w.mode = 0;
        if (w.mode == 0) w.off = p1;
    }
    if (lane) return;
    if (general) {
        w.mode = 0; w.L = 0; w.s = 0; w.sep = 0; w.v0 = 0; w.nfull = 0; w.r = 0; w.mc = 0; w.off = p0;
        w.k0 = k0;
    } else {
        w.k0 = k0 + kLineBlk;
    }
    w.cell = kErrNone; w.fail = early_fail ? 0 : LLONG_MAX; w.errk = s_errk; w.errt = s_errt;
    *li = w;
}

// Decode + verify in line mode.  A warp takes kLineBlk kept chars at a time:
// it stages their text span (chars + separators) in shared memory with
// lane-linear 16-byte loads; lane j copies line piece j of the span (whole
// words, funnel-shifted: col0 and L are multiples of 4) into a compact buffer
// and checks the separator after it; then lane l decodes 32 compacted chars
// per unit exactly as the fast kernels do (two LDS.128, 32 table look-ups,
// 3 x STG.64).  Any whitespace among the chars or a wrong separator flags the
// layout as broken.  The final quad is left to ws_finalize_kernel; when
// mc % 4 != 0 (LENGTH) the full quads are decoded as interior ones.
// x / d for 0 <= x < 2^31 and 32 <= d <= 2^30 without an integer division: a float estimate
// (relative error ~1e-7, so off by at most one here) corrected either way
__device__ __forceinline__ int32_t div_small(int32_t x, int32_t d, float inv) {
    int32_t q = __float2int_rz(__int2float_rn(x) * inv);
    if (int64_t(q) * d > x) --q;
    else if (int64_t(q + 1) * d <= x) ++q;
    return q;
}

#ifndef B64_LINE_MINB
#define B64_LINE_MINB 6
#endif
#ifndef B64_LINE_TMA
#define B64_LINE_TMA 1
#endif
__global__ void __launch_bounds__(kLineThreads, B64_LINE_MINB)
ws_line_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, WsLine* __restrict__ li,
               uint8_t* __restrict__ out) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(16) uint8_t s_stage[kLineThreads / 32][kLineStage];
    __shared__ __align__(16) uint8_t s_comp[kLineThreads / 32][kLineBlk + 48];
#if B64_LINE_TMA
    __shared__ __align__(8) uint64_t s_lbar[kLineThreads / 32];
#endif
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
#if B64_LINE_TMA
    if ((threadIdx.x & 31) == 0) {
        mbar_init(smem_u32(&s_lbar[threadIdx.x >> 5]), 1);
        mbar_init_fence();
    }
#endif
    griddep_wait();
    __syncthreads();
    if (__ldcg(&li->mode) != 1) return;
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const uint32_t lb = smem_u32(s_lut);
    const int lane = threadIdx.x & 31;
    uint8_t* stg = &s_stage[threadIdx.x >> 5][0];
    const int64_t kseg = li->k0;  // the segment's first kept index (a multiple of kLineBlk)
    out += 3 * (kseg >> 2);
    const int32_t L = li->L, S = li->s;             // L >= 32: a 32-char unit crosses <= 1 line end
    const float invL = 1.0f / float(L);
    const int64_t P = int64_t(L) + S, nfull = li->nfull, mc = li->mc, li_off = li->off;
    const uint32_t sep = uint32_t(li->sep);
    const uint32_t sep_mask = S == 2 ? 0xffffu : (S == 1 ? 0xffu : 0u);
    const bool dec = (mc & 3) == 0;
    // the final quad (ws_finalize_kernel); with mc % 4 != 0 (LENGTH -- or a layout guess that a
    // later block disproves) every full quad is interior and decoded: a segment's verified
    // blocks must be complete whatever its length turns out to be
    const int64_t qfin = dec ? (mc >> 2) - 1 : (mc >> 2);
    const int64_t W = (int64_t(gridDim.x) * blockDim.x) >> 5;
    int64_t it = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    // line / column of the warp's first kept char, advanced per grid-stride step without division
    const int64_t v0 = li->v0;  // virtual line coordinates: kept char K sits at line / col of K + v0
    int64_t line0 = (it * kLineBlk + v0) / L;
    int32_t col0 = int32_t(it * kLineBlk + v0 - line0 * L);
    const int64_t step_lines = (W * kLineBlk) / L;
    const int32_t step_col = int32_t(W * kLineBlk - step_lines * L);
    bool irregular = false;
    int64_t bad = INT64_MAX;  // first invalid kept index seen by this lane
    // a step's text span: [b0, b0 + 16 nch) holds its kept chars and the separators after them
    // (b0 = its first char rounded down to 16 bytes)
    auto span = [&](int64_t itx, int64_t l0, int32_t c0, int64_t& o0x, int64_t& b0x, int& nchx) {
        const int64_t K0x = itx * kLineBlk, K1x = min(K0x + kLineBlk, mc);
        const int32_t rlx = int32_t(K1x - 1 - K0x) + c0;  // last char, relative to line l0's start
        const int32_t dllx = div_small(rlx, L, invL);
        o0x = li_off + l0 * P + c0;
        const int64_t o1x = min(m, o0x + int64_t(dllx) * P + (rlx - dllx * L - c0) + 1 + S);
        b0x = o0x - int64_t(reinterpret_cast<uintptr_t>(in + o0x) & 15);
        nchx = int((o1x - b0x + 15) >> 4);
    };
#if B64_LINE_TMA
    // the span is staged by ONE bulk async copy per step, issued as soon as the previous step's
    // compaction has read the stage -- it lands while that step decodes
    const uint32_t bar = smem_u32(&s_lbar[threadIdx.x >> 5]);
    const uint32_t stg_s = smem_u32(stg);
    uint32_t phase = 0;
    bool pending = false;
    int64_t o0n = 0, b0n = 0;
    int nchn = 0;
    auto stage_async = [&](int64_t b0x, int nchx) {
        if (lane == 0) {
            fence_proxy_async_smem();  // the stage's previous reads (generic proxy) before the copy
            mbar_expect_tx(bar, uint32_t(16 * nchx));
            bulk_g2s(stg_s, in + b0x, uint32_t(16 * nchx), bar);
        }
        pending = true;
    };
    if (it * kLineBlk < mc && it < __ldcg(&li->fail)) {
        span(it, line0, col0, o0n, b0n, nchn);
        stage_async(b0n, nchn);
    }
#endif
    for (; it * kLineBlk < mc; it += W) {
        if (it >= __ldcg(&li->fail)) break;  // a block before this one broke the layout
        const int64_t K0 = it * kLineBlk, K1 = min(K0 + kLineBlk, mc);
#if B64_LINE_TMA
        const int64_t o0 = o0n, b0 = b0n;
        mbar_wait(bar, phase);
        phase ^= 1;
        pending = false;
#else
        int64_t o0, b0;
        int nch;
        span(it, line0, col0, o0, b0, nch);
        for (int c = lane; c < nch; c += 32)
            *reinterpret_cast<uint4*>(stg + 16 * c) = ld128_nc(in + b0 + 16 * c);
#endif
        __syncwarp();
        const int32_t sb = int32_t(o0 - b0) - col0;  // stage offset of line0's first char
        const int32_t krel = int32_t(K1 - K0);         // kept chars in this step
        // 1. separators out: lane j copies line piece j of the step (whole aligned words;
        //    col0 and L are multiples of 4) into the compact buffer and checks the separator
        //    after it (full lines ending inside the step)
        uint32_t* cw = reinterpret_cast<uint32_t*>(&s_comp[threadIdx.x >> 5][0]);
        const int32_t npieces = div_small(col0 + krel - 1, L, invL) + 1;
        for (int32_t jp = lane; jp < npieces; jp += 32) {
            const int32_t c_beg = jp == 0 ? col0 : 0;                         // first col of the piece
            const int32_t d_beg = jp == 0 ? 0 : jp * L - col0;                // its compact offset
            const int32_t c_end = min(L, col0 + krel - jp * L);               // one past its last col
            const int32_t so = jp * int32_t(P) + c_beg + sb;                  // stage offset of c_beg
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(stg + (so & ~3));
            const uint32_t sh = uint32_t(so & 3) * 8;
            uint32_t lo = sw[0];
            const int nw = (c_end - c_beg + 3) >> 2;
#pragma unroll 4  // (a full line is 19 words at L = 76: 0.646 -> 0.624 ms per GiB of MIME vs no unroll)
            for (int k = 0; k < nw; ++k) {
                const uint32_t hi = sw[k + 1];
                cw[(d_beg >> 2) + k] = __funnelshift_r(lo, hi, sh);
                lo = hi;
            }
            if (c_end == L && line0 + jp < nfull) {
                const int32_t sp = so + (c_end - c_beg);
                const uint32_t got = uint32_t(stg[sp]) | (uint32_t(stg[sp + 1]) << 8);
                irregular |= ((got ^ sep) & sep_mask) != 0;
            }
        }
        __syncwarp();
        if (krel < kLineBlk) {  // the segment's last step: 32 valid chars after its kept ones, so
            reinterpret_cast<uint8_t*>(cw)[krel + lane] = 'A';  // the unit loads past them vote
            __syncwarp();                                        // nothing (no per-quad mask)
        }
#if B64_LINE_TMA
        {  // the stage is free: the next step's span starts loading now
            int64_t l1 = line0 + step_lines;
            int32_t c1 = col0 + step_col;
            if (c1 >= L) {
                c1 -= L;
                ++l1;
            }
            if ((it + W) * kLineBlk < mc) {
                span(it + W, l1, c1, o0n, b0n, nchn);
                stage_async(b0n, nchn);
            }
        }
#endif
        // 2. decode the compacted chars, 32 per lane and unit (the fast kernels' per-lane code)
#pragma unroll 1
        for (int u = 0; u < kLineBlk / 1024; ++u) {
            const int32_t ru = 32 * (lane + 32 * u);     // unit's first char, relative to K0
            if (ru >= krel) break;
            const int nq = min(8, (krel - ru) >> 2);
            const int64_t q0 = (K0 + ru) >> 2;
            const uint4 a0 = *reinterpret_cast<const uint4*>(cw + (ru >> 2));
            const uint4 a1 = *reinterpret_cast<const uint4*>(cw + (ru >> 2) + 4);
            const uint32_t x[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            uint32_t v[8], err = 0;
            // (every quad votes: past the step's kept chars the buffer holds 'A's; the final
            // quad's '=' is sorted out below)
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = dec_quad_s(x[q], lb, err);
            irregular |= (err & kSkip) != 0;
            const bool tail = nq < 8 || q0 + 7 >= qfin;  // a partial unit or the final quad's
            if (err & kInvalid) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q < nq && q0 + q != qfin && bad == INT64_MAX) {
                        const int jb = first_bad_in_quad(x[q], lut);
                        if (jb < 4) bad = 4 * (q0 + q) + jb;
                    }
                }
            }
            if (!dec && nq < 8 && K1 == mc) {
                // LENGTH: the chars of the incomplete group must not be whitespace either
                const uint8_t* cb = reinterpret_cast<const uint8_t*>(cw);
                for (int32_t k = ru + 4 * nq; k < min(ru + 32, krel); ++k) irregular |= lut[cb[k]] == kSkip;
            }
            {
                uint32_t ov[6];
                dec_pack12(v[0], v[1], v[2], v[3], ov[0], ov[1], ov[2]);
                dec_pack12(v[4], v[5], v[6], v[7], ov[3], ov[4], ov[5]);
                uint8_t* o = out + 3 * q0;
                if (!tail) {
                    st64(o, ov[0], ov[1]);
                    st64(o + 8, ov[2], ov[3]);
                    st64(o + 16, ov[4], ov[5]);
                } else {
                    const int nst = int(min(int64_t(nq), qfin - q0)) * 3;  // bytes before the final quad
#pragma unroll
                    for (int b = 0; b < 24; ++b)
                        if (b < nst) o[b] = uint8_t(ov[b >> 2] >> (8 * (b & 3)));
                }
            }
        }
        __syncwarp();
        // the layout broke in this block: record it (the blocks before it stay valid; the
        // segment is cut here and the rest probed again, ws_line_reprobe_kernel) and stop
        if (__any_sync(kFull, irregular)) {
            if (lane == 0) atomicMin(&li->fail, static_cast<long long>(it));
            break;
        }
        line0 += step_lines;
        col0 += step_col;
        if (col0 >= L) {
            col0 -= L;
            ++line0;
        }
    }
#if B64_LINE_TMA
    if (pending) mbar_wait(bar, phase);  // no bulk copy may still be landing when the CTA exits
#endif
    const unsigned hi = __reduce_min_sync(kFull, unsigned(uint64_t(bad) >> 32));
    const unsigned lo = __reduce_min_sync(kFull, unsigned(uint64_t(bad) >> 32) == hi ? unsigned(bad) : ~0u);
    if (lane == 0 && hi != 0x7FFFFFFFu)
        atomicMin(&li->cell, pack_err(kseg + int64_t((uint64_t(hi) << 32) | lo), kBadChar));
}

// The general path decodes the suffix [li->off, m) of the text (all of it unless line
// segments decoded a prefix): its kernels see the text from A = li->off rounded down to a
// 16-byte-aligned address (not below 0), the first `excl` = off - A bytes excluded.
struct WsSuffix {
    int64_t A, excl;
};
__device__ __forceinline__ WsSuffix ws_suffix(const uint8_t* in, const WsLine* li) {
    const int64_t off = __ldcg(&li->off);
    int64_t A = off - int64_t((reinterpret_cast<uintptr_t>(in) + off) & 15);
    if (A < 0) A = 0;
    return WsSuffix{A, off - A};
}

template <bool SW>
__global__ void __launch_bounds__(kThreads)
ws_count_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, int64_t K, int32_t* __restrict__ counts,
                int64_t* __restrict__ cta_tot, const WsLine* __restrict__ li, int64_t ngroups,
                unsigned long long* __restrict__ ctr) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ unsigned long long s_tot;
    __shared__ int64_t s_vb;
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    griddep_wait();
    __syncthreads();
    if (__ldcg(&li->mode) != 0) return;  // line mode: ws_line_kernel did it all
    const WsSuffix sx = ws_suffix(in, li);
    in += sx.A;
    m -= sx.A;
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nch = (m + kWsChunk - 1) / kWsChunk;
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    // groups of K chunks taken from a counter (the probe kernel zeroes it): a resident grid, so a
    // call that ends on the line path launches few CTAs, and groups are balanced dynamically
    for (;;) {
    if (threadIdx.x == 0) {
        s_vb = int64_t(atomicAdd(ctr, 1ull));
        s_tot = 0;
    }
    __syncthreads();
    const int64_t vb = s_vb;
    if (vb >= ngroups) break;
    const int64_t c_lo = vb * K, c_hi = min(c_lo + K, nch);
    uint32_t mine = 0;
    for (int64_t c = c_lo + wib; c < c_hi; c += kThreads / 32) {
        const int64_t b0 = c * kWsChunk;
        const int64_t len = min(int64_t(kWsChunk), m - b0);
        uint32_t cnt = 0;
        if (vec && len == kWsChunk && b0 >= sx.excl) {
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
            for (int64_t i = lane; i < len; i += 32) cnt += (b0 + i >= sx.excl && ws_keep(lut, in[b0 + i])) ? 1u : 0u;
        }
        cnt = __reduce_add_sync(kFull, cnt);
        if (lane == 0) {
            counts[c] = int32_t(cnt);
            mine += cnt;
        }
    }
    if (lane == 0) atomicAdd(&s_tot, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0) cta_tot[vb] = int64_t(s_tot);
    __syncthreads();  // s_vb / s_tot are reused by the next group
    }
}

// One CTA: exclusive scan of n (<= 1024) CTA totals -> cta_base; *m_out = sum.
__global__ void __launch_bounds__(1024) ws_scan_kernel(const int64_t* __restrict__ cta_tot, int n,
                                                       int64_t* __restrict__ cta_base, int64_t* __restrict__ m_out,
                                                       const WsLine* __restrict__ li) {
    constexpr int E = (kWsMaxCtas + 1023) / 1024;  // totals per thread (consecutive)
    __shared__ int64_t s_warp[32];
    griddep_launch_dependents();
    griddep_wait();
    if (__ldcg(&li->mode) != 0) return;
    const int64_t k0 = __ldcg(&li->k0);  // kept chars the line segments decoded before the suffix
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int64_t e[E], v = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        e[i] = E * t + i < n ? cta_tot[E * t + i] : 0;
        v += e[i];
    }
    int64_t x = v;  // inclusive warp scan of the per-thread sums
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
    int64_t before = (w ? s_warp[w - 1] : 0) + x - v;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        if (E * t + i < n) cta_base[E * t + i] = k0 + before;
        before += e[i];
    }
    if (t == 0) {
        m_out[0] = k0 + s_warp[31];  // the total kept count
        m_out[1] = k0;               // where the suffix starts in the compacted text (dec_fast_kernel)
    }
}

template <bool SW>
__global__ void __launch_bounds__(kThreads)
ws_compact_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, int64_t K, const int32_t* __restrict__ counts,
                  const int64_t* __restrict__ cta_base, uint8_t* __restrict__ dst, const WsLine* __restrict__ li,
                  int64_t ngroups, unsigned long long* __restrict__ ctr) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ __align__(16) uint8_t s_buf[kThreads / 32][kWsChunk + 16];
    __shared__ int64_t s_pref[kThreads];   // per-thread partial sums of the CTA's chunk counts
    __shared__ int64_t s_wtot[kThreads / 32];
    __shared__ uint32_t s_sel[16];         // PRMT selector packing the kept bytes of a 4-bit mask
    griddep_launch_dependents();
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    if (threadIdx.x < 16) {
        uint32_t sel = 0x4444u;  // unused positions read the zero operand
        int k = 0;
        for (int b = 0; b < 4; ++b)
            if (threadIdx.x & (1 << b)) sel = (sel & ~(0xFu << (4 * k))) | (uint32_t(b) << (4 * k)), ++k;
        s_sel[threadIdx.x] = sel;
    }
    griddep_wait();
    if (__ldcg(&li->mode) != 0) return;
    const WsSuffix sx = ws_suffix(in, li);
    in += sx.A;
    m -= sx.A;
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nch = (m + kWsChunk - 1) / kWsChunk;
    uint8_t* buf = &s_buf[wib][0];
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    __shared__ int64_t s_vb;
    for (;;) {  // groups of K chunks from a counter, as ws_count_kernel
    if (threadIdx.x == 0) s_vb = int64_t(atomicAdd(ctr, 1ull));
    __syncthreads();
    const int64_t vb = s_vb;
    if (vb >= ngroups) break;
    const int64_t c_lo = vb * K, c_hi = min(c_lo + K, nch);
    const int64_t nloc = c_hi > c_lo ? c_hi - c_lo : 0;
    // exclusive prefix of the group's chunk counts: thread t sums the chunks
    // [t*per, (t+1)*per); s_pref[t] becomes the exclusive prefix of those sums
    const int64_t per = (nloc + kThreads - 1) / kThreads;
    int64_t part = 0;
    for (int64_t j = threadIdx.x * per; j < min(nloc, int64_t(threadIdx.x + 1) * per); ++j) part += counts[c_lo + j];
    {  // block-wide exclusive scan of the parts (warp scans + the warps' totals)
        int64_t x = part;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_wtot[wib] = x;
        __syncthreads();
        int64_t before = cta_base[vb];
        for (int w2 = 0; w2 < wib; ++w2) before += s_wtot[w2];
        s_pref[threadIdx.x] = before + x - part;
    }
    __syncthreads();
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
        if (vec && len == kWsChunk && b0 >= sx.excl) {
            // 32 rows of 128 B, lane l holding word l of a row (lane-linear LDG.32, 8 rows in
            // flight): a lane's kept bytes go to consecutive positions ~4 bytes after the
            // previous lane's, so the byte stores of a row hit distinct banks (the 16-byte-per-
            // lane layout put lanes 8 apart on one bank: 4-way conflicts on every byte store).
            // Per row: a 4-bit keep mask, the kept bytes packed by one PRMT (selector table in
            // shared memory), their count; the counts of 4 rows ride in one word (8 bits each,
            // <= 128) so ONE warp scan serves 4 rows.
#pragma unroll  // (all 4 groups: 48 instead of 59 registers, 1.81 -> 1.78 ms per GiB on the general path)
            for (int g = 0; g < kWsChunk / 1024; ++g) {
                uint32_t w[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) w[r] = ld32_nc(in + b0 + (g * 8 + r) * 128 + lane * 4);
                uint32_t km[8], pc[2] = {0u, 0u};
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    km[r] = keep4<SW>(lut, w[r]);
                    pc[r >> 2] |= uint32_t(__popc(km[r])) << (8 * (r & 3));
                }
                uint32_t ex[2], tot[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t x = pc[h];
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFull, x, d);
                        if (lane >= d) x += y;
                    }
                    tot[h] = __shfl_sync(kFull, x, 31);
                    ex[h] = x - pc[h];
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    // (byte r & 3 of the packed prefix by one PRMT; the selector table's nibbles
                    // are 0-4, so the raw prmt needs no masking of its selector)
                    const int pos = n_kept + int(__byte_perm(ex[r >> 2], 0u, 0x4440u | (r & 3)));
                    const uint32_t cw = prmt_raw(w[r], 0u, s_sel[km[r]]);
#if B64_WS_STORE_ALL
                    // All 4 bytes stored, the highest byte position first, one warp-wide store
                    // per position with a __syncwarp between: a lane's bytes past its kept count
                    // land on the next lanes' slots (pos + cnt on) and are overwritten by their
                    // stores of lower byte positions, which come later; past the row's last kept
                    // byte they are overwritten by the next row's stores or lie past the chunk's
                    // kept bytes (slack).  A lane with nothing kept (its pos is the next lane's)
                    // writes to a scratch word past the slack.  Branch-free, against a chain of
                    // count tests that ptxas compiles to branches.
                    const int sp = km[r] ? pos : kWsChunk + 8;
                    buf[sp + 3] = uint8_t(cw >> 24);
                    B64_WS_SYNC();
                    buf[sp + 2] = uint8_t(cw >> 16);
                    B64_WS_SYNC();
                    buf[sp + 1] = uint8_t(cw >> 8);
                    B64_WS_SYNC();
                    buf[sp] = uint8_t(cw);
#else
                    const int cnt = __popc(km[r]);
                    if (cnt > 0) buf[pos] = uint8_t(cw);
                    if (cnt > 1) buf[pos + 1] = uint8_t(cw >> 8);
                    if (cnt > 2) buf[pos + 2] = uint8_t(cw >> 16);
                    if (cnt > 3) buf[pos + 3] = uint8_t(cw >> 24);
#endif
                    n_kept += int(__byte_perm(tot[r >> 2], 0u, 0x4440u | (r & 3)));
                }
            }
        } else {
            for (int i0 = 0; i0 < len; i0 += 32) {
                const int i = i0 + lane;
                const uint32_t c = i < len ? in[b0 + i] : 0u;
                const bool keep = i < len && b0 + i >= sx.excl && ws_keep(lut, c);
                const uint32_t bal = __ballot_sync(kFull, keep);
                if (keep) buf[n_kept + __popc(bal & ((1u << lane) - 1u))] = uint8_t(c);
                n_kept += __popc(bal);
            }
        }
        __syncwarp();
        // copy the compacted chunk to dst + off: byte head up to 8-alignment, 8-byte units, byte
        // tail.  Unit t of the output = buffer bytes [h + 8t, h + 8t + 8): three aligned shared
        // words a = h / 4 + 2t .. a + 2 (one LDS.64 on the even-aligned pair, one LDS.32) and two
        // funnel shifts by h % 4 (h < 8 is uniform; the last word may lie past the kept bytes --
        // unused).  Pointers stepped by the warp's stride: immediate-offset addressing.
        uint8_t* d = dst + off;
        const int head = int((8 - (reinterpret_cast<uintptr_t>(d) & 7)) & 7);
        const int h = head < n_kept ? head : n_kept;
        if (lane < h) d[lane] = buf[lane];
        const int nu = (n_kept - h) >> 3;
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(buf) + (h >> 2) + 2 * lane;
        uint2* dw = reinterpret_cast<uint2*>(d + h) + lane;
        const uint32_t fsh = uint32_t(h & 3) * 8;
        if ((h >> 2) == 0) {
            for (int t = lane; t < nu; t += 32, bw += 64, dw += 32) {
                const uint2 p = *reinterpret_cast<const uint2*>(bw);
                const uint32_t c = bw[2];
                *dw = make_uint2(__funnelshift_r(p.x, p.y, fsh), __funnelshift_r(p.y, c, fsh));
            }
        } else {
            for (int t = lane; t < nu; t += 32, bw += 64, dw += 32) {
                const uint32_t a0 = bw[0];
                const uint2 p = *reinterpret_cast<const uint2*>(bw + 1);
                *dw = make_uint2(__funnelshift_r(a0, p.x, fsh), __funnelshift_r(p.x, p.y, fsh));
            }
        }
        const int tail0 = h + 8 * nu;
        if (lane < n_kept - tail0) d[tail0 + lane] = buf[tail0 + lane];
        __syncwarp();
    }
    __syncthreads();  // s_vb / s_pref are reused by the next group
    }
}

// ---------------------------------------------------------------- small texts: one launch
// For texts up to the single-launch size the whole whitespace-skipping decode
// is ONE cluster launch (the general path's steps, cluster-synchronised instead
// of separate kernels): every warp counts the kept chars of its slice; CTA and
// cluster prefix sums through shared memory and DSMEM; every warp writes its
// kept chars to the workspace at their compacted positions; cluster barrier;
// the interior quads are decoded by all threads, the final quad by the last
// one; CTA 0 maps the first error back to the original text.
constexpr int kWsSmallThreads = 512;
constexpr int kWsSmallWarps = kWsSmallThreads / 32;
constexpr int64_t kWsSmallMax = int64_t(16) * kWsSmallWarps * 4 * 512;  // 16 CTAs x warps x 4 steps of 512 B

__global__ void __launch_bounds__(kWsSmallThreads)
ws_small_kernel(const uint8_t* __restrict__ in, int64_t m, WsTab tab, uint32_t pad, uint32_t lenient,
                uint8_t* __restrict__ comp, uint8_t* __restrict__ out, int64_t* __restrict__ err_off,
                int32_t* __restrict__ status, int64_t* __restrict__ out_len) {
    __shared__ __align__(256) uint32_t s_lut[64];
    __shared__ int32_t s_wcnt[kWsSmallWarps], s_wpre[kWsSmallWarps];
    __shared__ int64_t s_tot, s_base, s_mc;
    __shared__ int32_t s_kfin;
    __shared__ unsigned long long s_min;
    cg::cluster_group cluster = cg::this_cluster();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < 64) s_lut[threadIdx.x] = tab.w[threadIdx.x];
    if (threadIdx.x == 0) {
        s_min = kErrNone;
        s_kfin = 3;
    }
    griddep_wait();
    __syncthreads();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    const int R = int(gridDim.x);  // the grid is one cluster
    const int64_t C = (((m + R - 1) / R) + 8191) & ~int64_t(8191);  // bytes per CTA (512 per warp-step)
    const int64_t Cw = C / kWsSmallWarps;
    const int64_t wb = min(m, int64_t(blockIdx.x) * C + w * Cw), we = min(m, wb + Cw);
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    // keep mask of lane's 16 bytes at i (bytes past `we` dropped)
    auto keep16 = [&](int64_t i, uint4& v) -> uint32_t {
        uint32_t mask = 0;
        if (vec && i + 16 <= we) {
            v = ld128_nc(in + i);
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) mask |= ws_keep4(lut, wv[q]) << (4 * q);
        } else {
            uint32_t wv[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; ++b) {
                if (i + b < we) {
                    const uint32_t c = in[i + b];
                    wv[b >> 2] |= c << (8 * (b & 3));
                    if (lut[c] != kSkip) mask |= 1u << b;
                }
            }
            v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        return mask;
    };
    // 1. kept chars per warp slice, CTA prefix, cluster prefix (DSMEM)
    int32_t cnt = 0;
    for (int64_t i0 = wb; i0 < we; i0 += 512) {
        uint4 v;
        const int64_t i = i0 + 16 * lane;
        cnt += i < we ? __popc(keep16(i, v)) : 0;
    }
    cnt = __reduce_add_sync(kFull, cnt);
    if (lane == 0) s_wcnt[w] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t run = 0;
        for (int k = 0; k < kWsSmallWarps; ++k) {
            s_wpre[k] = run;
            run += s_wcnt[k];
        }
        s_tot = run;
    }
    cluster.sync();
    if (threadIdx.x == 0) {
        int64_t base = 0, mc = 0;
        for (int q = 0; q < R; ++q) {
            const int64_t t = *cluster.map_shared_rank(&s_tot, q);
            if (q < int(blockIdx.x)) base += t;
            mc += t;
        }
        s_base = base;
        s_mc = mc;
    }
    __syncthreads();
    // 2. kept chars to their compacted positions (workspace)
    int64_t dst = s_base + s_wpre[w];
    for (int64_t i0 = wb; i0 < we; i0 += 512) {
        uint4 v = make_uint4(0, 0, 0, 0);
        const int64_t i = i0 + 16 * lane;
        const uint32_t mask = i < we ? keep16(i, v) : 0u;
        const int k = __popc(mask);
        int incl = k;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        int64_t pos = dst + incl - k;
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (mask & (1u << b)) comp[pos++] = uint8_t(wv[b >> 2] >> (8 * (b & 3)));
        dst += __shfl_sync(kFull, incl, 31);
    }
    cluster.sync();  // every CTA's compacted chars are visible cluster-wide
    // 3. strict decode of the compacted text (interior quads by all threads, the final one last)
    const int64_t mc = s_mc;
    if ((mc & 3) == 0 && mc > 0) {
        const int64_t Q = mc >> 2;
        const int64_t gthreads = int64_t(R) * kWsSmallThreads;
        const int64_t gtid = int64_t(blockIdx.x) * kWsSmallThreads + threadIdx.x;
        for (int64_t q = gtid; q < Q - 1; q += gthreads) {
            const uint32_t x = ld32(comp + 4 * q);
            uint32_t e = 0;
            const uint32_t v = dec_quad(x, lut, e);
            store_bytes(out + 3 * q, v, 3);
            if (e & kInvalid) atomicMin(&s_min, pack_err(4 * q + first_bad_in_quad(x, lut), kBadChar));
        }
        if (gtid == gthreads - 1) {
            int bad, k;
            uint32_t v;
            const uint32_t kind = final_quad(ld32(comp + 4 * (Q - 1)), lut, pad, lenient, &bad, &k, &v);
            if (kind == kOk) {
                store_bytes(out + 3 * (Q - 1), v, k);
                s_kfin = k;
            } else {
                atomicMin(&s_min, pack_err(4 * (Q - 1) + bad, kind));
            }
        }
    }
    cluster.sync();
    // 4. CTA 0, warp 0: results; the first error's kept index back to the text
    if (blockIdx.x == 0 && w == 0) {
        unsigned long long mn = kErrNone;
        for (int q = 0; q < R; ++q) {
            const unsigned long long v = *cluster.map_shared_rank(&s_min, q);
            mn = v < mn ? v : mn;
        }
        int64_t e = -1, ol = 0;
        int32_t kind = kOk;
        if (mc & 3) {
            e = mc - (mc & 3);
            kind = kLength;
        } else if (mn < kErrNone) {
            e = int64_t(mn >> 3);
            kind = int32_t(mn & 7);
        } else if (mc > 0) {
            ol = 3 * (mc >> 2) - 3 + *cluster.map_shared_rank(&s_kfin, R - 1);
        }
        int64_t pos = -1;
        if (e >= 0) {
            // the CTA, then the warp slice holding kept index e, then the byte
            int q = 0;
            int64_t base = 0;
            for (; q < R - 1; ++q) {
                const int64_t t = *cluster.map_shared_rank(&s_tot, q);
                if (base + t > e) break;
                base += t;
            }
            const int32_t* wpre = cluster.map_shared_rank(s_wpre, q);
            int ww = kWsSmallWarps - 1;
            while (ww > 0 && base + wpre[ww] > e) --ww;
            int64_t want = e - base - wpre[ww];
            const int64_t b0 = min(m, int64_t(q) * C + ww * Cw), b1 = min(m, b0 + Cw);
            for (int64_t i0 = b0; i0 < b1 && pos < 0; i0 += 32) {
                const int64_t i = i0 + lane;
                const uint32_t bal = __ballot_sync(kFull, i < b1 && lut[in[i]] != kSkip);
                const int k = __popc(bal);
                if (want < k) {
                    uint32_t b = bal;
                    for (int64_t t = 0; t < want; ++t) b &= b - 1;
                    pos = i0 + (__ffs(b) - 1);
                } else {
                    want -= k;
                }
            }
        }
        if (lane == 0) {
            *err_off = pos;
            if (status) *status = kind;
            if (out_len) *out_len = e < 0 ? ol : (kind == kLength ? 0 : 3 * (e >> 2));
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
}

// One warp.  Finalises a whitespace-skipping decode: the strict decode of the
// compacted text wrote its packed first error into *err_off (initialised to
// kErrNone); *m_c is the compacted length.  Maps the compacted position back
// to the original text and writes err_off / status / out_len.
__global__ void __launch_bounds__(32)
ws_finalize_kernel(int64_t* err_off, int32_t* status, int64_t* out_len, const int64_t* __restrict__ m_c,
                   const uint8_t* __restrict__ in, int64_t m, const uint8_t* __restrict__ comp, WsTab tab, uint32_t pad,
                   int64_t K, int ncta, const int32_t* __restrict__ counts, const int64_t* __restrict__ cta_base,
                   const WsLine* __restrict__ li, uint8_t* __restrict__ out, uint32_t lenient) {
    __shared__ __align__(256) uint32_t s_lut[64];
    griddep_wait();
    const int lane = threadIdx.x;
    s_lut[lane] = tab.w[lane];
    s_lut[lane + 32] = tab.w[lane + 32];
    __syncwarp();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(s_lut);
    // the first error of the segments decoded by the line path before (kept index + text position)
    const unsigned long long errk = __ldcg(&li->errk);
    const int64_t errt = __ldcg(&li->errt);
    if (__ldcg(&li->mode) == 2) {  // line segments did it all: kept index -> text position in closed form
        if (lane) return;
        const int64_t L = li->L, P = L + li->s, mcl = li->mc, k0 = li->k0, mtot = k0 + mcl, v0 = li->v0;
        unsigned long long w = __ldcg(&li->cell);  // the last segment's first interior error
        int64_t e = -1, et = -1, ol = 0;
        int32_t kind = kOk;
        if (mtot & 3) {  // LENGTH (R14 / R6): the first char of the incomplete group
            e = mtot - (mtot & 3);
            et = li->off + line_orig(e - k0 + v0, L, P);
            kind = kLength;
        } else {
            uint32_t x = 0;
            for (int b = 0; b < 4; ++b) x |= uint32_t(in[li->off + line_orig(mcl - 4 + b + v0, L, P)]) << (8 * b);
            int fb = 0, k = 0;
            uint32_t v = 0;
            const uint32_t fk = final_quad(x, lut, pad, lenient, &fb, &k, &v);
            if (fk != kOk) w = min(w, pack_err(mtot - 4 + fb, fk));
            if (errk < w) {  // an earlier segment's error comes first
                e = int64_t(errk >> 3);
                et = errt;
                kind = int32_t(errk & 7);
            } else if (w < kErrNone) {
                e = int64_t(w >> 3);
                et = li->off + line_orig(e - k0 + v0, L, P);
                kind = int32_t(w & 7);
            } else {
                ol = 3 * (mtot >> 2) - 3 + k;
                store_bytes(out + 3 * ((mtot >> 2) - 1), v, k);
            }
        }
        *err_off = e < 0 ? -1 : et;
        if (status) *status = kind;
        if (out_len) *out_len = e < 0 ? ol : (kind == kLength ? 0 : 3 * (e >> 2));
        return;
    }
    // the general path decoded the suffix [li->off, m) (kept indices from li->k0 on)
    const WsSuffix sx = ws_suffix(in, li);
    const int64_t mc = *m_c;
    const unsigned long long wv = *reinterpret_cast<unsigned long long*>(err_off);
    int64_t e = -1;
    int32_t kind = kOk;
    if (mc & 3) {
        e = mc - (mc & 3);
        kind = kLength;
    } else if (errk < kErrNone && errk < wv) {  // a line segment's error comes first
        if (lane == 0) {
            *err_off = errt;
            if (status) *status = int32_t(errk & 7);
            if (out_len) *out_len = 3 * (int64_t(errk >> 3) >> 2);
        }
        return;
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
    in += sx.A;
    m -= sx.A;
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
    // chunk: walk the CTA's counts 32 at a time (bounded: e lies in CTA lo's chunks)
    for (; c < c_end;) {
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
        const bool keep = i < len && b0 + i >= sx.excl && ws_keep(lut, in[b0 + i]);
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
        *err_off = sx.A + pos;
        if (status) *status = kind;
        if (out_len) *out_len = kind == kLength ? 0 : 3 * (e >> 2);  // LENGTH: nothing decoded (R6)
    }
}

}  // namespace b64
