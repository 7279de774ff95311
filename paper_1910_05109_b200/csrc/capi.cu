// capi.cu -- the C ABI of include/b64gpu.h: argument checks, alphabet
// validation, launch configuration and kernel dispatch for the single-stream,
// decode-variant, grouped and batched entry points (capi_ext.cu: streaming,
// peer combine, host pipelines).  No allocation, no per-call state; every
// launch goes to the caller's stream.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/b64gpu.h"
#include "b64_device.cuh"

using namespace b64;

namespace {

std::atomic<int64_t> g_launches{0};

// PAPER.md:239 (standard) and PAPER.md:93 (url: '+' '/' -> '-' '_').
const char kStdChars[65] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
const char kUrlChars[65] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789-_";

struct DevInfo {
    int sms = 0;
    int occ_group[4] = {0, 0, 0, 0};  // min over the enc / dec / codec group kernels
    int occ_enc_fast[4] = {0, 0, 0, 0}, occ_dec_fast[4] = {0, 0, 0, 0}, occ_enc_gen = 0, occ_dec_gen = 0;
    int occ_batch_bulk = 0, occ_fastu[3][8] = {}, occ_enc_fastu = 0, occ_ws_count = 0, occ_ws_compact = 0;
};
constexpr int kMaxDev = 64;
DevInfo g_dev[kMaxDev];
bool g_dev_ready[kMaxDev];
std::mutex g_dev_mu;

// Resident CTAs per SM of the grouped kernels at depth 1 / 2: the minimum over
// the decode, encode and mixed kernels (one grid size serves all three).
cudaError_t group_occupancy(int (&occ)[4]) {
    for (int d = 1; d <= 2; ++d) {
        int a = 0, b = 0, c = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &a, d == 1 ? enc_group_kernel<1> : enc_group_kernel<2>, kThreads, 0);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, d == 1 ? dec_group_kernel<1> : dec_group_kernel<2>,
                                                              kThreads, 0);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &c, d == 1 ? codec_group_kernel<1> : codec_group_kernel<2>, kThreads, 0);
        if (e != cudaSuccess) return e;
        occ[d] = std::min(a, std::min(b, c));
    }
    return cudaSuccess;
}

const DevInfo* dev_info() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) return nullptr;
    std::lock_guard<std::mutex> lock(g_dev_mu);
    if (g_dev_ready[d]) return &g_dev[d];
    DevInfo info;
    if (cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) return nullptr;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_enc_fast[1], enc_fast_kernel<1>, kThreads, 0) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_enc_fast[2], enc_fast_kernel<2>, kThreads, 0) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_dec_fast[1], dec_fast_kernel<1>, kThreads, 0) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_dec_fast[2], dec_fast_kernel<2>, kThreads, 0) ||
        group_occupancy(info.occ_group) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_enc_gen, enc_generic_kernel, kThreads, 0) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_dec_gen, dec_generic_kernel, kThreads, 0) ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_batch_bulk, dec_batch_bulk_kernel<2>, kThreads, 0))
        return nullptr;
    for (int i = 0; i < 4; ++i) {
        info.occ_enc_fast[i] = info.occ_enc_fast[i] < 1 ? 1 : info.occ_enc_fast[i];
        info.occ_dec_fast[i] = info.occ_dec_fast[i] < 1 ? 1 : info.occ_dec_fast[i];
        info.occ_group[i] = info.occ_group[i] < 1 ? 1 : info.occ_group[i];
    }
    info.occ_enc_gen = info.occ_enc_gen < 1 ? 1 : info.occ_enc_gen;
    info.occ_dec_gen = info.occ_dec_gen < 1 ? 1 : info.occ_dec_gen;
    info.occ_batch_bulk = info.occ_batch_bulk < 1 ? 1 : info.occ_batch_bulk;
    for (int d = 1; d <= 2; ++d)
        for (int w = 0; w < 8; ++w) {
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, d == 2 ? dec_fastu_pick<2>(w) : dec_fastu_pick<1>(w),
                                                              kThreads, 0) != cudaSuccess)
                return nullptr;
            info.occ_fastu[d][w] = o < 1 ? 1 : o;
        }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.occ_enc_fastu, enc_fastu_kernel<1, false>, kThreads, 0) !=
        cudaSuccess)
        return nullptr;
    info.occ_enc_fastu = info.occ_enc_fastu < 1 ? 1 : info.occ_enc_fastu;
    {
        int a = 0, b = 0, c = 0, d2 = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, ws_count_kernel<true>, kThreads, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ws_count_kernel<false>, kThreads, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, ws_compact_kernel<true>, kThreads, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d2, ws_compact_kernel<false>, kThreads, 0) != cudaSuccess)
            return nullptr;
        info.occ_ws_count = std::max(1, std::min(a, b));
        info.occ_ws_compact = std::max(1, std::min(c, d2));
    }
    if (cudaFuncSetAttribute(dec_small_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(ws_small_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return nullptr;
    g_dev[d] = info;
    g_dev_ready[d] = true;
    return &g_dev[d];
}

EncTab enc_tab(const b64_alphabet* a) {
    EncTab t;
    std::memcpy(t.w, a->enc, 64);
    return t;
}
DecTab dec_tab(const b64_alphabet* a) {
    DecTab t;
    std::memcpy(t.w, a->dec, 256);
    t.pad = a->pad;
    t.lenient = (a->flags & B64_ALPHA_LENIENT) ? 1u : 0u;
    return t;
}

// The first launch / runtime error since the last launched() of this thread: every launch
// records the return value of cudaLaunchKernelEx here, and launched() reports it (no
// cudaPeekAtLastError, which would pick up errors of unrelated earlier runtime calls).
thread_local cudaError_t t_launch_err = cudaSuccess;
inline void note(cudaError_t e) {
    if (e != cudaSuccess && t_launch_err == cudaSuccess) t_launch_err = e;
}

int launched() {
    const cudaError_t e = t_launch_err;
    t_launch_err = cudaSuccess;
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear the non-sticky error the failed call left behind
        return B64_ECUDA;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return B64_OK;
}

// Launch with programmatic dependent launch allowed (the kernels call
// griddepcontrol.wait before touching global memory), so back-to-back calls on
// one stream overlap launch latency and prologue with the previous kernel's
// tail.  B64_NO_PDL=1 in the environment falls back to plain launches.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("B64_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch(void (*kernel)(KArgs...), int64_t grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(block));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    note(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Prefetch depth of the register-direct bulk loops (chunks in flight per warp
// beyond the one being translated): B64_ENC_DEPTH / B64_DEC_DEPTH in 1..2.
// Default: 2 for inputs of at least 256 MiB (tools/sweep.py on B200: 95-98 %
// of the measured copy roofline at 1-4 GiB), 1 below (shorter kernels lose
// more to the deeper prologue than they gain).
int depth_env(const char* name) {
    const char* e = std::getenv(name);
    if (e && e[0] >= '1' && e[0] <= '2') return e[0] - '0';
    return 0;
}
int enc_depth(int64_t n) {
    static const int d = depth_env("B64_ENC_DEPTH");
    return d ? d : (n >= (int64_t(256) << 20) ? 2 : 1);
}
int dec_depth(int64_t m) {
    static const int d = depth_env("B64_DEC_DEPTH");
    return d ? d : (m >= (int64_t(256) << 20) ? 2 : 1);
}

// Largest input (chars) for the single-launch cluster decode (small.cu);
// B64_SMALL_MAX overrides (0 disables the path).
int64_t small_max() {
    static const int64_t v = [] {
        const char* e = std::getenv("B64_SMALL_MAX");
        return e ? int64_t(std::atoll(e)) : kSmallMax;
    }();
    return v;
}

// Resident CTAs per SM used by the single-stream kernels: at most 5 (40 warps;
// measured best for 64 MiB ops on B200, bench per_call), B64_MAX_BPS overrides.
int cap_bps(int occ) {
    static const int cap = [] {
        const char* e = std::getenv("B64_MAX_BPS");
        return e ? std::atoi(e) : 5;
    }();
    return (cap > 0 && cap < occ) ? cap : occ;
}

template <typename K>
K pick2(int d, K k1, K k2) { return d == 2 ? k2 : k1; }

// Misaligned decodes from this many chars on take dec_fastu_kernel (unaligned.cu), smaller
// ones the generic kernel; B64_UNALIGNED_MIN overrides (a huge value disables the kernel).
int64_t unaligned_min() {
    static const int64_t v = [] {
        const char* e = std::getenv("B64_UNALIGNED_MIN");
        return e ? int64_t(std::atoll(e)) : int64_t(64) << 10;
    }();
    return v;
}

// Blocks for a grid-stride loop over `units` warp-sized work units with at most
// `max_blocks` resident blocks: the number of rounds is fixed by the resident
// capacity, then the grid is shrunk so every round is (nearly) full -- no
// partial last round in which most warps idle.
int64_t balanced_blocks(int64_t units, int64_t max_blocks) {
    const int64_t wpb = kThreads / 32;
    const int64_t wmax = max_blocks * wpb;
    if (units <= 0) return 1;
    const int64_t rounds = (units + wmax - 1) / wmax;
    const int64_t w = (units + rounds - 1) / rounds;
    const int64_t b = (w + wpb - 1) / wpb;
    return b < 1 ? 1 : (b > max_blocks ? max_blocks : b);
}

// Warp partition of a grouped launch: stream i with C[i] warp-chunks gets
// W_i = ceil(C[i] / t) warps, t = the smallest per-warp chunk count with
// sum W_i <= wmax (the resident warps).  Fills wstart[0..count] (exclusive scan
// of W_i) and returns the blocks the warps need.
int64_t group_partition(const int64_t* C, int count, int64_t wmax, int32_t* wstart) {
    int64_t cmax = 0;
    for (int i = 0; i < count; ++i) cmax = std::max(cmax, C[i]);
    auto need = [&](int64_t t) {
        int64_t s = 0;
        for (int i = 0; i < count; ++i) s += (C[i] + t - 1) / t;
        return s;
    };
    int64_t lo = 1, hi = cmax < 1 ? 1 : cmax;  // need(cmax) <= count <= wmax
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (need(mid) <= wmax) hi = mid; else lo = mid + 1;
    }
    wstart[0] = 0;
    for (int i = 0; i < count; ++i) wstart[i + 1] = wstart[i] + int32_t((C[i] + lo - 1) / lo);
    const int64_t wpb = kThreads / 32;
    const int64_t b = (int64_t(wstart[count]) + wpb - 1) / wpb;
    return b < 1 ? 1 : b;
}

int64_t clamp_grid(int64_t want, int64_t cap) { return want < 1 ? 1 : (want > cap ? cap : want); }

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

int alpha_ok(const b64_alphabet* a) { return a != nullptr; }

}  // namespace

namespace {
template <int LAW>
int batch_offsets(const int64_t* d_in_off, int64_t count, int64_t* d_out_off, b64_stream_t stream) {
    if (count < 0 || !d_out_off || (count > 0 && !d_in_off)) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (count == 0) {
        note(cudaMemsetAsync(d_out_off, 0, sizeof(int64_t), s));
        const int r = launched();
        if (r == B64_OK) g_launches.fetch_sub(1, std::memory_order_relaxed);  // a memset, not a kernel
        return r;
    }
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    const int64_t ntile = (count + kScanTile - 1) / kScanTile;
    const int64_t grid = clamp_grid(ntile, int64_t(di->sms) * 8);
    launch(off_tile_sum_kernel<LAW>, grid, kThreads, s, d_in_off, count, d_out_off);
    int r = launched();
    if (r != B64_OK) return r;
    launch(off_tile_scan_kernel, 1, 1024, s, d_out_off, count);
    if ((r = launched()) != B64_OK) return r;
    launch(off_fill_kernel<LAW>, grid, kThreads, s, d_in_off, count, d_out_off);
    return launched();
}
}  // namespace

extern "C" {

int b64_alphabet_init(b64_alphabet* a, const char chars[64], char pad, int* bad_index) {
    if (bad_index) *bad_index = -1;
    if (!a || !chars) return B64_EINVAL;
    const uint8_t* c = reinterpret_cast<const uint8_t*>(chars);
    const uint8_t p = static_cast<uint8_t>(pad);
    for (int i = 0; i < 64; ++i)
        if (c[i] >= 0x80) { if (bad_index) *bad_index = i; return B64_EALPHA_NONASCII; }
    if (p >= 0x80) { if (bad_index) *bad_index = 64; return B64_EALPHA_NONASCII; }
    bool seen[128] = {false};
    for (int i = 0; i < 64; ++i) {
        if (seen[c[i]]) { if (bad_index) *bad_index = i; return B64_EALPHA_DUP; }
        seen[c[i]] = true;
    }
    for (int i = 0; i < 64; ++i)
        if (c[i] == p) { if (bad_index) *bad_index = i; return B64_EALPHA_PAD; }
    std::memcpy(a->enc, c, 64);
    std::memset(a->dec, 0x80, 256);
    for (int v = 0; v < 64; ++v) a->dec[c[v]] = static_cast<uint8_t>(v);
    a->pad = p;
    a->flags = 0;
    a->reserved[0] = a->reserved[1] = 0;
    return B64_OK;
}

int b64_alphabet_set_flags(b64_alphabet* a, unsigned flags) {
    if (!a || (flags & ~unsigned(B64_ALPHA_LENIENT))) return B64_EINVAL;
    a->flags = static_cast<uint8_t>(flags);
    return B64_OK;
}

const b64_alphabet* b64_alphabet_standard(void) {
    static b64_alphabet a;
    static int once = (b64_alphabet_init(&a, kStdChars, '=', nullptr), 0);
    (void)once;
    return &a;
}

const b64_alphabet* b64_alphabet_url(void) {
    static b64_alphabet a;
    static int once = (b64_alphabet_init(&a, kUrlChars, '=', nullptr), 0);
    (void)once;
    return &a;
}

int64_t b64_encoded_len(int64_t n) { return n < 0 ? -1 : 4 * ((n + 2) / 3); }
int64_t b64_decoded_len_max(int64_t m) { return m < 0 ? -1 : 3 * (m / 4); }
int64_t b64_decoded_len_max_unpadded(int64_t m) {
    if (m < 0 || m % 4 == 1) return -1;
    return 3 * (m / 4) + (m % 4 ? m % 4 - 1 : 0);  // a 2 / 3-char tail -> 1 / 2 bytes (R13)
}

// ---------------------------------------------------------------- batch output offsets (offsets.cu)

int b64_encode_batch_offsets(const int64_t* d_in_off, int64_t count, int64_t* d_out_off, b64_stream_t stream) {
    return batch_offsets<0>(d_in_off, count, d_out_off, stream);
}
int b64_decode_batch_offsets(const int64_t* d_in_off, int64_t count, int64_t* d_out_off, b64_stream_t stream) {
    return batch_offsets<1>(d_in_off, count, d_out_off, stream);
}

// The single-stream encode launch (fast, misaligned-fast or generic kernel by alignment).
// `early` (an overlapped streaming piece, caller-checked: n >= unaligned_min(), d_out 4-byte
// aligned): enc_fastu_kernel<1, true> whatever the alignment, with `join` riding along.
static int encode_launch(const uint8_t* d_in, int64_t n, uint8_t* d_out, const b64_alphabet* a, cudaStream_t s,
                         bool early = false, const EncJoin* join = nullptr) {
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    if (early || (!aligned(d_in, 8) || !aligned(d_out, 32)) && aligned(d_out, 4) && n >= unaligned_min()) {
        // any input alignment, 4-byte aligned output: enc_fast's loop with a uniform byte
        // shift, from the first triple whose output is 32-byte aligned (unaligned.cu)
        const int64_t T = n / 3;
        const uintptr_t ou = reinterpret_cast<uintptr_t>(d_out);
        const int64_t q0 = std::min<int64_t>(int64_t(((32 - (ou & 31)) & 31) >> 2), T);
        const int64_t nchunk = (T - q0) / 256;
        // (one chunk in flight per warp at every size: two measured 3 % slower at 1 GiB)
        const int64_t blocks = balanced_blocks(nchunk, int64_t(di->sms) * cap_bps(di->occ_enc_fastu));
        const EncJoin ej = join ? *join : EncJoin{};
        launch(early ? enc_fastu_kernel<1, true> : enc_fastu_kernel<1, false>, blocks, kThreads, s, d_in, n, d_out,
               enc_tab(a), a->pad, q0, int32_t(nchunk), ej);
    } else if (aligned(d_in, 8) && aligned(d_out, 32)) {
        const int64_t nchunk = n / 768;
        const int dd = enc_depth(n);
        const int64_t blocks = balanced_blocks(nchunk, int64_t(di->sms) * cap_bps(di->occ_enc_fast[dd]));
        launch(pick2(dd, enc_fast_kernel<1>, enc_fast_kernel<2>), blocks, kThreads, s, d_in, n,
               d_out, enc_tab(a), a->pad);
    } else {
        Offsets off{nullptr, nullptr, 1, n};
        const int64_t blocks = clamp_grid((n / 12 + kThreads - 1) / kThreads, int64_t(di->sms) * di->occ_enc_gen);
        launch(enc_generic_kernel, blocks, kThreads, s, d_in, d_out, off, enc_tab(a), a->pad);
    }
    return launched();
}

int b64_encode(const uint8_t* d_in, int64_t n, uint8_t* d_out, const b64_alphabet* a, b64_stream_t stream) {
    if (n < 0 || !alpha_ok(a)) return B64_EINVAL;
    if (n == 0) return B64_OK;
    if (!d_in || !d_out) return B64_EINVAL;
    return encode_launch(d_in, n, d_out, a, reinterpret_cast<cudaStream_t>(stream));
}

static int decode_launch(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, int64_t base,
                         int is_final, int64_t* cell, int64_t* out_len, cudaStream_t s,
                         const StreamJoin* join = nullptr, bool* joined = nullptr, bool early = false) {
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    unsigned long long* c = reinterpret_cast<unsigned long long*>(cell);
    if (joined) *joined = false;
    if (aligned(d_in, 32) && aligned(d_out, 16)) {
        const int64_t nchunk = (m / 4) / 256;
        const int dd = dec_depth(m);
        const int64_t blocks = balanced_blocks(nchunk, int64_t(di->sms) * cap_bps(di->occ_dec_fast[dd]));
        auto k = early ? pick2(dd, dec_fast_kernel<1, true>, dec_fast_kernel<2, true>)
                       : pick2(dd, dec_fast_kernel<1>, dec_fast_kernel<2>);
        StreamJoin sj = {};
        if (join && joined) {  // the stream join rides along (its last thread)
            sj = *join;
            *joined = true;
        }
        launch(k, blocks, kThreads, s, d_in, m, d_out, dec_tab(a), base, is_final, c, out_len,
               static_cast<const int64_t*>(nullptr), sj);
    } else if (m >= unaligned_min()) {
        // any alignment, the fast loop over aligned 32-byte blocks (unaligned.cu)
        const int64_t Q = m / 4, Qint = is_final ? Q - 1 : Q;
        const uintptr_t ou = reinterpret_cast<uintptr_t>(d_out);
        UnalignedBulk ub;
        ub.q0 = std::min<int64_t>(int64_t(((8 - (ou & 7)) * 3) & 7), Qint);  // out + 3 q0 is 8-byte aligned
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(d_in) + 4 * uintptr_t(ub.q0);
        ub.b = uint32_t(s0 & 3);
        ub.A0 = reinterpret_cast<const uint8_t*>(s0 & ~uintptr_t(31));
        ub.out0 = d_out + 3 * ub.q0;
        ub.nchunk = int32_t((Qint - ub.q0) / 256);
        const int ws = int((s0 & 31) >> 2);
        const int dd = dec_depth(m);
        const int64_t blocks = balanced_blocks(ub.nchunk, int64_t(di->sms) * cap_bps(di->occ_fastu[dd][ws]));
        StreamJoin sj = {};
        if (join && joined) {
            sj = *join;
            *joined = true;
        }
        const DecFastuFn kf = early ? (dd == 2 ? dec_fastu_pick<2, true>(ws) : dec_fastu_pick<1, true>(ws))
                                    : (dd == 2 ? dec_fastu_pick<2>(ws) : dec_fastu_pick<1>(ws));
        launch(kf, blocks, kThreads, s, d_in, m, d_out,
               dec_tab(a), base, is_final, c, out_len, ub, sj);
    } else {
        Offsets off{nullptr, nullptr, 1, m};
        const int64_t blocks = clamp_grid((m / 16 + kThreads - 1) / kThreads, int64_t(di->sms) * di->occ_dec_gen);
        launch(dec_generic_kernel, blocks, kThreads, s, d_in, d_out, off, dec_tab(a), base, is_final, c, out_len,
               static_cast<const BatchCtx*>(nullptr));
    }
    return launched();
}

int b64_decode_ex(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, int64_t* d_err_off,
                  int32_t* d_status, int64_t* d_out_len, b64_stream_t stream) {
    if (m < 0 || !alpha_ok(a) || !d_err_off) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    if (m > 0 && (!d_in || !d_out)) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m <= small_max() && (m == 0 || (aligned(d_in, 32) && aligned(d_out, 16)))) {
        // small input: one cluster launch does init, decode and finalize (small.cu)
        if (!dev_info()) return B64_ECUDA;
        const int64_t nchunk = (m / 4) / 256;
        int64_t r = (nchunk + kSmallThreads / 32 - 1) / (kSmallThreads / 32);
        r = r < 1 ? 1 : (r > kSmallCluster ? kSmallCluster : r);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(r));
        cfg.blockDim = dim3(kSmallThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(r);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        if (r == 1) {  // one CTA: a plain launch (implicit 1-CTA cluster), ~0.6-1 us cheaper than a cluster launch
            attr[0] = attr[1];
            cfg.attrs = attr;
            cfg.numAttrs = pdl_enabled() ? 1 : 0;
        } else {
            cfg.attrs = attr;
            cfg.numAttrs = pdl_enabled() ? 2 : 1;
        }
        note(cudaLaunchKernelEx(&cfg, dec_small_kernel, d_in, m, d_out, dec_tab(a), d_err_off, d_status, d_out_len));
        return launched();
    }
    if (cudaMemsetAsync(d_err_off, 0x7F, sizeof(int64_t), s) != cudaSuccess) return B64_ECUDA;
    {
        const int r = decode_launch(d_in, m, d_out, a, 0, 1, d_err_off, nullptr, s);
        if (r != B64_OK) return r;
    }
    launch(dec_finalize_single_kernel, 1, 1, s, d_err_off, d_status, d_out_len, d_in, m, a->pad);
    return launched();
}

int b64_decode_unpadded(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a,
                        int64_t* d_err_off, int32_t* d_status, int64_t* d_out_len, b64_stream_t stream) {
    if (m < 0 || !alpha_ok(a) || !d_err_off) return B64_EINVAL;
    if (m % 4 == 1) return B64_ELENGTH;
    if (m % 4 == 0) return b64_decode_ex(d_in, m, d_out, a, d_err_off, d_status, d_out_len, stream);
    if (!d_in || !d_out) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(d_err_off, 0x7F, sizeof(int64_t), s) != cudaSuccess) return B64_ECUDA;
    const int64_t full = m - m % 4;
    if (full > 0) {  // every full quad is interior (no '=' allowed before the trailing group)
        const int r = decode_launch(d_in, full, d_out, a, 0, 0, d_err_off, nullptr, s);
        if (r != B64_OK) return r;
    }
    launch(dec_finalize_unpadded_kernel, 1, 1, s, d_err_off, d_status, d_out_len, d_in, m, d_out, dec_tab(a));
    return launched();
}

// ---------------------------------------------------------------- whitespace-skipping decode (mime.cu)
namespace {
struct WsLayout {
    int64_t nch, ncta, K;
    int64_t off_counts, off_tot, off_base, off_mc, total;
};
int64_t up256(int64_t v) { return (v + 255) / 256 * 256; }
WsLayout ws_layout(int64_t m) {
    WsLayout L;
    L.nch = (m + kWsChunk - 1) / kWsChunk;
    // groups of the general path (count / compaction, K chunks each, taken by resident CTAs from
    // a counter): 4096 once that still leaves >= 16 chunks per group, else 1024 -- measured on
    // random layouts (tools/ws_probe.py random) with one CTA per group: 1 GiB of data 1.74 ms with
    // 1024, 1.66 with 2048, 1.62 with 4096, 1.63 / 1.68 with 8192 / 16384; 256 MiB 0.511 / 0.502
    // / 0.502 with 1024 / 2048 / 4096 (0.54 with 1384); 64 MiB 0.216 with 1024, 0.241 with 4096
    const int64_t want = L.nch >= int64_t(16) * kWsMaxCtas ? kWsMaxCtas : 1024;
    L.ncta = L.nch < want ? (L.nch > 0 ? L.nch : 1) : want;
    L.K = (L.nch + L.ncta - 1) / L.ncta;
    if (L.K < 1) L.K = 1;
    L.ncta = (L.nch + L.K - 1) / L.K;
    if (L.ncta < 1) L.ncta = 1;
    L.off_counts = up256(m + 64);
    L.off_tot = L.off_counts + up256(4 * (L.nch + 1));
    L.off_base = L.off_tot + up256(8 * kWsMaxCtas);
    L.off_mc = L.off_base + up256(8 * kWsMaxCtas);
    L.total = L.off_mc + 256 + 256;  // + slack to align the caller's pointer
    return L;
}
}  // namespace

int64_t b64_decode_ws_workspace_bytes(int64_t m) { return m < 0 ? -1 : ws_layout(m).total; }

int b64_decode_ws(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, uint8_t* d_ws,
                  int64_t ws_bytes, int64_t* d_err_off, int32_t* d_status, int64_t* d_out_len, b64_stream_t stream) {
    if (m < 0 || !alpha_ok(a) || !d_err_off) return B64_EINVAL;
    if (m > 0 && (!d_in || !d_out || !d_ws)) return B64_EINVAL;
    if (m > 0 && !aligned(d_out, 16)) return B64_EINVAL;
    const WsLayout L = ws_layout(m);
    if (m > 0 && ws_bytes < L.total) return B64_EINVAL;
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m > 0 && m <= std::min(small_max(), kWsSmallMax)) {
        // small text: the whole decode is ONE cluster launch (mime.cu ws_small_kernel)
        uint8_t* comp = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(d_ws) + 255) & ~uintptr_t(255));
        WsTab wt;
        uint8_t* wb = reinterpret_cast<uint8_t*>(wt.w);
        std::memcpy(wb, a->dec, 256);
        for (int c : {0x09, 0x0A, 0x0B, 0x0C, 0x0D, 0x20})
            if (wb[c] == 0x80) wb[c] = kSkip;
        int64_t r = (m + 8191) / 8192;  // one 512-byte step per warp and CTA at 8 KiB
        r = r < 1 ? 1 : (r > kSmallCluster ? kSmallCluster : r);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(r));
        cfg.blockDim = dim3(kWsSmallThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(r);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        note(cudaLaunchKernelEx(&cfg, ws_small_kernel, d_in, m, wt, uint32_t(a->pad),
                                uint32_t((a->flags & B64_ALPHA_LENIENT) ? 1 : 0), comp, d_out, d_err_off, d_status,
                                d_out_len));
        return launched();
    }
    if (cudaMemsetAsync(d_err_off, 0x7F, sizeof(int64_t), s) != cudaSuccess) return B64_ECUDA;
    if (m == 0) {
        launch(dec_finalize_packed_kernel, 1, 1, s, static_cast<const int64_t*>(d_err_off), d_err_off, d_status);
        if (d_out_len && cudaMemsetAsync(d_out_len, 0, sizeof(int64_t), s) != cudaSuccess) return B64_ECUDA;
        return launched();
    }
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(d_ws) + 255) & ~uintptr_t(255));
    uint8_t* comp = base;
    int32_t* counts = reinterpret_cast<int32_t*>(base + L.off_counts);
    int64_t* tot = reinterpret_cast<int64_t*>(base + L.off_tot);
    int64_t* cbase = reinterpret_cast<int64_t*>(base + L.off_base);
    int64_t* mc = reinterpret_cast<int64_t*>(base + L.off_mc);
    WsTab wt;
    uint8_t* wb = reinterpret_cast<uint8_t*>(wt.w);
    std::memcpy(wb, a->dec, 256);
    for (int c : {0x09, 0x0A, 0x0B, 0x0C, 0x0D, 0x20})
        if (wb[c] == 0x80) wb[c] = kSkip;
    bool sw = true;  // no whitespace char is data: the arithmetic whitespace test applies
    for (int c : {0x09, 0x0A, 0x0B, 0x0C, 0x0D, 0x20}) sw = sw && a->dec[c] >= 64;
    // line-structured text (MIME / PEM) is decoded in one pass by ws_line_kernel; the general
    // path's kernels then return at once (they run when the probe or the line kernel clears
    // the mode)
    WsLine* li = reinterpret_cast<WsLine*>(base + L.off_mc + 64);
    const WsLine* lic = li;
    launch(ws_line_probe_kernel, 1, 32, s, d_in, m, wt, li, mc);
    // up to kLineSegs line segments (B64_WS_SEGS overrides, >= 1): a text whose layout breaks
    // somewhere (a stray byte) is cut there and the rest probed again; after the last one the
    // general path takes the rest
    static const int nseg = [] {
        const char* e = std::getenv("B64_WS_SEGS");
        const int v = e ? std::atoi(e) : kLineSegs;
        return v < 1 ? 1 : v;
    }();
    for (int seg = 0; seg < nseg; ++seg) {
        launch(ws_line_kernel, int64_t(di->sms) * B64_LINE_MINB, kLineThreads, s, d_in, m, wt, li, d_out);
        launch(ws_line_reprobe_kernel, 1, kPatchThreads, s, d_in, m, wt, li, d_out, seg == nseg - 1 ? 1 : 0);
    }
    // the count / compaction kernels: resident grids taking the L.ncta groups from counters
    unsigned long long* gctr = reinterpret_cast<unsigned long long*>(mc + 2);
    launch(sw ? ws_count_kernel<true> : ws_count_kernel<false>,
           std::min<int64_t>(L.ncta, int64_t(di->sms) * di->occ_ws_count), kThreads, s, d_in, m, wt, L.K, counts, tot,
           lic, L.ncta, gctr);
    launch(ws_scan_kernel, 1, 1024, s, static_cast<const int64_t*>(tot), int(L.ncta), cbase, mc, lic);
    launch(sw ? ws_compact_kernel<true> : ws_compact_kernel<false>,
           std::min<int64_t>(L.ncta, int64_t(di->sms) * di->occ_ws_compact), kThreads, s, d_in, m, wt, L.K,
           static_cast<const int32_t*>(counts), static_cast<const int64_t*>(cbase), comp, lic, L.ncta, gctr + 1);
    {  // strict decode of the compacted text; its length m' is read on the device
        const int64_t blocks = balanced_blocks(m / 1024, int64_t(di->sms) * cap_bps(di->occ_dec_fast[1]));
        launch(dec_fast_kernel<1>, blocks, kThreads, s, static_cast<const uint8_t*>(comp), m, d_out, dec_tab(a),
               int64_t(0), 1, reinterpret_cast<unsigned long long*>(d_err_off), static_cast<int64_t*>(nullptr),
               static_cast<const int64_t*>(mc), StreamJoin{});
    }
    launch(ws_finalize_kernel, 1, 32, s, d_err_off, d_status, d_out_len, static_cast<const int64_t*>(mc), d_in, m,
           static_cast<const uint8_t*>(comp), wt, uint32_t(a->pad), L.K, int(L.ncta),
           static_cast<const int32_t*>(counts), static_cast<const int64_t*>(cbase), lic, d_out,
           uint32_t((a->flags & B64_ALPHA_LENIENT) ? 1 : 0));
    g_launches.fetch_add(5 + 2 * nseg, std::memory_order_relaxed);
    return launched();
}

int b64_decode(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, int64_t* d_err_off,
               b64_stream_t stream) {
    return b64_decode_ex(d_in, m, d_out, a, d_err_off, nullptr, nullptr, stream);
}

int b64_decode_chunk(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, int64_t base_offset,
                     int is_final_chunk, int64_t* d_err_min, int64_t* d_out_len, b64_stream_t stream) {
    if (m < 0 || base_offset < 0 || !alpha_ok(a) || !d_err_min) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    if (m > 0 && (!d_in || !d_out)) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m == 0) {
        if (d_out_len && cudaMemsetAsync(d_out_len, 0, sizeof(int64_t), s) != cudaSuccess) return B64_ECUDA;
        return B64_OK;
    }
    return decode_launch(d_in, m, d_out, a, base_offset, is_final_chunk ? 1 : 0, d_err_min, d_out_len, s);
}

int b64_encode_shard(int64_t n, int world, int rank, b64_shard* sh) {
    if (n < 0 || world < 1 || rank < 0 || rank >= world || !sh) return B64_EINVAL;
    const int64_t units = n / 768, u0 = units * rank / world, u1 = units * (rank + 1) / world;
    const bool last = rank == world - 1;
    sh->start = 768 * u0;
    sh->stop = last ? n : 768 * u1;
    sh->out_start = 4 * (sh->start / 3);
    sh->out_len = last ? b64_encoded_len(sh->stop - sh->start) : 4 * ((sh->stop - sh->start) / 3);
    sh->is_final = last ? 1 : 0;
    sh->reserved = 0;
    return B64_OK;
}

int b64_decode_shard(int64_t m, int world, int rank, b64_shard* sh) {
    if (m < 0 || world < 1 || rank < 0 || rank >= world || !sh) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    const int64_t units = m / 1024, u0 = units * rank / world, u1 = units * (rank + 1) / world;
    const bool last = rank == world - 1;
    sh->start = 1024 * u0;
    sh->stop = last ? m : 1024 * u1;
    sh->out_start = 3 * (sh->start / 4);
    sh->out_len = b64_decoded_len_max(sh->stop - sh->start);
    sh->is_final = last ? 1 : 0;
    sh->reserved = 0;
    return B64_OK;
}

int b64_decode_finalize(const int64_t* d_err_min, int64_t* d_err_off, int32_t* d_status, b64_stream_t stream) {
    if (!d_err_min || !d_err_off) return B64_EINVAL;
    launch(dec_finalize_packed_kernel, 1, 1, reinterpret_cast<cudaStream_t>(stream), d_err_min, d_err_off, d_status);
    return launched();
}

// ---------------------------------------------------------------- grouped launches
// Items are collected into one pending group of up to kGroupMax decodes and
// kGroupMax encodes; a flush launches dec_group_kernel, enc_group_kernel, or --
// when both kinds are pending -- ONE codec_group_kernel (decode CTAs + encode
// CTAs).  Items whose pointers are not fast-path aligned, or whose chunk count
// does not fit the group's int32 chunk indices, get their own single-stream
// launch.
namespace {
constexpr int64_t kGroupChunkMax = int64_t(INT32_MAX) / 2;

struct GroupBuilder {
    const DevInfo* di;
    b64_stream_t stream;
    CodecGroup g;
    int64_t bytes = 0;

    GroupBuilder(const DevInfo* d, b64_stream_t st) : di(d), stream(st) { std::memset(&g, 0, sizeof(g)); }

    bool fused = false;  // b64_codec_group_fused: everything in ONE codec launch, nothing else

    int flush() {
        const int nd = g.d.count, ne = g.e.count;
        if (nd + ne == 0 && !fused) return B64_OK;
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        const int dd = enc_depth(bytes);
        const int64_t wmax = int64_t(di->sms) * cap_bps(di->occ_group[dd]) * (kThreads / 32);
        int64_t C[2 * kGroupMax];
        for (int i = 0; i < nd; ++i) C[i] = g.d.cstart[i + 1] - g.d.cstart[i];
        for (int i = 0; i < ne; ++i) C[nd + i] = g.e.cstart[i + 1] - g.e.cstart[i];
        if ((nd && ne) || fused) {
            // one partition over both kinds (a decode and an encode chunk move the same 1792 B);
            // each kind's warps are rounded up to whole CTAs, so one CTA of headroom is kept
            int32_t w[2 * kGroupMax + 1];
            group_partition(C, nd + ne, wmax - 2 * (kThreads / 32), w);
            for (int i = 0; i <= nd; ++i) g.d.wstart[i] = w[i];
            for (int i = 0; i <= ne; ++i) g.e.wstart[i] = w[nd + i] - w[nd];
            const int64_t wpb = kThreads / 32;
            g.dec_blocks = nd ? std::max<int64_t>(1, (int64_t(w[nd]) + wpb - 1) / wpb) : 0;
            const int64_t eb = ne ? std::max<int64_t>(1, (int64_t(w[nd + ne] - w[nd]) + wpb - 1) / wpb) : 0;
            if (fused && g.dec_blocks == 0) g.dec_blocks = 1;  // the finalizing (peer-meeting) CTA, no decodes
            launch(pick2(dd, codec_group_kernel<1>, codec_group_kernel<2>), g.dec_blocks + eb, kThreads, s, g);
        } else if (nd) {
            const int64_t blocks = group_partition(C, nd, wmax, g.d.wstart);
            launch(pick2(dd, dec_group_kernel<1>, dec_group_kernel<2>), blocks, kThreads, s, g.d);
        } else {
            const int64_t blocks = group_partition(C, ne, wmax, g.e.wstart);
            launch(pick2(dd, enc_group_kernel<1>, enc_group_kernel<2>), blocks, kThreads, s, g.e);
        }
        const int r = launched();
        std::memset(&g, 0, sizeof(g));
        bytes = 0;
        return r;
    }

    int add(const b64_encode_item& it) {
        if (it.n == 0) return B64_OK;
        const int64_t nc = it.n / 768;
        if (!(aligned(it.d_in, 8) && aligned(it.d_out, 32)) || nc >= kGroupChunkMax) {  // its own launch
            if (fused) return B64_EINVAL;
            return b64_encode(it.d_in, it.n, it.d_out, it.a, stream);
        }
        EncGroup& e = g.e;
        if (e.count == kGroupMax || e.cstart[e.count] + nc >= kGroupChunkMax) {
            if (fused) return B64_EINVAL;
            const int r = flush();
            if (r != B64_OK) return r;
        }
        const int k = e.count;
        e.in[k] = it.d_in;
        e.out[k] = it.d_out;
        e.n[k] = it.n;
        e.pad[k] = it.a->pad;
        std::memcpy(e.lut[k], it.a->enc, 64);
        e.cstart[k + 1] = e.cstart[k] + nc;
        e.count = k + 1;
        bytes += it.n;
        return B64_OK;
    }

    int add(const b64_decode_item& it, int index = 0) {
        if (it.m == 0 && !fused) return B64_OK;  // (fused: even an empty stream gets its result)
        const int64_t Q = it.m / 4;
        const int64_t Qint = (it.is_final && Q > 0) ? Q - 1 : Q;
        const int64_t nc = Qint / 256;
        if (!(aligned(it.d_in, 32) && aligned(it.d_out, 16)) || nc >= kGroupChunkMax) {
            if (fused) return B64_EINVAL;
            return b64_decode_chunk(it.d_in, it.m, it.d_out, it.a, it.base_offset, it.is_final, it.d_err_min,
                                    nullptr, stream);
        }
        DecGroup& d = g.d;
        if (d.count == kGroupMax || d.cstart[d.count] + nc >= kGroupChunkMax) {
            if (fused) return B64_EINVAL;
            const int r = flush();
            if (r != B64_OK) return r;
        }
        const int k = d.count;
        d.in[k] = it.d_in;
        d.out[k] = it.d_out;
        d.m[k] = it.m;
        d.base[k] = it.base_offset;
        d.cell[k] = reinterpret_cast<unsigned long long*>(it.d_err_min);
        d.is_final[k] = it.is_final ? 1 : 0;
        d.pad[k] = it.a->pad;
        d.lenient[k] = (it.a->flags & B64_ALPHA_LENIENT) ? 1u : 0u;
        std::memcpy(d.lut[k], it.a->dec, 256);
        d.cstart[k + 1] = d.cstart[k] + nc;
        d.count = k + 1;
        g.didx[k] = index;
        bytes += it.m;
        return B64_OK;
    }
};

int check_enc_items(const b64_encode_item* items, int64_t count) {
    if (count < 0 || (count > 0 && !items)) return B64_EINVAL;
    for (int64_t i = 0; i < count; ++i)
        if (items[i].n < 0 || !alpha_ok(items[i].a) || (items[i].n > 0 && (!items[i].d_in || !items[i].d_out)))
            return B64_EINVAL;
    return B64_OK;
}

int check_dec_items(const b64_decode_item* items, int64_t count) {
    if (count < 0 || (count > 0 && !items)) return B64_EINVAL;
    for (int64_t i = 0; i < count; ++i) {
        const b64_decode_item& it = items[i];
        if (it.m < 0 || it.base_offset < 0 || !alpha_ok(it.a) || !it.d_err_min || (it.m > 0 && (!it.d_in || !it.d_out)))
            return B64_EINVAL;
        if (it.m % 4) return B64_ELENGTH;
    }
    return B64_OK;
}
}  // namespace

int b64_codec_group(const b64_encode_item* enc, int64_t n_enc, const b64_decode_item* dec, int64_t n_dec,
                    b64_stream_t stream) {
    int r = check_enc_items(enc, n_enc);
    if (r == B64_OK) r = check_dec_items(dec, n_dec);
    if (r != B64_OK) return r;
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    GroupBuilder gb(di, stream);
    // interleaved so that a group pairs decodes with encodes when both lists are long
    for (int64_t i = 0; i < std::max(n_enc, n_dec); ++i) {
        if (i < n_dec && (r = gb.add(dec[i])) != B64_OK) return r;
        if (i < n_enc && (r = gb.add(enc[i])) != B64_OK) return r;
    }
    return gb.flush();
}

int b64_codec_group_fused(const b64_encode_item* enc, int64_t n_enc, const b64_decode_item* dec, int64_t n_dec,
                          int64_t* d_err_off, int32_t* d_status, uint32_t* d_ticket, b64_stream_t stream) {
    return b64_codec_group_fused_peer(enc, n_enc, dec, n_dec, d_err_off, d_status, d_ticket, nullptr, 1, 0, 0, stream);
}

int b64_codec_group_fused_peer(const b64_encode_item* enc, int64_t n_enc, const b64_decode_item* dec, int64_t n_dec,
                               int64_t* d_err_off, int32_t* d_status, uint32_t* d_ticket, uint8_t* const* d_peer_bufs,
                               int world, int rank, uint64_t epoch, b64_stream_t stream) {
    if (d_peer_bufs && (world < 1 || world > 32 || rank < 0 || rank >= world)) return B64_EINVAL;
    int r = check_enc_items(enc, n_enc);
    if (r == B64_OK) r = check_dec_items(dec, n_dec);
    if (r != B64_OK) return r;
    if (n_enc > kGroupMax || n_dec > kGroupMax || !d_ticket || (n_dec > 0 && !d_err_off)) return B64_EINVAL;
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    GroupBuilder gb(di, stream);
    gb.fused = true;
    for (int64_t i = 0; i < n_dec; ++i)
        if ((r = gb.add(dec[i], int(i))) != B64_OK) return r;
    for (int64_t i = 0; i < n_enc; ++i)
        if ((r = gb.add(enc[i])) != B64_OK) return r;
    gb.g.ticket = d_ticket;
    gb.g.err_off = d_err_off;
    gb.g.status = d_status;
    gb.g.peer_bufs = d_peer_bufs;
    gb.g.world = world;
    gb.g.rank = rank;
    gb.g.epoch = static_cast<unsigned long long>(epoch);
    return gb.flush();
}

int b64_decode_ctx_init(uint8_t* d_ctx, b64_stream_t stream) {
    if (!d_ctx) return B64_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(d_ctx, 0x7F, 8, s) != cudaSuccess || cudaMemsetAsync(d_ctx + 8, 0, 8, s) != cudaSuccess)
        return (cudaGetLastError(), B64_ECUDA);
    return B64_OK;
}

int b64_decode_fused(const uint8_t* d_in, int64_t m, uint8_t* d_out, const b64_alphabet* a, int64_t* d_err_off,
                     int32_t* d_status, int64_t* d_out_len, uint8_t* d_ctx, b64_stream_t stream) {
    if (m < 0 || !alpha_ok(a) || !d_err_off || !d_ctx) return B64_EINVAL;
    if (m % 4) return B64_ELENGTH;
    if (m > 0 && (!d_in || !d_out)) return B64_EINVAL;
    // small inputs: the single-launch cluster kernel needs no context; unaligned: the 3-op path
    if (m <= small_max() || !aligned(d_in, 32) || !aligned(d_out, 16))
        return b64_decode_ex(d_in, m, d_out, a, d_err_off, d_status, d_out_len, stream);
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    b64_decode_item it = {d_in, m, d_out, a, 0, 1, 0, reinterpret_cast<int64_t*>(d_ctx)};
    GroupBuilder gb(di, stream);
    gb.fused = true;
    const int r = gb.add(it, 0);
    if (r != B64_OK) return r;
    gb.g.ticket = reinterpret_cast<unsigned int*>(d_ctx + 8);
    gb.g.err_off = d_err_off;
    gb.g.status = d_status;
    gb.g.out_len = d_out_len;
    return gb.flush();
}

int b64_encode_group(const b64_encode_item* items, int64_t count, b64_stream_t stream) {
    return b64_codec_group(items, count, nullptr, 0, stream);
}

int b64_decode_group(const b64_decode_item* items, int64_t count, b64_stream_t stream) {
    return b64_codec_group(nullptr, 0, items, count, stream);
}

int b64_decode_finalize_n(const int64_t* d_err_min, int64_t count, int64_t* d_err_off, int32_t* d_status,
                          b64_stream_t stream) {
    if (count < 0 || (count > 0 && (!d_err_min || !d_err_off))) return B64_EINVAL;
    if (count == 0) return B64_OK;
    const int64_t blocks = (count + kThreads - 1) / kThreads;
    launch(dec_finalize_n_kernel, blocks > 1024 ? 1024 : blocks, kThreads, reinterpret_cast<cudaStream_t>(stream),
           d_err_min, count, d_err_off, d_status);
    return launched();
}

int b64_encode_batch(const uint8_t* d_in, const int64_t* d_in_off, int64_t count, uint8_t* d_out,
                     const int64_t* d_out_off, const b64_alphabet* a, b64_stream_t stream) {
    if (count < 0 || !alpha_ok(a)) return B64_EINVAL;
    if (count == 0) return B64_OK;
    if (!d_in || !d_in_off || !d_out || !d_out_off) return B64_EINVAL;
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    Offsets off{d_in_off, d_out_off, count, 0};
    const int64_t blocks = int64_t(di->sms) * di->occ_enc_gen;
    launch(enc_generic_kernel, blocks, kThreads, reinterpret_cast<cudaStream_t>(stream), d_in, d_out, off, enc_tab(a), a->pad);
    return launched();
}

int b64_decode_batch(const uint8_t* d_in, const int64_t* d_in_off, int64_t count, uint8_t* d_out,
                     const int64_t* d_out_off, const b64_alphabet* a, int32_t* d_status, int64_t* d_err_off,
                     int64_t* d_out_len, b64_stream_t stream) {
    return b64_decode_batch_ex(d_in, d_in_off, count, d_out, d_out_off, a, d_status, d_err_off, d_out_len, 0, nullptr,
                               stream);
}

int b64_decode_batch_ex(const uint8_t* d_in, const int64_t* d_in_off, int64_t count, uint8_t* d_out,
                        const int64_t* d_out_off, const b64_alphabet* a, int32_t* d_status, int64_t* d_err_off,
                        int64_t* d_out_len, int64_t index_base, int64_t* d_first_bad, b64_stream_t stream) {
    return b64_decode_batch_fast(d_in, d_in_off, count, d_out, d_out_off, a, d_status, d_err_off, d_out_len,
                                 index_base, d_first_bad, nullptr, stream);
}

int b64_batch_ctx_init(uint8_t* d_ctx, b64_stream_t stream) {
    if (!d_ctx) return B64_EINVAL;
    note(cudaMemsetAsync(d_ctx, 0, B64_BATCH_CTX_BYTES, reinterpret_cast<cudaStream_t>(stream)));
    const int r = launched();
    if (r == B64_OK) g_launches.fetch_sub(1, std::memory_order_relaxed);  // a memset, not a kernel
    return r;
}

int b64_decode_batch_fast(const uint8_t* d_in, const int64_t* d_in_off, int64_t count, uint8_t* d_out,
                          const int64_t* d_out_off, const b64_alphabet* a, int32_t* d_status, int64_t* d_err_off,
                          int64_t* d_out_len, int64_t index_base, int64_t* d_first_bad, uint8_t* d_ctx,
                          b64_stream_t stream) {
    if (count < 0 || !alpha_ok(a) || index_base < 0 || (d_first_bad && count > INT64_MAX - index_base))
        return B64_EINVAL;
    if (count == 0) return B64_OK;
    if (!d_in || !d_in_off || !d_out || !d_out_off || !d_err_off) return B64_EINVAL;
    const DevInfo* di = dev_info();
    if (!di) return B64_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    BatchCtx* ctx = reinterpret_cast<BatchCtx*>(d_ctx);
    unsigned long long* cells = reinterpret_cast<unsigned long long*>(d_err_off);
    const int64_t small = clamp_grid((count + kThreads - 1) / kThreads, int64_t(di->sms) * 8);
    int r;
    if (ctx) {
        // the concatenation path (batch.cu): layout check, bulk, final quads; the generic
        // kernel below then only runs when the layout is not eligible or a pad is misplaced
        launch(dec_batch_prep_kernel, small, kThreads, s, d_in, d_in_off, static_cast<const uint8_t*>(d_out),
               d_out_off, count, d_err_off, ctx);
        if ((r = launched()) != B64_OK) return r;
        DecTab bt = dec_tab(a);
        reinterpret_cast<uint8_t*>(bt.w)[a->pad] = uint8_t(kPadCand);
        launch(dec_batch_bulk_kernel<2>, int64_t(di->sms) * cap_bps(di->occ_batch_bulk), kThreads, s, d_in, d_in_off,
               d_out, d_out_off, count, bt, cells, ctx);
        if ((r = launched()) != B64_OK) return r;
        const int64_t per = clamp_grid((count + 4 * kThreads - 1) / (4 * kThreads), INT32_MAX);  // 4 strings per thread
        launch(dec_batch_strfinal_kernel, per, kThreads, s, d_in, d_in_off, d_out, d_out_off, count, dec_tab(a),
               d_err_off, d_status, d_out_len, index_base, reinterpret_cast<unsigned long long*>(d_first_bad), ctx);
        if ((r = launched()) != B64_OK) return r;
    }
    // the per-string path (b64_decode_batch_ex); with a context every kernel is gated on
    // ctx->generic and returns at once when the concatenation path finished the batch
    launch(dec_batch_init_kernel, small, kThreads, s, d_err_off, count, static_cast<const BatchCtx*>(ctx));
    if ((r = launched()) != B64_OK) return r;
    Offsets off{d_in_off, d_out_off, count, 0};
    const int64_t blocks = int64_t(di->sms) * di->occ_dec_gen;
    launch(dec_generic_kernel, blocks, kThreads, s, d_in, d_out, off, dec_tab(a), 0, 1, cells, nullptr,
           static_cast<const BatchCtx*>(ctx));
    if ((r = launched()) != B64_OK) return r;
    launch(dec_batch_finalize_kernel, small, kThreads, s, d_in, d_in_off, count, a->pad, d_status,
           d_err_off, d_out_len, index_base, reinterpret_cast<unsigned long long*>(d_first_bad), ctx);
    return launched();
}

int64_t b64_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* b64_build_info(void) {
#define B64_STR2(x) #x
#define B64_STR(x) B64_STR2(x)
    return "b64gpu sm_100a, nvcc " B64_STR(__CUDACC_VER_MAJOR__) "." B64_STR(__CUDACC_VER_MINOR__)
           "; kernels enc_fast dec_fast enc_generic dec_generic {enc,dec,codec}_group dec_small ws_* "
           "{enc,dec}_stream_* peer_combine ws_line_* dec_finalize_* dec_batch_*";
}

}  // extern "C"
