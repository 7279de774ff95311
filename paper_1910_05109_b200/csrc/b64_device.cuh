// b64_device.cuh -- device building blocks of the sm_100a base64 codec.
//
// The paper's AVX-512 design (Sec. 3, 512-bit registers, vpermb /
// vpmultishiftqb / vpermi2b / vpmaddubsw / vpmaddwd) is prior art; the B200
// mapping used here:
//   * one 32-bit register holds one triple (encode) or one quad (decode);
//     PRMT (__byte_perm) is the vpermb gather and the
//     vpermb compaction, SHF/LOP3 the bit relayout
//     (PAPER.md:201-237), IMAD the multiply-add packing;
//   * the alphabet / decode tables are runtime kernel parameters staged to a
//     64 B / 256 B shared-memory table per CTA: the vpermb / vpermi2b lookups
//     become one LDS.U8 per character (64 B spans 16 banks and ASCII indexes of
//     the 256 B table fall in 32 distinct banks: conflict-free);
//   * deferred validation: a per-thread OR accumulator of the
//     translated values, tested once per 32 characters; only when a bit 0x80 is
//     set does the warp locate the first bad character (vote + __reduce_min_sync
//     + one 64-bit atomicMin) -- the paper stops at "invalid", we report where.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace b64 {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kThreads = 256;          // threads per CTA for every kernel
constexpr int kBulkCtasPerSm = 5;      // resident CTAs per SM of the bulk kernels (<= 48 registers)
constexpr uint32_t kInvalid = 0x80u;   // decode-table sentinel

constexpr unsigned long long kErrNone = 0x7F7F7F7F7F7F7F7FULL;  // B64_ERR_NONE
enum : uint32_t { kOk = 0, kBadChar = 1, kBadPad = 2, kNonCanon = 3, kLength = 4 };

// Alphabet tables passed BY VALUE as kernel parameters (runtime constants,
// PAPER.md:240).
struct EncTab { uint32_t w[16]; };             // enc[64] chars
struct DecTab { uint32_t w[64]; uint32_t pad; uint32_t lenient; };  // dec[256] + pad char + R16 flag

// Programmatic dependent launch (PDL): kernels are launched so the next
// kernel on the stream may start its prologue while this one drains; each
// kernel waits for its predecessor's memory before touching global memory.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// A pointer whose value is (re)defined by an asm volatile placed after griddep_wait(): no load
// through it -- not even an LDG.CONSTANT of a `const __restrict__` parameter, which the
// compiler treats as invariant and may hoist -- can be scheduled before the wait, where it
// would read the predecessor grid's output before it is written (tools/check_pdl_order.py).
template <class T>
__device__ __forceinline__ T* after_wait(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}

__device__ __forceinline__ unsigned long long pack_err(int64_t pos, uint32_t kind) {
    return ((unsigned long long)pos << 3) | kind;
}

// ----------------------------------------------------------------- memory ops
// 256-bit lane-linear load, no L1 allocation (streamed once).
__device__ __forceinline__ void ld256_stream(const void* p, uint32_t (&r)[8]) {
    asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "l"(p));
}
// 64-bit load that allocates in L1: three of them at a lane stride of 24 B
// cover 768 contiguous bytes per warp; the first one brings every sector into
// L1 and the next two hit there (DRAM reads each byte once).
__device__ __forceinline__ uint2 ld64_l1(const void* p) {
    uint2 r;
    asm("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld128_nc(const void* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld32_nc(const void* p) {  // streamed once: no L1 allocation
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld32(const void* p) {
    uint32_t r;
    asm("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void st256(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void st64(void* p, uint32_t a, uint32_t b) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void st128(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ----------------------------------------------------------------- shared memory by 32-bit address
// The look-up tables are addressed with 32-bit shared-window addresses so the
// table base can be merged into the index computation (one PRMT or LOP3 per
// character instead of extract + add).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t r;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" :: "r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}

// mbarrier + bulk async copy (TMA, non-tensor form): one elected lane arms the barrier with
// the byte count and issues the copy; every lane waits on the phase parity before reading.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global -> shared bulk copy: src / dst 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}

// Encode one triple (x: byte3 = s1, byte2 = s2, byte1 = s3) with the 64-entry
// alphabet at the 64-byte-aligned shared address lb: index | lb == lb + index.
// The right shifts are done as high halves of multiplies (IMAD.HI, FMA pipe)
// and the four chars are packed with IMADs, so the ALU pipe only carries the
// PRMT gather and one LOP3 per char: the two integer pipes are balanced.
__device__ __forceinline__ uint32_t enc_triple_s(uint32_t x, uint32_t lb) {
    const uint32_t c0 = lds_u8(__umulhi(x, 1u << 6) + lb);
    const uint32_t c1 = lds_u8((__umulhi(x, 1u << 12) & 63u) | lb);
    const uint32_t c2 = lds_u8((__umulhi(x, 1u << 18) & 63u) | lb);
    const uint32_t c3 = lds_u8((__umulhi(x, 1u << 24) & 63u) | lb);
    return (c3 * 256u + c2) * 65536u + (c1 * 256u + c0);
}

// Decode one quad with the 256-entry table at the 256-byte-aligned shared
// address lb: PRMT drops each char into the low byte of lb -> its entry address.
__device__ __forceinline__ uint32_t dec_quad_s(uint32_t x, uint32_t lb, uint32_t& err) {
    const uint32_t a = lds_u8(__byte_perm(x, lb, 0x7650));
    const uint32_t b = lds_u8(__byte_perm(x, lb, 0x7651));
    const uint32_t c = lds_u8(__byte_perm(x, lb, 0x7652));
    const uint32_t d = lds_u8(__byte_perm(x, lb, 0x7653));
    err |= a | b | c | d;
    return (((a * 64u + b) * 64u + c) * 64u) + d;
}

// 4 aligned words starting at an arbitrary byte address p, funnel-shifted to
// the bytes p[0..16) (little-endian).  Reads only the aligned words that
// contain p[0..16) (b64gpu.h conventions).
template <int NW>
__device__ __forceinline__ void ld_unaligned(const uint8_t* p, uint32_t (&w)[NW]) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const uint32_t* pa = reinterpret_cast<const uint32_t*>(u & ~uintptr_t(3));
    const uint32_t sh = uint32_t(u & 3) * 8u;
    uint32_t a[NW + 1];
#pragma unroll
    for (int i = 0; i < NW; ++i) a[i] = ld32(pa + i);
    if (sh == 0) {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = a[i];
    } else {
        a[NW] = ld32(pa + NW);
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = __funnelshift_r(a[i], a[i + 1], sh);
    }
}

// 24 / 32 bytes at any address, as 8-byte-aligned LDG.64 + funnel shifts.
// Reads only the naturally aligned 8-byte words that contain p[0..NB)
// (b64gpu.h conventions).
template <int NW>  // NW = 6 (24 B) or 8 (32 B)
__device__ __forceinline__ void ld_unaligned64(const uint8_t* p, uint32_t (&w)[NW]) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const uint2* pa = reinterpret_cast<const uint2*>(u & ~uintptr_t(7));
    const uint32_t sb = uint32_t(u & 7);
    uint32_t v[NW + 4];
#pragma unroll
    for (int i = 0; i < NW / 2; ++i) {
        const uint2 q = ld64_l1(pa + i);
        v[2 * i] = q.x;
        v[2 * i + 1] = q.y;
    }
    if (sb) {
        const uint2 q = ld64_l1(pa + NW / 2);
        v[NW] = q.x;
        v[NW + 1] = q.y;
    } else {
        v[NW] = 0;
        v[NW + 1] = 0;
    }
    const bool ws = sb >= 4;
    const uint32_t sh = (sb & 3) * 8;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const uint32_t lo = ws ? v[i + 1] : v[i];
        const uint32_t hi = ws ? v[i + 2] : v[i + 1];
        w[i] = __funnelshift_r(lo, hi, sh);
    }
}
__device__ __forceinline__ void ld24_unaligned(const uint8_t* p, uint32_t (&w)[6]) { ld_unaligned64<6>(p, w); }
// NW words at any alignment from 2-3 aligned 16-byte loads (L1-allocating: a neighbouring
// lane's unit shares the edge blocks) -- fewer L1 wavefronts than LDG.64 for the batch
// decode, whose 32-char units sit at a 32-byte lane stride (tools/ab_batch.sh: configs[3]
// decode +0.6 %, 64 KiB strings +2.6 %; the 24-byte encode units measured 11 % slower).
__device__ __forceinline__ uint4 ld128_l1(const void* p) {
    uint4 r;
    asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
template <int NW>
__device__ __forceinline__ void ld_unaligned128(const uint8_t* p, uint32_t (&x)[NW]) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const uint4* pa = reinterpret_cast<const uint4*>(u & ~uintptr_t(15));
    const uint32_t sb = uint32_t(u & 15);
    const uint4 a = ld128_l1(pa), b = ld128_l1(pa + 1);
    const uint4 c = (4 * NW + sb > 32) ? ld128_l1(pa + 2) : make_uint4(0, 0, 0, 0);
    const uint32_t v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    const int ws = int(sb >> 2);
    const uint32_t sh = (sb & 3) * 8;
    uint32_t wsel[NW + 1];
#pragma unroll
    for (int i = 0; i <= NW; ++i)
        wsel[i] = ws == 0 ? v[i] : ws == 1 ? v[i + 1] : ws == 2 ? v[i + 2] : v[i + 3 < 12 ? i + 3 : 11];
#pragma unroll
    for (int i = 0; i < NW; ++i) x[i] = __funnelshift_r(wsel[i], wsel[i + 1], sh);
}
__device__ __forceinline__ void ld32_unaligned128(const uint8_t* p, uint32_t (&x)[8]) { ld_unaligned128<8>(p, x); }

__device__ __forceinline__ void ld32_unaligned(const uint8_t* p, uint32_t (&w)[8]) { ld_unaligned64<8>(p, w); }

// ----------------------------------------------------------------- encode
// One triple, given x with byte3 = s1, byte2 = s2, byte1 = s3 (byte0 unused):
// the four 6-bit values of PAPER.md:88-92 are bits [26,32), [20,26), [14,20),
// [8,14) of x; each indexes the 64-entry alphabet.
__device__ __forceinline__ uint32_t enc_triple(uint32_t x, const uint8_t* __restrict__ lut) {
    const uint32_t c0 = lut[x >> 26];
    const uint32_t c1 = lut[(x >> 20) & 63u];
    const uint32_t c2 = lut[(x >> 14) & 63u];
    const uint32_t c3 = lut[(x >> 8) & 63u];
    return __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
}

// 12 input bytes (3 LE words) -> 16 chars (4 LE words).  The PRMT selectors
// gather (s1, s2, s3) of triple t from bytes 3t..3t+2 -- the role of the
// paper's first vpermb with indexes (3i+1, 3i, 3i+2, 3i+1).
__device__ __forceinline__ void enc12(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t (&o)[4],
                                      const uint8_t* __restrict__ lut) {
    o[0] = enc_triple(__byte_perm(w0, w1, 0x0122), lut);
    o[1] = enc_triple(__byte_perm(w0, w1, 0x3455), lut);
    o[2] = enc_triple(__byte_perm(w1, w2, 0x2344), lut);
    o[3] = enc_triple(__byte_perm(w2, w2, 0x1233), lut);
}

// r (1 or 2) leftover bytes s1[, s2] -> 4 chars with '=' padding.
__device__ __forceinline__ uint32_t enc_partial(uint32_t s1, uint32_t s2, int r,
                                                const uint8_t* __restrict__ lut, uint32_t pad) {
    const uint32_t x = (s1 << 24) | (r == 2 ? (s2 << 16) : 0u);
    const uint32_t c0 = lut[x >> 26];
    const uint32_t c1 = lut[(x >> 20) & 63u];
    const uint32_t c2 = (r == 2) ? uint32_t(lut[(x >> 14) & 63u]) : pad;
    return c0 | (c1 << 8) | (c2 << 16) | (pad << 24);
}

// ----------------------------------------------------------------- decode
// One quad (4 chars, LE in x) -> 24-bit value a*2^18 + b*2^12 + c*2^6 + d
// (PAPER.md:98-99, 540-548); err collects the translated values so a set bit
// 0x80 marks an invalid character.
__device__ __forceinline__ uint32_t dec_quad(uint32_t x, const uint8_t* __restrict__ lut, uint32_t& err) {
    const uint32_t a = lut[x & 0xffu];
    const uint32_t b = lut[__byte_perm(x, 0, 0x4441)];
    const uint32_t c = lut[__byte_perm(x, 0, 0x4442)];
    const uint32_t d = lut[x >> 24];
    err |= a | b | c | d;
    return (((a * 64u + b) * 64u + c) * 64u) + d;
}

// 4 decoded quads -> 12 output bytes in 3 LE words, in stream order
// (v>>16, v>>8, v per quad): the paper's compaction vpermb (PAPER.md:551-556,
// read most-significant byte first per dword, R3).
__device__ __forceinline__ void dec_pack12(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3,
                                           uint32_t& o0, uint32_t& o1, uint32_t& o2) {
    o0 = __byte_perm(v0, v1, 0x6012);
    o1 = __byte_perm(v1, v2, 0x5601);
    o2 = __byte_perm(v2, v3, 0x4560);
}

// Index (0..3) of the first invalid char of quad x, or 4.
__device__ __forceinline__ int first_bad_in_quad(uint32_t x, const uint8_t* __restrict__ lut) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (lut[(x >> (8 * j)) & 0xffu] & kInvalid) return j;
    return 4;
}

// The stream's final quad (R6, "final and separate code path",
// PAPER.md:569).  Returns the error kind (kOk when valid); *bad = 0..3 the
// offending position within the quad; *k = output bytes (1..3) when valid and
// *v = the 24-bit value.  lenient (R16): non-zero trailing bits are
// dropped instead of reported as NONCANON.
__device__ __forceinline__ uint32_t final_quad(uint32_t x, const uint8_t* __restrict__ lut, uint32_t pad,
                                               uint32_t lenient, int* bad, int* k, uint32_t* v) {
    const uint32_t ch0 = x & 0xffu, ch1 = (x >> 8) & 0xffu, ch2 = (x >> 16) & 0xffu, ch3 = x >> 24;
    const uint32_t a = lut[ch0], b = lut[ch1], c = lut[ch2], d = lut[ch3];
    const bool p2 = ch2 == pad, p3 = ch3 == pad;
    *k = p2 ? 1 : (p3 ? 2 : 3);
    *v = 0;
    if (a & kInvalid) { *bad = 0; return kBadChar; }
    if (b & kInvalid) { *bad = 1; return kBadChar; }
    if ((c & kInvalid) && !p2) { *bad = 2; return kBadChar; }
    if ((d & kInvalid) && !p3) { *bad = 3; return kBadChar; }
    if (p2 && !p3) { *bad = 3; return kBadPad; }
    if (!lenient && p2 && (b & 15u)) { *bad = 1; return kNonCanon; }
    if (!lenient && !p2 && p3 && (c & 3u)) { *bad = 2; return kNonCanon; }
    *v = (a << 18) | (b << 12) | ((p2 ? 0u : c) << 6) | (p3 ? 0u : d);
    return kOk;
}

__device__ __forceinline__ void store_bytes(uint8_t* o, uint32_t v, int k) {
    o[0] = uint8_t(v >> 16);
    if (k >= 2) o[1] = uint8_t(v >> 8);
    if (k >= 3) o[2] = uint8_t(v);
}

// Offsets of a batch of strings concatenated in one buffer; in_off == nullptr
// means a single stream [0, n).  (b64gpu.h batched conventions.)
struct Offsets {
    const int64_t* in_off;
    const int64_t* out_off;
    int64_t count;
    int64_t n;
    __device__ __forceinline__ int64_t in(int64_t i) const { return in_off ? in_off[i] : (i == 0 ? 0 : n); }
    __device__ __forceinline__ int64_t out(int64_t i) const { return out_off ? out_off[i] : 0; }
};

// First string s whose end in_off[s+1] > pos: strings ending at or before pos
// own nothing at or after pos.
__device__ __forceinline__ int64_t first_string_ending_after(const Offsets& off, int64_t pos) {
    int64_t lo = 0, hi = off.count;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (off.in(mid + 1) > pos) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// Context of the batched decode's concatenation path (batch.cu): caller-owned,
// self-resetting (B64_BATCH_CTX_BYTES = 32, all zero initially).
struct BatchCtx {
    uint32_t generic;          // 1: the per-string generic kernel must run
    uint32_t ticket;           // strfinal's last-CTA ticket
    unsigned long long eq;     // pad chars the bulk pass saw
    unsigned long long legit;  // pad chars at positions len-2 / len-1 of the strings
    uint32_t reserved[2];      // [0]: the gated finalize's last-CTA ticket
};
static_assert(sizeof(BatchCtx) == 32, "B64_BATCH_CTX_BYTES");

// Kernel entry points (defined in encode.cu / decode.cu, launched by capi.cu).
template <int D>
__global__ void enc_fast_kernel(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out, EncTab tab,
                                uint32_t pad);
__global__ void enc_generic_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, Offsets off, EncTab tab,
                                   uint32_t pad);
// A streaming decode's join (stream.cu): the quad made of the H held chars and the piece's
// first 4 - H chars, and the carry update (the piece's last R chars), folded into the piece's
// bulk kernel when that is dec_fast (active = 0: nothing to do).
// A streaming encode's join riding along with an overlapped piece's enc_fastu_kernel<true>
// (its last thread, after the wait).
struct EncJoin {
    uint8_t* carry;
    const uint8_t* in;   // the piece
    uint8_t* out;        // the piece's output (the straddling triple's 4 chars go first)
    int64_t n;           // piece bytes
    int32_t H;           // held bytes before the piece
    int32_t active;
};
struct StreamJoin {
    uint8_t* carry;
    const uint8_t* in;   // the piece
    uint8_t* out;        // the piece's output (the join quad's 3 bytes go first)
    int64_t m;           // piece chars
    int64_t base;        // stream position of the join quad (consumed - H)
    int32_t H;           // held chars before the piece
    int32_t active;
};
template <int D, bool EARLY = false>
__global__ void dec_fast_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab,
                                int64_t base, int is_final, unsigned long long* __restrict__ err_cell,
                                int64_t* __restrict__ out_len, const int64_t* __restrict__ m_dev, StreamJoin join);
__global__ void dec_generic_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, Offsets off,
                                   DecTab tab, int64_t base, int is_final_single,
                                   unsigned long long* __restrict__ err_cells, int64_t* __restrict__ out_len_single,
                                   const BatchCtx* gate);
__global__ void dec_small_kernel(const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out, DecTab tab,
                                 int64_t* __restrict__ err_off, int32_t* __restrict__ status,
                                 int64_t* __restrict__ out_len);
__global__ void dec_finalize_single_kernel(int64_t* err_off, int32_t* status, int64_t* out_len,
                                           const uint8_t* __restrict__ in, int64_t m, uint32_t pad);
__global__ void dec_finalize_unpadded_kernel(int64_t* err_off, int32_t* status, int64_t* out_len,
                                             const uint8_t* __restrict__ in, int64_t m, uint8_t* __restrict__ out,
                                             DecTab tab);
__global__ void dec_finalize_packed_kernel(const int64_t* cell, int64_t* err_off, int32_t* status);
__global__ void dec_finalize_len_kernel(const int64_t* cell, int64_t* err_off, int32_t* status, int64_t* out_len,
                                        int64_t out_base);
__global__ void dec_batch_init_kernel(int64_t* err, int64_t count, const BatchCtx* gate);
__global__ void dec_batch_finalize_kernel(const uint8_t* __restrict__ in, const int64_t* __restrict__ in_off,
                                          int64_t count, uint32_t pad, int32_t* status, int64_t* err,
                                          int64_t* out_len, int64_t index_base, unsigned long long* first_bad,
                                          BatchCtx* ctx);

}  // namespace b64
