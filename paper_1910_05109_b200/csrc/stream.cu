// stream.cu -- streaming (chunked) encode and validating decode with a carry
// between calls (reading R15).
//
// Input arrives in pieces of any length.  Whole triples (encode) / quads
// (decode) are coded as soon as they are complete; the bytes / chars of an
// incomplete group are held in a small caller-owned device buffer (the carry)
// until the next call.  Decode always holds the last 1-4 chars back, so the
// stream's final quad -- the only one where '=' may appear (R6) --
// is checked by the end call with the final-quad rules, and every quad decoded
// earlier is an interior quad.  The result equals the one-shot encode / decode
// of the concatenated input byte for byte, with error positions in the
// coordinates of the concatenation.
//
// Per update: ONE single-thread join kernel (the group that straddles the
// previous piece and this one, and the new carry), then the bulk of the piece
// through the single-stream kernels (b64_encode / b64_decode_chunk, which pick
// the fast or the generic kernel by alignment).  The carry is kept in device
// memory so no call waits for the device.
#include "b64_device.cuh"

namespace b64 {

// The join of a streaming encode on its own (enc_stream_join, encode.cu), when it cannot ride
// along with the piece's bulk kernel.
__global__ void enc_stream_join_kernel(uint8_t* __restrict__ carry, int H, const uint8_t* __restrict__ in, int64_t n,
                                       uint8_t* __restrict__ out, EncTab tab) {
    griddep_wait();
    carry = after_wait(carry);  // written by the previous piece's kernel
    enc_stream_join(carry, H, in, n, out, reinterpret_cast<const uint8_t*>(tab.w));
}

// The end of an encode stream: the H (1 or 2) held bytes -> 4 chars with '='
// padding.
__global__ void enc_stream_end_kernel(const uint8_t* __restrict__ carry, int H, uint8_t* __restrict__ out, EncTab tab,
                                      uint32_t pad) {
    griddep_wait();
    carry = after_wait(carry);  // written by the previous piece's kernel
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(tab.w);
    const uint32_t v = enc_partial(carry[0], H == 2 ? carry[1] : 0u, H, lut, pad);
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = uint8_t(v >> (8 * k));
}

// carry[0..H) are held chars (H <= 4) starting at global position base;
// in[0..m) is the new piece.  A = H + m chars are available; Q = (A - 1) / 4
// quads are decoded now (the last R = A - 4Q chars, 1..4, are held).  If
// H > 0 and Q >= 1 the first of them is the straddling quad carry ++ in[0 ..
// 4-H), decoded here as an interior quad to out[0..3) (errors into *cell at
// their global position).  The new carry is the last R chars.
__global__ void dec_stream_join_kernel(uint8_t* __restrict__ carry, int H, const uint8_t* __restrict__ in, int64_t m,
                                       uint8_t* __restrict__ out, DecTab tab, int64_t base,
                                       unsigned long long* __restrict__ cell) {
    griddep_wait();
    stream_join(carry, H, in, m, out, reinterpret_cast<const uint8_t*>(tab.w), base, cell);
}

// The end of a decode stream of `total` chars: carry[0..H) holds its last
// H chars (H == 4 when total % 4 == 0 and total > 0).  total % 4 != 0 ->
// LENGTH at total - total % 4 (no content verdict, as the one-shot rule);
// else the final quad (R6) -> 1-3 bytes at out.  Then the packed
// error word -> (err_off, status, out_len) as b64_decode_ex.
__global__ void dec_stream_end_kernel(const uint8_t* __restrict__ carry, int H, int64_t total,
                                      uint8_t* __restrict__ out, DecTab tab,
                                      const unsigned long long* __restrict__ cell, int64_t* __restrict__ err_off,
                                      int32_t* __restrict__ status, int64_t* __restrict__ out_len) {
    griddep_wait();
    const uint8_t* lut = reinterpret_cast<const uint8_t*>(tab.w);
    unsigned long long wv = *cell;
    int64_t ol = 0;
    if (total & 3) {
        wv = pack_err(total - (total & 3), kLength);
    } else if (total > 0) {
        const uint32_t x = uint32_t(carry[0]) | (uint32_t(carry[1]) << 8) | (uint32_t(carry[2]) << 16) |
                           (uint32_t(carry[3]) << 24);
        int bad, k;
        uint32_t v;
        const uint32_t kind = final_quad(x, lut, tab.pad, tab.lenient, &bad, &k, &v);
        if (kind == kOk) store_bytes(out, v, k);
        else wv = min(wv, pack_err(total - 4 + bad, kind));
        ol = 3 * (total / 4 - 1) + k;
    }
    if (wv >= kErrNone) {
        *err_off = -1;
        if (status) *status = kOk;
        if (out_len) *out_len = ol;
    } else {
        const int64_t pos = int64_t(wv >> 3);
        const int32_t kind = int32_t(wv & 7);
        *err_off = pos;
        if (status) *status = kind;
        if (out_len) *out_len = kind == int32_t(kLength) ? 0 : 3 * (pos >> 2);
    }
}

}  // namespace b64
