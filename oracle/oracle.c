/*
 * oracle.c -- plain scalar lookup-table base64 codec.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1910_05109_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * What it computes is the plain definition of base64 as the paper states it
 * (arXiv 1910.05109, Mula & Lemire), written out one byte / one quad at a time
 * with no blocking, fusion or reordering:
 *
 *   encode  PAPER.md:88-92 (Sec. 2): s1 div 4, (s2 div 16) + (s1*16) mod 64,
 *           (s2*4) mod 64 + (s3 div 64), s3 mod 64, each mapped to a char
 *           through the 64-entry alphabet.
 *           Padding '=' so the length is a multiple of 4.
 *   decode  PAPER.md:96-99 (Sec. 2): a char -> [0,64) or a special "invalid"
 *           value via a lookup table; (a*4) + (b div 16),
 *           (b*16) mod 256 + (c div 4), (c*64) mod 256 + d.
 *
 * Where the paper is silent (strict padding, error offset) this follows the
 * readings listed in DESIGN.md "Readings of the paper" (R5-R8), which are
 * SURVEY.md Sec. 8(c):
 *   - m % 4 != 0  -> status LENGTH, err_off = m - m % 4, nothing decoded;
 *   - err_off = smallest bad position; interior chars must be in the alphabet;
 *     the final quad allows '=' at m-2 and m-1 only, no data after '=',
 *     and zero trailing bits (canonical), checked in that order;
 *   - out_len = bytes that are exact: the whole decoded length when valid,
 *     3 * floor(err_off / 4) otherwise.
 *
 * Pinned by tests/test_oracle_pins.py (Python base64 library exhaustively,
 * the paper's Sec. 3.1 / 3.2 vector algorithms emulated from their printed
 * constants, Fig. 2's worked values, the padding round-trip invariant, and
 * error injection).  Parity status per function is listed in DESIGN.md.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INVALID 0xFFu /* the paper's "special value" */

enum {
    ORACLE_ST_OK = 0,
    ORACLE_ST_BADCHAR = 1,  /* byte outside the alphabet (or misplaced pad) */
    ORACLE_ST_BADPAD = 2,   /* data after padding                          */
    ORACLE_ST_NONCANON = 3, /* non-zero trailing bits in a padded quad     */
    ORACLE_ST_LENGTH = 4    /* m % 4 != 0                                  */
};

/* Alphabet validity (R4): 64 distinct chars < 0x80,
 * pad < 0x80 and not one of them.  Returns 0, or -3 duplicate, -4 non-ASCII,
 * -5 pad in alphabet; *bad_index gets the offending index (64 = the pad). */
int oracle_alphabet_check(const uint8_t chars[64], uint8_t pad, int *bad_index)
{
    int i, j;
    *bad_index = -1;
    for (i = 0; i < 64; i++) {
        if (chars[i] >= 0x80) { *bad_index = i; return -4; }
    }
    if (pad >= 0x80) { *bad_index = 64; return -4; }
    for (i = 0; i < 64; i++) {
        for (j = 0; j < i; j++) {
            if (chars[i] == chars[j]) { *bad_index = i; return -3; }
        }
    }
    for (i = 0; i < 64; i++) {
        if (chars[i] == pad) { *bad_index = i; return -5; }
    }
    return 0;
}

/* Length law: 4 * ceil(n / 3). */
int64_t oracle_encoded_len(int64_t n)
{
    return 4 * ((n + 2) / 3);
}

/* Encode n bytes; writes exactly oracle_encoded_len(n) chars; returns that. */
int64_t oracle_encode(const uint8_t *in, int64_t n, uint8_t *out,
                      const uint8_t chars[64], uint8_t pad)
{
    int64_t i = 0, o = 0;
    /* full triples */
    for (; i + 3 <= n; i += 3) {
        unsigned s1 = in[i], s2 = in[i + 1], s3 = in[i + 2];
        out[o++] = chars[s1 / 4];
        out[o++] = chars[(s2 / 16) + (s1 * 16) % 64];
        out[o++] = chars[(s2 * 4) % 64 + (s3 / 64)];
        out[o++] = chars[s3 % 64];
    }
    /* leftover 1 or 2 bytes: the same formulas with the missing bytes taken
     * as zero, then '=' so the output length is a multiple of four
     * ("conventional code path"). */
    if (n - i == 1) {
        unsigned s1 = in[i], s2 = 0;
        out[o++] = chars[s1 / 4];
        out[o++] = chars[(s2 / 16) + (s1 * 16) % 64];
        out[o++] = pad;
        out[o++] = pad;
    } else if (n - i == 2) {
        unsigned s1 = in[i], s2 = in[i + 1], s3 = 0;
        out[o++] = chars[s1 / 4];
        out[o++] = chars[(s2 / 16) + (s1 * 16) % 64];
        out[o++] = chars[(s2 * 4) % 64 + (s3 / 64)];
        out[o++] = pad;
    }
    return o;
}

/* The decode look-up table of: every byte value maps to the
 * special value except the 64 alphabet chars, which map to their index. */
static void build_decode_table(const uint8_t chars[64], uint8_t dec[256])
{
    int v;
    memset(dec, ORACLE_INVALID, 256);
    for (v = 0; v < 64; v++) dec[chars[v]] = (uint8_t)v;
}

/* Decode m chars.  Returns the status kind; *out_len and *err_off as in the
 * header comment (err_off = -1 when valid).  lenient != 0 (DESIGN.md reading
 * R16): the canonical-bits check is skipped -- the low bits of the last char
 * before the padding are dropped, as Python's binascii strict mode and GNU
 * coreutils do; every other rule is unchanged. */
static int decode_opt(const uint8_t *in, int64_t m, uint8_t *out,
                      const uint8_t chars[64], uint8_t pad, int lenient,
                      int64_t *out_len, int64_t *err_off)
{
    uint8_t dec[256];
    int64_t q, nq;
    build_decode_table(chars, dec);
    *out_len = 0;
    *err_off = -1;
    if (m % 4 != 0) {
        *err_off = m - m % 4;
        return ORACLE_ST_LENGTH;
    }
    nq = m / 4;
    for (q = 0; q < nq; q++) {
        const uint8_t *c = in + 4 * q;
        int64_t p = 4 * q;
        uint8_t *o = out + 3 * q;
        if (q < nq - 1) {
            /* interior quad: all four chars must be in the alphabet */
            int j;
            for (j = 0; j < 4; j++) {
                if (dec[c[j]] == ORACLE_INVALID) {
                    *err_off = p + j;
                    *out_len = 3 * q;
                    return ORACLE_ST_BADCHAR;
                }
            }
            {
                unsigned a = dec[c[0]], b = dec[c[1]], cc = dec[c[2]], d = dec[c[3]];
                o[0] = (uint8_t)((a * 4) + (b / 16));
                o[1] = (uint8_t)((b * 16) % 256 + (cc / 4));
                o[2] = (uint8_t)((cc * 64) % 256 + d);
            }
        } else {
            /* the final quad ("final and separate code path") */
            int kind = ORACLE_ST_OK;
            int64_t bad = -1;
            int pad2 = (c[2] == pad), pad3 = (c[3] == pad);
            if (dec[c[0]] == ORACLE_INVALID) { bad = p; kind = ORACLE_ST_BADCHAR; }
            else if (dec[c[1]] == ORACLE_INVALID) { bad = p + 1; kind = ORACLE_ST_BADCHAR; }
            else if (dec[c[2]] == ORACLE_INVALID && !pad2) { bad = p + 2; kind = ORACLE_ST_BADCHAR; }
            else if (dec[c[3]] == ORACLE_INVALID && !pad3) { bad = p + 3; kind = ORACLE_ST_BADCHAR; }
            else if (pad2 && !pad3) { bad = p + 3; kind = ORACLE_ST_BADPAD; }
            else if (!lenient && pad2 && pad3 && (dec[c[1]] % 16) != 0) { bad = p + 1; kind = ORACLE_ST_NONCANON; }
            else if (!lenient && !pad2 && pad3 && (dec[c[2]] % 4) != 0) { bad = p + 2; kind = ORACLE_ST_NONCANON; }
            if (kind != ORACLE_ST_OK) {
                *err_off = bad;
                *out_len = 3 * q;
                return kind;
            }
            {
                unsigned a = dec[c[0]], b = dec[c[1]];
                unsigned cc = pad2 ? 0 : dec[c[2]];
                unsigned d = pad3 ? 0 : dec[c[3]];
                int k = pad2 ? 1 : (pad3 ? 2 : 3);
                o[0] = (uint8_t)((a * 4) + (b / 16));
                if (k >= 2) o[1] = (uint8_t)((b * 16) % 256 + (cc / 4));
                if (k >= 3) o[2] = (uint8_t)((cc * 64) % 256 + d);
                *out_len = 3 * q + k;
            }
        }
    }
    if (nq == 0) *out_len = 0;
    return ORACLE_ST_OK;
}

int oracle_decode(const uint8_t *in, int64_t m, uint8_t *out,
                  const uint8_t chars[64], uint8_t pad,
                  int64_t *out_len, int64_t *err_off)
{
    return decode_opt(in, m, out, chars, pad, 0, out_len, err_off);
}

int oracle_decode_lenient(const uint8_t *in, int64_t m, uint8_t *out,
                          const uint8_t chars[64], uint8_t pad,
                          int64_t *out_len, int64_t *err_off)
{
    return decode_opt(in, m, out, chars, pad, 1, out_len, err_off);
}

/* Padding-optional decode (reading R13):
 * the encoded length law of PAPER.md:84-87 without the '=' ("may be
 * appended").  m % 4 == 0: exactly oracle_decode.  m % 4 == 1: LENGTH at
 * m - 1.  m % 4 in {2, 3}: every full quad is interior (all chars in the
 * alphabet), then the last 2 or 3 chars must be alphabet chars and decode to
 * 1 or 2 bytes by the same formulas (missing values taken as zero), with the
 * dropped low bits zero (canonical; NONCANON at m - 1). */
static int decode_unpadded_opt(const uint8_t *in, int64_t m, uint8_t *out,
                               const uint8_t chars[64], uint8_t pad, int lenient,
                               int64_t *out_len, int64_t *err_off)
{
    uint8_t dec[256];
    int64_t q, nq, r, p;
    if (m % 4 == 0) return decode_opt(in, m, out, chars, pad, lenient, out_len, err_off);
    build_decode_table(chars, dec);
    *out_len = 0;
    *err_off = -1;
    r = m % 4;
    if (r == 1) {
        *err_off = m - 1;
        return ORACLE_ST_LENGTH;
    }
    nq = m / 4;
    for (q = 0; q < nq; q++) {
        const uint8_t *c = in + 4 * q;
        int j;
        for (j = 0; j < 4; j++) {
            if (dec[c[j]] == ORACLE_INVALID) {
                *err_off = 4 * q + j;
                *out_len = 3 * q;
                return ORACLE_ST_BADCHAR;
            }
        }
        {
            unsigned a = dec[c[0]], b = dec[c[1]], cc = dec[c[2]], d = dec[c[3]];
            out[3 * q] = (uint8_t)((a * 4) + (b / 16));
            out[3 * q + 1] = (uint8_t)((b * 16) % 256 + (cc / 4));
            out[3 * q + 2] = (uint8_t)((cc * 64) % 256 + d);
        }
    }
    p = 4 * nq;
    for (q = 0; q < r; q++) {
        if (dec[in[p + q]] == ORACLE_INVALID) {
            *err_off = p + q;
            *out_len = 3 * nq;
            return ORACLE_ST_BADCHAR;
        }
    }
    {
        unsigned a = dec[in[p]], b = dec[in[p + 1]], cc = (r == 3) ? dec[in[p + 2]] : 0;
        if (!lenient && ((r == 2 && (b % 16) != 0) || (r == 3 && (cc % 4) != 0))) {
            *err_off = m - 1;
            *out_len = 3 * nq;
            return ORACLE_ST_NONCANON;
        }
        out[3 * nq] = (uint8_t)((a * 4) + (b / 16));
        if (r == 3) out[3 * nq + 1] = (uint8_t)((b * 16) % 256 + (cc / 4));
        *out_len = 3 * nq + (r - 1);
    }
    return ORACLE_ST_OK;
}

int oracle_decode_unpadded(const uint8_t *in, int64_t m, uint8_t *out,
                           const uint8_t chars[64], uint8_t pad,
                           int64_t *out_len, int64_t *err_off)
{
    return decode_unpadded_opt(in, m, out, chars, pad, 0, out_len, err_off);
}

/* Padding-optional AND lenient (R13 + R16): the dropped low bits of a 2/3-char
 * tail (or of the char before '=') may be non-zero. */
int oracle_decode_unpadded_lenient(const uint8_t *in, int64_t m, uint8_t *out,
                                   const uint8_t chars[64], uint8_t pad,
                                   int64_t *out_len, int64_t *err_off)
{
    return decode_unpadded_opt(in, m, out, chars, pad, 1, out_len, err_off);
}

/* Whitespace-skipping decode (reading R14; SURVEY.md Sec. 8(f) f2;
 * the MIME use of PAPER.md:44): the bytes 0x09-0x0D and 0x20 that are not
 * alphabet chars are removed, the remaining text is decoded by oracle_decode,
 * and err_off is mapped back to the position of the offending byte in the
 * ORIGINAL text (for LENGTH: the first char of the incomplete group). */
static int decode_ws_opt(const uint8_t *in, int64_t m, uint8_t *out,
                         const uint8_t chars[64], uint8_t pad, int lenient,
                         int64_t *out_len, int64_t *err_off)
{
    uint8_t skip[256];
    uint8_t *txt;
    int64_t *orig, i, k = 0;
    int v, st;
    memset(skip, 0, sizeof skip);
    for (v = 0x09; v <= 0x0D; v++) skip[v] = 1;
    skip[0x20] = 1;
    for (v = 0; v < 64; v++) skip[chars[v]] = 0;
    txt = (uint8_t *)malloc((size_t)(m > 0 ? m : 1));
    orig = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    for (i = 0; i < m; i++) {
        if (!skip[in[i]]) {
            txt[k] = in[i];
            orig[k] = i;
            k++;
        }
    }
    st = decode_opt(txt, k, out, chars, pad, lenient, out_len, err_off);
    if (*err_off >= 0) *err_off = orig[*err_off];
    free(txt);
    free(orig);
    return st;
}

int oracle_decode_ws(const uint8_t *in, int64_t m, uint8_t *out,
                     const uint8_t chars[64], uint8_t pad,
                     int64_t *out_len, int64_t *err_off)
{
    return decode_ws_opt(in, m, out, chars, pad, 0, out_len, err_off);
}

int oracle_decode_ws_lenient(const uint8_t *in, int64_t m, uint8_t *out,
                             const uint8_t chars[64], uint8_t pad,
                             int64_t *out_len, int64_t *err_off)
{
    return decode_ws_opt(in, m, out, chars, pad, 1, out_len, err_off);
}

/* Batched forms: the single-stream definitions applied string by string over
 * concatenated buffers with int64 offsets[count + 1] (BASELINE.json
 * configs[3]).  Encode output string i starts at out_off[i]. */
void oracle_encode_batch(const uint8_t *in, const int64_t *in_off, int64_t count,
                         uint8_t *out, const int64_t *out_off,
                         const uint8_t chars[64], uint8_t pad)
{
    int64_t i;
    for (i = 0; i < count; i++)
        oracle_encode(in + in_off[i], in_off[i + 1] - in_off[i], out + out_off[i], chars, pad);
}

/* Decode output string i starts at out_off[i]; err_off is relative to the
 * string start, -1 when valid. */
void oracle_decode_batch_opt(const uint8_t *in, const int64_t *in_off, int64_t count,
                             uint8_t *out, const int64_t *out_off,
                             const uint8_t chars[64], uint8_t pad, int lenient,
                             int32_t *status, int64_t *err_off, int64_t *out_len)
{
    int64_t i;
    for (i = 0; i < count; i++)
        status[i] = decode_opt(in + in_off[i], in_off[i + 1] - in_off[i], out + out_off[i],
                               chars, pad, lenient, &out_len[i], &err_off[i]);
}

void oracle_decode_batch(const uint8_t *in, const int64_t *in_off, int64_t count,
                         uint8_t *out, const int64_t *out_off,
                         const uint8_t chars[64], uint8_t pad,
                         int32_t *status, int64_t *err_off, int64_t *out_len)
{
    oracle_decode_batch_opt(in, in_off, count, out, out_off, chars, pad, 0, status, err_off, out_len);
}
