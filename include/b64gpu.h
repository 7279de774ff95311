/*
 * b64gpu.h -- C ABI of the B200-native (sm_100a) base64 codec.
 *
 * Method: W. Mula, D. Lemire, "Base64 encoding and decoding at almost the
 * speed of a memory copy", arXiv 1910.05109 (PAPER.md in the task reference).
 * Citations "PAPER.md:L" are line numbers of that file; "DESIGN.md Rn" are the
 * numbered readings of the paper listed in DESIGN.md.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  - Every pointer named d_* is a DEVICE pointer (cudaMalloc / torch CUDA
 *    storage) on the current device; every other pointer is a host pointer.
 *  - All sizes, offsets and positions are int64_t (streams may exceed 2^32).
 *  - Ownership: the caller allocates and owns every buffer.  The library never
 *    allocates, frees or keeps per-call state and is re-entrant on any stream.
 *  - Ordering: every call only enqueues work on `stream` (0 = legacy default
 *    stream) and returns; results are visible to later work on that stream.
 *  - Return value: synchronous argument / launch errors only (B64_OK or a
 *    negative B64_E* code).  Data errors (invalid base64) are asynchronous and
 *    are written to device memory (err_off / status).
 *  - Input bytes are only read and output bytes only written inside the
 *    ranges stated per call, with one exception: the generic (unaligned /
 *    batched) and whitespace kernels may read whole naturally aligned 16-byte
 *    blocks that contain input bytes, and the unaligned fast decode whole
 *    aligned 32-byte blocks -- at most 15 (31) bytes before the first and
 *    after the last input byte, never a block that holds no input byte.  A
 *    block that holds an input byte lies in the same 256-byte-aligned region
 *    as that byte, and cudaMalloc (and the torch caching allocator) hands out
 *    whole 256-byte-aligned regions, so such reads stay inside the allocation;
 *    a caller passing a sub-allocation must keep the 32-byte blocks that
 *    contain its bytes readable (checked by hardware: tests/test_guard_pages.py
 *    puts every buffer of every entry point against an unmapped page).  The
 *    values read there never affect a result.
 *  - Inputs and outputs must not overlap.
 */
#ifndef B64GPU_H
#define B64GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same type as cudaStream_t (struct CUstream_st*); no CUDA header needed. */
typedef struct CUstream_st *b64_stream_t;

/* ---- status codes ------------------------------------------------------ */
enum {
    B64_OK = 0,
    B64_EINVAL = -1,          /* null pointer with non-zero size, negative size, bad flag */
    B64_ELENGTH = -2,         /* b64_decode*: m % 4 != 0 (nothing launched, nothing written) */
    B64_EALPHA_DUP = -3,      /* alphabet: duplicate character        */
    B64_EALPHA_NONASCII = -4, /* alphabet: character or pad >= 0x80   */
    B64_EALPHA_PAD = -5,      /* alphabet: pad is one of the 64 chars */
    B64_ECUDA = -6            /* a CUDA launch / runtime call failed  */
};

/* per-stream / per-string decode status (asynchronous, device memory) */
enum {
    B64_ST_OK = 0,
    B64_ST_BADCHAR = 1,  /* byte outside the alphabet, or '=' where it may not be  */
    B64_ST_BADPAD = 2,   /* alphabet char after '=' in the final quad              */
    B64_ST_NONCANON = 3, /* non-zero trailing bits in 'xx==' / 'xxx=' (DESIGN R6)  */
    B64_ST_LENGTH = 4    /* batched string with len % 4 != 0                        */
};

/* Packed error word used by the chunk API and the multi-GPU MIN reduction
 * (a deliberate deviation from SURVEY.md Sec. 8(b), whose d_err_min is a plain
 * offset with INT64_MAX = none; R8): the word carries the status kind
 * with the position, so the one all_reduce(MIN) that combines the ranks also
 * yields the kind -- the order of packed words is the order of positions.
 * b64_decode_finalize(_n) maps a word to the plain form (-1 or the offset,
 * plus the kind); tests/test_abi.py pins the packing and its MIN order. */
/* Packed error word layout:
 * (global_position << 3) | status.  Positions are unique, so the MIN over
 * packed words is the first error together with its kind.  B64_ERR_NONE
 * means "no error" (R8); it is the byte 0x7F repeated, so a
 * cudaMemsetAsync(p, 0x7F, 8) initialises a cell, and it exceeds every packed
 * word of a position < 2^59. */
#define B64_ERR_NONE ((int64_t)0x7F7F7F7F7F7F7F7FLL)
#define B64_ERR_POS(w) ((int64_t)(w) >> 3)
#define B64_ERR_KIND(w) ((int)((w)&7))

/* ---- alphabet ----------------------------- */
/* A validated alphabet, passed BY VALUE to the kernels as runtime constants
 * ("adapted -- even at runtime -- to any base64 variant by only changing
 * constants"; "any 64-byte mapping is feasible, even if
 * determined dynamically at runtime").
 *   enc[v]  : the character for 6-bit value v (v < 64).
 *   dec[c]  : the 6-bit value of character c, or 0x80 when c is not one of
 *             the 64 (the paper's sentinel, indexed here by
 *             the full byte instead of its low 7 bits).
 *   pad     : the padding character, '=' for both variants. */
typedef struct b64_alphabet {
    uint8_t enc[64];
    uint8_t dec[256];
    uint8_t pad;
    uint8_t flags;       /* B64_ALPHA_* decode options; 0 after b64_alphabet_init */
    uint8_t reserved[2];
} b64_alphabet;

/* Lenient decode (R16): every strict rule applies except the
 * canonical-bits check -- the low bits of the char before '=' (or of the last
 * char of an unpadded 2/3-char tail) are dropped instead of reported as
 * B64_ST_NONCANON, as Python's binascii strict mode and GNU coreutils do.
 * Honoured by every decode entry point that takes the alphabet. */
#define B64_ALPHA_LENIENT 1u

/* Validate `chars` (64 bytes) + `pad` and fill `*a`.  Rules (R4):
 * 64 distinct bytes < 0x80, pad < 0x80 and not among them.  On failure
 * returns B64_EALPHA_* and sets *bad_index (nullable) to the offending index
 * (64 = the pad); *a is then unspecified.  Host only, O(1). */
int b64_alphabet_init(b64_alphabet *a, const char chars[64], char pad, int *bad_index);

/* Set the decode options of a validated alphabet (B64_ALPHA_* bits; unknown
 * bits -> B64_EINVAL).  Host only. */
int b64_alphabet_set_flags(b64_alphabet *a, unsigned flags);

/* Built-in alphabets (static storage, never freed; strict: flags 0). */
const b64_alphabet *b64_alphabet_standard(void);
const b64_alphabet *b64_alphabet_url(void);

/* ---- sizes ----------------------------------------------------------------- */
int64_t b64_encoded_len(int64_t n);     /* 4*ceil(n/3); -1 if n < 0 */
int64_t b64_decoded_len_max(int64_t m); /* 3*(m/4): capacity a decode output needs   */
/* Capacity b64_decode_unpadded needs: 3*(m/4) plus 1 / 2 bytes for a 2 / 3-char
 * tail (R13); -1 if m < 0 or m % 4 == 1. */
int64_t b64_decoded_len_max_unpadded(int64_t m);

/* ---- single stream --------------------------------------------------------- */
/* Encode n bytes d_in[0..n) to exactly b64_encoded_len(n) chars at d_out, with
 * '=' padding (R5).  No NUL terminator.
 * d_out capacity >= b64_encoded_len(n).  n == 0 is valid and launches nothing. */
int b64_encode(const uint8_t *d_in, int64_t n, uint8_t *d_out, const b64_alphabet *a,
               b64_stream_t stream);

/* Validating decode of m chars (DESIGN.md
 * R5-R8).  m % 4 != 0 returns B64_ELENGTH synchronously.  Asynchronously
 * writes *d_err_off (device int64) = -1 when the text is valid, else the
 * position of the first invalid character.  Output: 3*m/4 - pads bytes at
 * d_out when valid; on error only the bytes of quads before the quad holding
 * err_off are defined.  d_out capacity >= b64_decoded_len_max(m). */
int b64_decode(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a,
               int64_t *d_err_off, b64_stream_t stream);

/* b64_decode plus the status kind and the number of exact output bytes
 * (3*m/4 - pads when valid, else 3*floor(err_off/4)).  d_status and
 * d_out_len are nullable device pointers; d_err_off is required. */
int b64_decode_ex(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a,
                  int64_t *d_err_off, int32_t *d_status, int64_t *d_out_len,
                  b64_stream_t stream);

/* Padding-optional decode (R13; e.g. base64url without '='):
 * m % 4 == 0 behaves exactly as b64_decode_ex; m % 4 == 1 returns B64_ELENGTH
 * synchronously; m % 4 in {2, 3}: all full quads must be alphabet chars and
 * the trailing 2 / 3 chars decode to 1 / 2 bytes with zero dropped bits
 * (B64_ST_NONCANON at m - 1 otherwise).  Outputs as b64_decode_ex; d_out
 * capacity >= b64_decoded_len_max_unpadded(m). */
int b64_decode_unpadded(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a,
                        int64_t *d_err_off, int32_t *d_status, int64_t *d_out_len, b64_stream_t stream);

/* Whitespace-skipping decode (MIME line-wrapped text; R14): the
 * bytes 0x09-0x0D and 0x20 that are not alphabet chars are ignored, the rest
 * is decoded under the strict rules (length and padding rules apply to the
 * text without whitespace); *d_err_off is the position of the offending byte
 * in the ORIGINAL text (for B64_ST_LENGTH: of the first char of the
 * incomplete group).  *d_out_len is 0 for B64_ST_LENGTH (nothing is
 * decoded, as in b64_decode_ex), else the exact prefix as in b64_decode_ex.
 * Needs a device workspace of
 * b64_decode_ws_workspace_bytes(m) bytes (~m + m/1000 + 17 KiB) and d_out
 * 16-byte aligned with capacity 3*(m/4).  Asynchronous on `stream`: texts up
 * to 512 KiB are one cluster launch; larger line-structured text (MIME / PEM)
 * is decoded in one pass; anything else goes through count, scan, compact,
 * decode and finalize kernels. */
int64_t b64_decode_ws_workspace_bytes(int64_t m);
int b64_decode_ws(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a, uint8_t *d_ws,
                  int64_t ws_bytes, int64_t *d_err_off, int32_t *d_status, int64_t *d_out_len, b64_stream_t stream);

/* Shard-aware decode used by the multi-GPU driver.
 * Decodes chars [base_offset, base_offset + m) of a larger stream, m % 4 == 0.
 * Only when is_final_chunk != 0 is the last quad treated as the stream's
 * final quad (padding allowed); otherwise every quad is interior.
 * *d_err_min (device, caller-initialised to B64_ERR_NONE) is lowered with an
 * atomic MIN to the packed word (global_pos << 3 | status) of every error found
 * (at least the first one of this chunk).  *d_out_len (nullable) receives the
 * bytes written assuming the chunk is valid (3*m/4, minus the pads when final). */
int b64_decode_chunk(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a,
                     int64_t base_offset, int is_final_chunk, int64_t *d_err_min,
                     int64_t *d_out_len, b64_stream_t stream);

/* Multi-GPU sharding rule, host
 * only: rank's part of a world-way split of an n-byte encode / m-char decode
 * (m % 4 == 0), cut at multiples of 768 bytes / 1024 chars (one warp-chunk, so
 * every shard keeps the aligned fast path); the last rank also owns the tail
 * (encode: the n mod 3 bytes and the '=' padding; decode: the final quad).
 *   start, stop : the shard's input range
 *   out_start   : where its output begins in the whole stream's output
 *   out_len     : its output length (encode chars; decode capacity 3*len/4)
 *   is_final    : 1 for the rank that owns the tail (pass it to b64_decode_chunk)
 * B64_EINVAL for world < 1, rank outside [0, world), n/m < 0; B64_ELENGTH for
 * m % 4 != 0. */
typedef struct b64_shard {
    int64_t start, stop, out_start, out_len;
    int32_t is_final, reserved;
} b64_shard;
int b64_encode_shard(int64_t n, int world, int rank, b64_shard *sh);
int b64_decode_shard(int64_t m, int world, int rank, b64_shard *sh);

/* Map a packed error word (after any cross-rank MIN) to the API form:
 * *d_err_off = -1 or position, *d_status (nullable) = kind.  One tiny kernel. */
int b64_decode_finalize(const int64_t *d_err_min, int64_t *d_err_off, int32_t *d_status,
                        b64_stream_t stream);

/* ---- grouped launches -------------------------------------------------------- */
/* Several independent streams (each with its own alphabet, input, output and
 * length) processed by one kernel per group of up to 8: the same computation as
 * one b64_encode / b64_decode_chunk per item, with the per-launch fixed cost
 * paid once per group.  Items whose pointers are not fast-path aligned (encode:
 * d_in 8 B, d_out 32 B; decode: d_in 32 B, d_out 16 B) get their own launch.
 * `items` is a host array read during the call only. */
typedef struct b64_encode_item {
    const uint8_t *d_in; /* device, n bytes                         */
    int64_t n;
    uint8_t *d_out;      /* device, b64_encoded_len(n) bytes        */
    const b64_alphabet *a;
} b64_encode_item;

typedef struct b64_decode_item {
    const uint8_t *d_in; /* device, m chars, m % 4 == 0             */
    int64_t m;
    uint8_t *d_out;      /* device, 3*m/4 bytes capacity             */
    const b64_alphabet *a;
    int64_t base_offset; /* as b64_decode_chunk                      */
    int32_t is_final;    /* as b64_decode_chunk                      */
    int32_t reserved;
    int64_t *d_err_min;  /* device packed error word, caller-initialised to B64_ERR_NONE */
} b64_decode_item;

int b64_encode_group(const b64_encode_item *items, int64_t count, b64_stream_t stream);
int b64_decode_group(const b64_decode_item *items, int64_t count, b64_stream_t stream);
/* A mixed job list: n_enc encodes and n_dec decodes, all independent (no item
 * may read another's output).  Up to 8 + 8 items run as ONE kernel whose CTAs
 * take either role (one launch instead of an encode group + a decode group).
 * Same results as b64_encode_group + b64_decode_group; both lists are checked
 * before anything is launched. */
int b64_codec_group(const b64_encode_item *enc, int64_t n_enc, const b64_decode_item *dec, int64_t n_dec,
                    b64_stream_t stream);
/* b64_codec_group with the finalize fused into the kernel: ONE launch, no
 * initialisation and no finalize launch.  Every item must be fast-path aligned
 * (encode d_in 8 B / d_out 32 B, decode d_in 32 B / d_out 16 B), n_enc <= 8,
 * n_dec <= 8 (else B64_EINVAL, nothing launched).  Each decode item's
 * *d_err_min must hold B64_ERR_NONE before the call; d_ticket (device uint32)
 * must be 0.  The last decode CTA to finish (encode CTAs may still be running;
 * with n_dec == 0 one idle decode CTA is launched) writes d_err_off[i] (-1 or the first
 * error position, positions base_offset-relative as b64_decode_chunk) and
 * d_status[i] (nullable) for decode item i, then resets every item's
 * *d_err_min to B64_ERR_NONE and *d_ticket to 0 -- so back-to-back calls need
 * no set-up in between.  (Items sharing one error word get the same result.) */
int b64_codec_group_fused(const b64_encode_item *enc, int64_t n_enc, const b64_decode_item *dec, int64_t n_dec,
                          int64_t *d_err_off, int32_t *d_status, uint32_t *d_ticket, b64_stream_t stream);
/* b64_codec_group_fused for one rank of a multi-GPU job:
 * that last decode CTA also combines the error words with every rank's over
 * peer memory (the b64_peer_combine protocol below: d_peer_bufs / world / rank /
 * epoch exactly as for b64_peer_combine, buffers sized
 * b64_peer_combine_bytes(n_dec)) before it finalises, so d_err_off / d_status
 * hold the GLOBAL first error -- decode, collective and finalize in ONE
 * kernel.  Every rank must make the call with the same n_dec and epoch; on a
 * peer timeout d_err_off[i] = -2, d_status[i] = -1.  d_peer_bufs == NULL is
 * b64_codec_group_fused. */
int b64_codec_group_fused_peer(const b64_encode_item *enc, int64_t n_enc, const b64_decode_item *dec, int64_t n_dec,
                               int64_t *d_err_off, int32_t *d_status, uint32_t *d_ticket, uint8_t *const *d_peer_bufs,
                               int world, int rank, uint64_t epoch, b64_stream_t stream);
/* Single-launch validating decode with a caller-owned, self-resetting context
 * (the fixed-overhead regime of PAPER.md:582, 613):
 * the same results as b64_decode_ex (d_err_off required; d_status, d_out_len
 * nullable) from ONE kernel -- no initialisation and no finalize launch.
 * d_ctx: a device buffer of B64_DECODE_CTX_BYTES bytes, set up once with
 * b64_decode_ctx_init; every call leaves it ready for the next, so calls that
 * share a context must be ordered (the same stream, or events); use one
 * context per stream.  Inputs up to the single-launch cluster size, and
 * inputs that are not fast-path aligned (d_in 32 B, d_out 16 B), take
 * b64_decode_ex's own path (the context is not touched). */
#define B64_DECODE_CTX_BYTES 16
int b64_decode_ctx_init(uint8_t *d_ctx, b64_stream_t stream);
int b64_decode_fused(const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a, int64_t *d_err_off,
                     int32_t *d_status, int64_t *d_out_len, uint8_t *d_ctx, b64_stream_t stream);
/* b64_decode_finalize for `count` consecutive packed words. */
int b64_decode_finalize_n(const int64_t *d_err_min, int64_t count, int64_t *d_err_off, int32_t *d_status,
                          b64_stream_t stream);

/* ---- streaming: input in pieces, carry between calls (R15) ------ */
/* Input arrives in pieces of any length (e.g. network / file reads); the result
 * is exactly the one-shot b64_encode / b64_decode_ex of the concatenation, with
 * error positions in its coordinates.  Whole triples / quads are coded as soon
 * as they are complete; the bytes of an incomplete group are held in d_carry
 * (device, >= 8 bytes, caller-owned, used only by this stream).  Decode always
 * holds back the last 1-4 chars, so the stream's final quad (the only place
 * '=' may appear, R6) is decoded by the end call.  The host struct
 * carries only lengths: no call waits for the device.  Every call of one
 * stream must use the same alphabet and the same CUDA stream (or be ordered by
 * the caller); pieces may be reused / freed once the work queued by the call
 * has run.  Calls on a finished stream (or the wrong kind) return B64_EINVAL. */
typedef struct b64_stream {
    int64_t consumed;   /* input bytes (encode) / chars (decode) accepted so far */
    int64_t produced;   /* output bytes written so far                           */
    int32_t held;       /* bytes (0-2) / chars (0-4) currently held in d_carry    */
    int32_t state;      /* internal: 1 encoding, 2 decoding, 3 finished           */
    uint8_t *d_carry;   /* device carry buffer (>= 8 bytes)                       */
    int64_t *d_err_min; /* decode: device packed error word of the stream         */
} b64_stream;
#define B64_STREAM_OVERLAP 1u /* b64_{encode,decode}_stream_begin_ex flag: overlapped pieces (below) */

/* Output sizes, host-side (no device access): b64_stream_update_len = the
 * chars (encode: 4*floor((held + len)/3)) / bytes (decode: 3*floor((held +
 * len - 1)/4)) the next update with a piece of `len` writes; b64_stream_end_len
 * = the capacity the end call needs (encode 4 or 0, decode 3 or 0).  -1 for a
 * finished stream or len < 0. */
int64_t b64_stream_update_len(const b64_stream *st, int64_t len);
int64_t b64_stream_end_len(const b64_stream *st);

int b64_encode_stream_begin(b64_stream *st, uint8_t *d_carry);
/* b64_encode_stream_begin with flags (0: the same, no device work).  B64_STREAM_OVERLAP
 * (defined with b64_decode_stream_begin_ex below; same contract): d_carry is zeroed on
 * `stream` (8 bytes) as the ordering point, and from the second piece on each update of at
 * least 64 Ki bytes runs its bulk while the previous piece's kernel drains, with the join
 * (straddling triple, new carry) at the kernel's end after the wait -- ONE launch per piece.
 * Every later call of the stream must use the same `stream`.  Unknown flags -> B64_EINVAL. */
int b64_encode_stream_begin_ex(b64_stream *st, uint8_t *d_carry, uint32_t flags, b64_stream_t stream);
/* Encode piece d_in[0..n): writes *n_out = 4*floor((held + n)/3) chars at d_out
 * (capacity >= that; *n_out is known on return, host-side). */
int b64_encode_stream_update(b64_stream *st, const uint8_t *d_in, int64_t n, uint8_t *d_out, const b64_alphabet *a,
                             int64_t *n_out, b64_stream_t stream);
/* Finish: the 1-2 held bytes -> 4 chars with '=' padding at d_out (*n_out = 4),
 * or nothing (*n_out = 0).  Total output = b64_encoded_len(consumed). */
int b64_encode_stream_end(b64_stream *st, uint8_t *d_out, const b64_alphabet *a, int64_t *n_out,
                          b64_stream_t stream);

/* Decode: d_err_min (device int64) is set to B64_ERR_NONE on `stream` and
 * lowered by every later call (packed global position << 3 | status). */
int b64_decode_stream_begin(b64_stream *st, uint8_t *d_carry, int64_t *d_err_min, b64_stream_t stream);
/* b64_decode_stream_begin with flags (0 = b64_decode_stream_begin).
 * B64_STREAM_OVERLAP: from the second piece on, each update's bulk kernel starts
 * while the previous piece's kernel is still draining (its bulk loads and stores
 * run before the programmatic-dependency wait; the join with the held chars, the
 * error word and the carry still wait).  Measured: 1 GiB in 64 MiB pieces 0.51 ->
 * 0.39 ms (R15).  The caller guarantees, for the whole stream: every
 * piece's input is written before the begin call is enqueued (e.g. the text is
 * resident, as for windows over a decoded region); nothing else is enqueued on
 * `stream` between the begin and end calls that writes any piece's input or
 * output; no piece's input overlaps any piece's output.  Results, as without
 * the flag, are complete once later work on the stream runs.  Unknown flag bits
 * -> B64_EINVAL. */
int b64_decode_stream_begin_ex(b64_stream *st, uint8_t *d_carry, int64_t *d_err_min, uint32_t flags,
                               b64_stream_t stream);
/* Decode piece d_in[0..m) (any m >= 0): writes *n_out = 3*Q bytes at d_out,
 * Q = floor((held + m - 1)/4) interior quads (capacity >= *n_out). */
int b64_decode_stream_update(b64_stream *st, const uint8_t *d_in, int64_t m, uint8_t *d_out, const b64_alphabet *a,
                             int64_t *n_out, b64_stream_t stream);
/* Finish: total = consumed chars.  total % 4 != 0 -> status B64_ST_LENGTH at
 * total - total % 4 (as b64_decode_batch); else the held final quad -> 1-3
 * bytes at d_out (capacity >= 3, *n_out = 3 = the most it may write).  Then
 * *d_err_off / *d_status / *d_out_len (device; the last two nullable) exactly
 * as b64_decode_ex for the whole concatenated text (*d_out_len = 0 for
 * B64_ST_LENGTH). */
int b64_decode_stream_end(b64_stream *st, uint8_t *d_out, const b64_alphabet *a, int64_t *d_err_off,
                          int32_t *d_status, int64_t *d_out_len, int64_t *n_out, b64_stream_t stream);

/* ---- one-sided cross-GPU error combine ------------ */
/* The multi-GPU decode's only exchange -- the MIN over ranks of `count` packed
 * error words -- done by ONE small kernel over peer memory instead of an NCCL
 * all_reduce: each rank stores its words into every rank's buffer (system
 * scope, over NVLink) as 64-bit cells tagged with the epoch, then polls its
 * own buffer until every rank's cells of the epoch are there and takes their
 * MIN -- no fence, no atomics.
 *   - Every rank owns one buffer of b64_peer_combine_bytes(count) bytes, set
 *     up once with b64_peer_combine_init, then mapped into every other rank
 *     (CUDA IPC); d_bufs is a DEVICE array of `world` device pointers, d_bufs[p]
 *     = rank p's buffer as seen by the caller.  All ranks must have initialised
 *     their buffers before any rank's first combine (e.g. a host barrier).
 *   - epoch = number of combines this group already did (0, 1, 2, ... the same
 *     sequence on every rank); one combine per epoch per rank.
 *   - Output as b64_decode_finalize_n: d_err_off[k] = -1 or the global first
 *     error position, d_status[k] (nullable) its kind.  If a peer does not
 *     arrive within 5 s the kernel gives up: d_err_off[k] = -2, d_status = -1.
 *   - count <= 4096, world <= 32. */
int64_t b64_peer_combine_bytes(int64_t count);
int b64_peer_combine_init(uint8_t *d_buf, int64_t count, b64_stream_t stream);
int b64_peer_combine(uint8_t *const *d_bufs, int world, int rank, const int64_t *d_local, int64_t count,
                     uint64_t epoch, int64_t *d_err_off, int32_t *d_status, b64_stream_t stream);
/* Buffer plumbing for the combine (the one place the library allocates: an IPC
 * handle needs a cudaMalloc base address).  b64_peer_buffer_alloc: cudaMalloc
 * `bytes` on the current device and export its 64-byte IPC handle;
 * b64_peer_buffer_open: map a peer's buffer from its handle (another process,
 * peer access enabled); b64_peer_buffer_release: cudaFree (opened = 0) or
 * close the mapping (opened = 1). */
int b64_peer_buffer_alloc(int64_t bytes, uint8_t **d_buf, uint8_t handle[64]);
int b64_peer_buffer_open(const uint8_t handle[64], uint8_t **d_buf);
int b64_peer_buffer_release(uint8_t *d_buf, int opened);
/* Test hook: `world` ranks emulated on ONE GPU by one cooperative kernel (block
 * r = rank r; d_bufs = the world buffers on this device) running `epochs`
 * combines: rank r contributes d_local[(e*world + r)*count + k] in epoch e and
 * writes the MIN it sees to d_out[(e*world + r)*count + k] (packed words);
 * *d_ok (device int, caller sets 1) becomes 0 on a timeout. */
int b64_peer_combine_emulate(uint8_t *const *d_bufs, int world, const int64_t *d_local, int64_t count, int epochs,
                             int64_t *d_out, int *d_ok, b64_stream_t stream);

/* ---- host buffers, overlapped (SURVEY.md Sec. 8(f) f3 ingest pipeline) ------ */
/* Encode / decode HOST buffers (h_*: host pointers, pinned for the copies to be
 * asynchronous) through a caller-owned DEVICE workspace d_ws of ws_bytes.  The
 * stream is cut into chunks that rotate through 3 device buffers: chunk j is
 * copied H2D on s_h2d, coded on s_comp, copied D2H on s_d2h, so both PCIe
 * directions and the kernels overlap.  Results are complete once all three
 * streams have been synchronised (they may be the same stream).  A call's
 * first copy waits for the work already queued on s_comp and s_d2h, so
 * back-to-back calls may share one workspace and stream triple.
 * b64_host_workspace_bytes(c) = workspace for encode chunks of ~c input bytes
 * (decode with the same workspace uses chunks of ~4c/3 chars).
 * Encode writes b64_encoded_len(n) chars to h_out.  Decode writes up to 3*m/4
 * bytes to h_out and, on s_comp, *d_err_off (device) = -1 or the first invalid
 * position, *d_status (nullable, device) = its kind and *d_out_len (nullable,
 * device) = the exact output length: 3*m/4 - (number of '=' at m-2, m-1) when
 * valid, 3*floor(err/4) otherwise (same rules as b64_decode_ex), computed on
 * the device from the final chunk. */
int64_t b64_host_workspace_bytes(int64_t chunk_bytes);
int b64_encode_host(const uint8_t *h_in, int64_t n, uint8_t *h_out, const b64_alphabet *a, uint8_t *d_ws,
                    int64_t ws_bytes, b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h);
int b64_decode_host(const uint8_t *h_in, int64_t m, uint8_t *h_out, const b64_alphabet *a, uint8_t *d_ws,
                    int64_t ws_bytes, int64_t *d_err_off, int32_t *d_status, int64_t *d_out_len,
                    b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h);
/* The same with flags.  B64_HOST_CALLER_ORDERED: the caller guarantees that
 * no earlier work still uses d_ws (e.g. it alternates two workspaces and makes
 * s_h2d wait for the end of the call before last that used this one), so the
 * call does not wait for the work already queued on s_comp / s_d2h -- back-to-
 * back calls then overlap (one call's last chunks with the next call's first
 * copies: both PCIe directions stay busy across calls). */
#define B64_HOST_CALLER_ORDERED 1u
int b64_encode_host_ex(const uint8_t *h_in, int64_t n, uint8_t *h_out, const b64_alphabet *a, uint8_t *d_ws,
                       int64_t ws_bytes, b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h,
                       unsigned flags);
int b64_decode_host_ex(const uint8_t *h_in, int64_t m, uint8_t *h_out, const b64_alphabet *a, uint8_t *d_ws,
                       int64_t ws_bytes, int64_t *d_err_off, int32_t *d_status, int64_t *d_out_len,
                       b64_stream_t s_h2d, b64_stream_t s_comp, b64_stream_t s_d2h, unsigned flags);

/* ---- decode -> consumer through an L2-resident ring ---- */
/* "process large files in small parts that fit in cache" (the simdjson hand-off,
 * PAPER.md:642): the text d_in[0..m) (m % 4 == 0, else B64_ELENGTH) is decoded in chunks of C
 * chars into the caller's device ring d_ring (ring_bytes, 16-byte aligned; C =
 * b64_consume_chunk_chars(ring_bytes), a multiple of 4096) and after each chunk `consumer` is
 * called on the host with the chunk's decoded bytes (d_chunk = d_ring, len = 3*C/4 bytes or
 * fewer for the last chunk, out_offset = their offset in the whole output) and `stream`: it
 * enqueues its own work on `stream`, which then reads the bytes while they are still in L2,
 * before the next chunk's decode overwrites the ring -- the decoded text never makes the HBM
 * round trip.  All work is queued on `stream`; the call returns when every chunk has been
 * handed over (not when the device finished).  Results as b64_decode_ex: *d_err_off (device,
 * required) = -1 or the first invalid position, *d_status / *d_out_len (nullable); the last
 * chunk's exact length is *d_out_len - its out_offset.  Bytes of quads at or after the first
 * error are unspecified (the consumer still sees every chunk).  Every chunk costs one decode
 * launch plus the consumer's launches, so the ring should be as large as L2 allows: measured
 * on 1 GiB with a 3-launch checksum consumer, 16 MiB 1.27 ms, 32 MiB 0.88, 64 MiB 0.67, 96 MiB
 * 0.60 -- against 0.46 ms for decode-to-HBM then the same checksum (tools/consume_probe.py): a
 * consumer this light gains less from L2 than the extra launches cost. */
typedef void (*b64_consumer_fn)(const uint8_t *d_chunk, int64_t len, int64_t out_offset, void *user,
                                b64_stream_t stream);
int64_t b64_consume_chunk_chars(int64_t ring_bytes);
int b64_decode_consume(const uint8_t *d_in, int64_t m, uint8_t *d_ring, int64_t ring_bytes, const b64_alphabet *a,
                       b64_consumer_fn consumer, void *user, int64_t *d_err_off, int32_t *d_status,
                       int64_t *d_out_len, b64_stream_t stream);

/* ---- batched (BASELINE.json configs[3]) ------------------------------------ */
/* (d_in / d_out must be valid device pointers when count > 0, even if every
 * string is empty -- the library cannot see the total length without reading
 * the device offsets.)
 * `count` independent strings concatenated in d_in; string i is
 * d_in[d_in_off[i] .. d_in_off[i+1]) (d_in_off: device int64[count+1],
 * non-decreasing, d_in_off[0] >= 0).  Output string i is written at
 * d_out + d_out_off[i] (device int64[count], caller-computed):
 *   encode: d_out_off = exclusive scan of 4*ceil(len_i/3); each string padded.
 *   decode: d_out_off = exclusive scan of 3*(len_i/4).                        */
/* The output offsets the batch calls expect, computed on `stream` from the
 * device offsets d_in_off[count+1] (no host access): d_out_off[count+1]
 * (device) = exclusive scan of 4*ceil(len_i/3) (encode) or of
 * 3*floor(len_i/4) (decode capacity), d_out_off[0] = 0 and d_out_off[count] =
 * the total output.  Three small kernels (a tile-sum / tile-scan / fill scan
 * that uses d_out_off itself as its scratch; no workspace). */
int b64_encode_batch_offsets(const int64_t *d_in_off, int64_t count, int64_t *d_out_off, b64_stream_t stream);
int b64_decode_batch_offsets(const int64_t *d_in_off, int64_t count, int64_t *d_out_off, b64_stream_t stream);

int b64_encode_batch(const uint8_t *d_in, const int64_t *d_in_off, int64_t count,
                     uint8_t *d_out, const int64_t *d_out_off, const b64_alphabet *a,
                     b64_stream_t stream);

/* Per string i (all device arrays of length count; d_err_off required, the
 * other two nullable): d_status[i] (B64_ST_*), d_err_off[i] = -1 or the first
 * invalid position RELATIVE to the string start (len - len%4 for
 * B64_ST_LENGTH), d_out_len[i] = exact output bytes (as b64_decode_ex). */
int b64_decode_batch(const uint8_t *d_in, const int64_t *d_in_off, int64_t count,
                     uint8_t *d_out, const int64_t *d_out_off, const b64_alphabet *a,
                     int32_t *d_status, int64_t *d_err_off, int64_t *d_out_len,
                     b64_stream_t stream);
/* b64_decode_batch that also lowers *d_first_bad (device int64, nullable,
 * caller-initialised, e.g. to B64_ERR_NONE) to the index of the batch's first
 * failing string, counted from index_base (>= 0): MIN over i with
 * d_status[i] != B64_ST_OK of index_base + i, taken inside the finalize kernel
 * (no extra launch).  A multi-GPU batch sharded by cumulative bytes (DESIGN.md
 * "Multi-GPU") passes its first string's global index and
 * all_reduce(MIN)s the word to get the global first failing string. */
int b64_decode_batch_ex(const uint8_t *d_in, const int64_t *d_in_off, int64_t count,
                        uint8_t *d_out, const int64_t *d_out_off, const b64_alphabet *a,
                        int32_t *d_status, int64_t *d_err_off, int64_t *d_out_len,
                        int64_t index_base, int64_t *d_first_bad, b64_stream_t stream);

/* b64_decode_batch_ex with a caller-owned context that enables the
 * concatenation path: when every string length is
 * a multiple of 4, d_out_off[i] - d_out_off[0] = 3*(d_in_off[i] - d_in_off[0])/4
 * (the b64_decode_batch_offsets layout), d_in + d_in_off[0] is 32-byte and
 * d_out + d_out_off[0] 16-byte aligned, the bulk of the batch is decoded as
 * ONE stream (the single-stream fast kernel over the concatenated text) and
 * only the strings' final quads get a per-string pass; otherwise -- or when a
 * '=' sits anywhere but the last two chars of its string -- the per-string
 * kernel of b64_decode_batch_ex runs.  The results (d_status, d_err_off,
 * d_out_len, d_first_bad, and the bytes up to each string's out_len) are
 * those of b64_decode_batch_ex; the bytes of a string's slot after its
 * out_len may be overwritten.  The eligibility is decided on the device (no
 * host sync).  d_ctx: B64_BATCH_CTX_BYTES of device memory set up once with
 * b64_batch_ctx_init; every call leaves it ready for the next, so calls that
 * share a context must be ordered (one context per stream).  d_ctx == NULL is
 * b64_decode_batch_ex.  Five launches (the per-string kernel returns at once
 * when the concatenation path did the work). */
#define B64_BATCH_CTX_BYTES 32
int b64_batch_ctx_init(uint8_t *d_ctx, b64_stream_t stream);
int b64_decode_batch_fast(const uint8_t *d_in, const int64_t *d_in_off, int64_t count,
                          uint8_t *d_out, const int64_t *d_out_off, const b64_alphabet *a,
                          int32_t *d_status, int64_t *d_err_off, int64_t *d_out_len,
                          int64_t index_base, int64_t *d_first_bad, uint8_t *d_ctx, b64_stream_t stream);

/* ---- introspection ---------------------------------------------------------- */
/* Number of kernels the library launched on this process so far (all calls),
 * counted on the host at each launch -- used by bench.py's gpu_launches. */
int64_t b64_launch_count(void);
/* Static description of the build ("sm_100a ..."). */
const char *b64_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* B64GPU_H */
