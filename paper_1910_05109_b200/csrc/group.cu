// group.cu -- grouped launches: up to kGroupMax independent streams (each with
// its own alphabet, length, input and output) encoded or decoded by ONE kernel.
//
// A launch has a fixed cost (~3-4 us on B200: CTA launch, first DRAM latency,
// tail) that a 64 MiB op (~25 us of HBM time) does not amortise; one grid whose
// warps are partitioned among several streams pays it once (DESIGN.md "Grouped
// launches").  Per stream the work is exactly the single-stream kernels'
// (enc_fast_kernel / dec_fast_kernel): the same bulk loop (EncBulk / DecBulk),
// warp-chunk split, tail / final-quad / error handling.
#include "b64_device.cuh"

namespace b64 {

constexpr int kGroupMax = 8;

struct EncGroup {
    const uint8_t* in[kGroupMax];
    uint8_t* out[kGroupMax];
    int64_t n[kGroupMax];
    int64_t cstart[kGroupMax + 1];  // exclusive scan of warp-chunks per stream (only differences are used)
    int32_t wstart[kGroupMax + 1];  // warps [wstart[i], wstart[i+1]) own stream i's chunks
    uint32_t pad[kGroupMax];
    uint32_t lut[kGroupMax][16];    // enc[64] per stream
    int count;
};

struct DecGroup {
    const uint8_t* in[kGroupMax];
    uint8_t* out[kGroupMax];
    int64_t m[kGroupMax];
    int64_t base[kGroupMax];
    unsigned long long* cell[kGroupMax];
    int64_t cstart[kGroupMax + 1];
    int32_t wstart[kGroupMax + 1];
    int32_t is_final[kGroupMax];
    uint32_t pad[kGroupMax];
    uint32_t lenient[kGroupMax];    // DESIGN.md R16
    uint32_t lut[kGroupMax][64];    // dec[256] per stream
    int count;
};

// ---------------------------------------------------------------- warp-partitioned groups
// Each stream gets its own contiguous set of warps, sized by the host so the
// per-warp chunk counts are as even as the resident grid allows
// (group_partition in capi.cu); a warp finds its stream once and then runs
// exactly the single-stream bulk loop (EncBulk / DecBulk) over that stream with
// the stream's warp count as the stride.  No per-chunk stream bookkeeping: the
// per-chunk instruction count is the single-stream kernels'.  The streams are
// swept concurrently, each as one contiguous window.

template <typename G>
__device__ __forceinline__ int warp_stream(const G& g, int32_t w) {
    int it = 0;
    while (it < g.count && w >= g.wstart[it + 1]) ++it;
    return it;  // == g.count: an idle warp (no bulk work)
}

// The grouped encode as run by CTA `bid` of `nblocks` (a whole enc_group_kernel
// grid, or the encode CTAs of a codec_group_kernel grid).
template <int D>
__device__ __forceinline__ void enc_group_body(const EncGroup& g, int64_t bid, int64_t nblocks) {
    __shared__ __align__(64) uint32_t s_lut[kGroupMax][16];
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = bid * blockDim.x + threadIdx.x;
    const int64_t gthreads = nblocks * blockDim.x;
    const int32_t w = int32_t(gtid >> 5);
    const int it = warp_stream(g, w);

    griddep_wait();
    EncBulk<D> bulk;
    if (it < g.count) {
        bulk.prime(g.in[it], g.out[it], w - g.wstart[it], int32_t(g.cstart[it + 1] - g.cstart[it]),
                   g.wstart[it + 1] - g.wstart[it], lane);
    }
    if (threadIdx.x < g.count * 16) (&s_lut[0][0])[threadIdx.x] = (&g.lut[0][0])[threadIdx.x];
    __syncthreads();
    if (it < g.count) bulk.run(smem_u32(&s_lut[it][0]));

    // per-stream remainder quads (whole triples + the padded tail), one per thread
    for (int is = 0; is < g.count; ++is) {
        const int64_t n = g.n[is];
        const int64_t T = n / 3, Q = (n + 2) / 3;
        const uint8_t* in = g.in[is];
        const uint8_t* lut = reinterpret_cast<const uint8_t*>(&s_lut[is][0]);
        for (int64_t q = (g.cstart[is + 1] - g.cstart[is]) * 256 + gtid; q < Q; q += gthreads) {
            const uint8_t* s = in + 3 * q;
            uint32_t word;
            if (q < T) {
                word = enc_triple((uint32_t(s[0]) << 24) | (uint32_t(s[1]) << 16) | (uint32_t(s[2]) << 8), lut);
            } else {
                const int r = int(n - 3 * q);
                word = enc_partial(s[0], r == 2 ? s[1] : 0u, r, lut, g.pad[is]);
            }
            *reinterpret_cast<uint32_t*>(g.out[is] + 4 * q) = word;
        }
    }
}

// The grouped decode as run by CTA `bid` of `nblocks`.
template <int D>
__device__ __forceinline__ void dec_group_body(const DecGroup& g, int64_t bid, int64_t nblocks) {
    __shared__ __align__(256) uint32_t s_lut[kGroupMax][64];
    __shared__ __align__(128) uint32_t s_stage[kThreads / 32][768 / 4];
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = bid * blockDim.x + threadIdx.x;
    const int64_t gthreads = nblocks * blockDim.x;
    const int32_t w = int32_t(gtid >> 5);
    const int it = warp_stream(g, w);

    griddep_wait();
    DecBulk<D> bulk;
    if (it < g.count) {
        bulk.prime(g.in[it], g.out[it], w - g.wstart[it], int32_t(g.cstart[it + 1] - g.cstart[it]),
                   g.wstart[it + 1] - g.wstart[it], lane, g.pad[it] >> 8);  // pad < 0x80
    }
    for (int t = threadIdx.x; t < g.count * 64; t += blockDim.x) (&s_lut[0][0])[t] = (&g.lut[0][0])[t];
    __syncthreads();
    if (it < g.count) {
        bulk.run(smem_u32(&s_lut[it][0]), reinterpret_cast<const uint8_t*>(&s_lut[it][0]),
                 smem_u32(&s_stage[threadIdx.x >> 5][0]), lane, g.base[it], g.cell[it]);
    }

    // per-stream leftover interior quads, then the final quad (grid's last thread)
    for (int is = 0; is < g.count; ++is) {
        const uint8_t* lut = reinterpret_cast<const uint8_t*>(&s_lut[is][0]);
        const int64_t Q = g.m[is] >> 2;
        const int64_t Qint = (g.is_final[is] && Q > 0) ? Q - 1 : Q;
        const uint8_t* in = g.in[is];
        uint8_t* out = g.out[is];
        for (int64_t q = (g.cstart[is + 1] - g.cstart[is]) * 256 + gtid; q < Qint; q += gthreads) {
            const uint32_t x = ld32(in + 4 * q);
            uint32_t err = 0;
            const uint32_t v = dec_quad(x, lut, err);
            store_bytes(out + 3 * q, v, 3);
            if (err & kInvalid)
                atomicMin(g.cell[is], pack_err(g.base[is] + 4 * q + first_bad_in_quad(x, lut), kBadChar));
        }
        if (gtid == gthreads - 1 && g.is_final[is] && Q > 0) {
            const int64_t q = Q - 1;
            int bad, k;
            uint32_t v;
            const uint32_t kind = final_quad(ld32(in + 4 * q), lut, g.pad[is], g.lenient[is], &bad, &k, &v);
            if (kind == kOk) store_bytes(out + 3 * q, v, k);
            else atomicMin(g.cell[is], pack_err(g.base[is] + 4 * q + bad, kind));
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads, kBulkCtasPerSm) enc_group_kernel(const __grid_constant__ EncGroup g) {
    enc_group_body<D>(g, blockIdx.x, gridDim.x);
}

template <int D>
__global__ void __launch_bounds__(kThreads, kBulkCtasPerSm) dec_group_kernel(const __grid_constant__ DecGroup g) {
    dec_group_body<D>(g, blockIdx.x, gridDim.x);
}

// Mixed job list in ONE launch: CTAs [0, dec_blocks) run the grouped decode,
// the rest the grouped encode (each CTA one role, so each role's code, table
// staging and barrier are exactly the single-role kernel's).  Saves one kernel
// boundary (launch, ramp, drain) per encode + decode pair of groups.
struct CodecGroup {
    DecGroup d;
    EncGroup e;
    int64_t dec_blocks;
    // Fused finalize (b64_codec_group_fused; ticket == nullptr: none).  The last DECODE CTA
    // to finish (dec_blocks >= 1 whenever a ticket is given) maps every decode stream's error word to (err_off, status) at index didx[k]
    // and resets the word to kErrNone and the ticket to 0, so the next call needs no
    // initialisation launch and no finalize launch.
    unsigned int* ticket;
    int64_t* err_off;
    int64_t* out_len;  // nullable: exact output bytes per decode item (as b64_decode_ex)
    int32_t* status;
    int32_t didx[kGroupMax];
    // Fused cross-rank MIN (b64_codec_group_fused_peer; peer_bufs == nullptr: none): the last
    // CTA combines the error words with every rank's over peer memory (peer.cu) before it
    // finalises -- the decode, the collective and the finalize in ONE kernel.
    uint8_t* const* peer_bufs;
    int32_t world, rank;
    unsigned long long epoch;
};

// "Last block" epilogue of the fused finalize (the classic threadfence reduction):
// every thread fences its own writes (outputs, error-word atomics), the CTA barriers,
// one thread takes a ticket; the CTA holding the last ticket sees every other CTA's
// writes and finalises.
__device__ __forceinline__ void codec_fused_finalize(const CodecGroup& g) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(g.ticket, 1u) == unsigned(g.dec_blocks) - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ unsigned long long s_w[kGroupMax], s_g[kGroupMax];
    __shared__ bool s_ok;
    const int k = threadIdx.x;
    if (k < g.d.count) s_w[k] = atomicMax(g.d.cell[k], 0ull);  // atomic read (L2), never stale
    if (k == 0) s_ok = true;
    __syncthreads();
    if (g.peer_bufs) {  // one warp: MIN with every rank's words over peer memory
        if (k < 32) {
            const bool ok = peer_min_epoch(g.peer_bufs, g.world, g.rank, s_w, g.d.count, g.epoch, s_g);
            if (k == 0) s_ok = ok;
        }
    } else if (k < g.d.count) {
        s_g[k] = s_w[k];
    }
    __syncthreads();
    if (k < g.d.count) {
        const unsigned long long wv = s_g[k];
        if (!s_ok) {  // a peer never arrived (peer.cu timeout)
            g.err_off[g.didx[k]] = -2;
            if (g.status) g.status[g.didx[k]] = -1;
            if (g.out_len) g.out_len[g.didx[k]] = 0;
        } else if (wv >= kErrNone) {
            g.err_off[g.didx[k]] = -1;
            if (g.status) g.status[g.didx[k]] = kOk;
            if (g.out_len) {
                const int64_t m = g.d.m[k];
                const uint32_t pad = g.d.pad[k] & 0xffu;
                int64_t ol = 3 * (m >> 2);
                if (g.d.is_final[k] && m >= 4) ol -= (g.d.in[k][m - 2] == pad) ? 2 : (g.d.in[k][m - 1] == pad ? 1 : 0);
                g.out_len[g.didx[k]] = ol;
            }
        } else {
            g.err_off[g.didx[k]] = int64_t(wv >> 3);
            if (g.status) g.status[g.didx[k]] = int32_t(wv & 7);
            if (g.out_len) {
                const int64_t rel = int64_t(wv >> 3) - g.d.base[k];
                g.out_len[g.didx[k]] = rel > 0 ? 3 * (rel >> 2) : 0;
            }
        }
    }
    __syncthreads();  // every word read before any (possibly shared) word is reset
    if (k < g.d.count) *g.d.cell[k] = kErrNone;
    if (k == 0) *g.ticket = 0u;
}

template <int D>
__global__ void __launch_bounds__(kThreads, kBulkCtasPerSm) codec_group_kernel(const __grid_constant__ CodecGroup g) {
    const int64_t b = blockIdx.x;
    if (b < g.dec_blocks) {
        dec_group_body<D>(g.d, b, g.dec_blocks);
        // only the decode CTAs take a ticket: the last of them finalises (and, multi-GPU, meets
        // the other ranks) while encode CTAs may still be running, off the kernel's tail
        if (g.ticket) codec_fused_finalize(g);
    } else {
        enc_group_body<D>(g.e, b - g.dec_blocks, int64_t(gridDim.x) - g.dec_blocks);
    }
}

// Packed error words -> (err_off, status) for count streams.
__global__ void dec_finalize_n_kernel(const int64_t* cells, int64_t count, int64_t* err_off, int32_t* status) {
    griddep_wait();
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long wv = static_cast<unsigned long long>(cells[i]);
        if (wv >= kErrNone) {
            err_off[i] = -1;
            if (status) status[i] = kOk;
        } else {
            err_off[i] = int64_t(wv >> 3);
            if (status) status[i] = int32_t(wv & 7);
        }
    }
}

}  // namespace b64
