// peer.cu -- one-sided cross-GPU first-error combine over peer memory
// (DESIGN.md "Multi-GPU").
//
// The multi-GPU decode's only exchange is a MIN over ranks of K packed error
// words (pos << 3 | kind).  Instead of an NCCL all_reduce, every rank PUSHES
// its words straight into every rank's buffer over NVLink (peer pointers from
// CUDA IPC) and then reads the world x K words that arrived in its own buffer
// and takes their MIN.  There is no fence, no atomic and no separate arrival
// flag: every word travels as two 64-bit cells {32-bit half, 32-bit epoch
// tag}, and a single aligned 64-bit store is single-copy atomic, so a reader
// polling a cell sees either the old cell or the whole new one -- the tag
// says which (the low-latency protocol NCCL calls LL).  One NVLink one-way
// latency per combine instead of a round trip for a fence plus the arrival.
//
// Per-rank buffer (b64_peer_combine_bytes): two parity slots x kPeerMaxWorld
// ranks x K words x 2 cells.  Epoch e uses slot e & 1 and tag e + 1.  Rank p
// overwrites slot e & 1 of another rank's buffer next in epoch e + 2, which it
// only reaches after epoch e + 1 completed for it -- and that needs this
// rank's words of epoch e + 1, pushed after this rank finished reading epoch
// e.  Tags only grow (mod 2^32; a slot is rewritten every other epoch, so a
// stale tag can never equal the awaited one); the buffer starts zeroed.
#include "b64_device.cuh"

namespace b64 {

constexpr int kPeerMaxWorld = 32;
constexpr unsigned long long kSpinTimeoutNs = 5ull * 1000 * 1000 * 1000;  // 5 s: a peer never arrived

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_relaxed_sys_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void ld_relaxed_sys_v2(const unsigned long long* p, unsigned long long& a,
                                                  unsigned long long& b) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Cell pair of word k from rank p in parity slot `par` of a buffer.
__device__ __forceinline__ unsigned long long* peer_cells(uint8_t* buf, int par, int p, int64_t K, int64_t k) {
    return reinterpret_cast<unsigned long long*>(buf) + ((int64_t(par) * kPeerMaxWorld + p) * K + k) * 2;
}

// One rank's side of epoch `epoch`, executed by one warp.  bufs[p] is rank p's
// buffer (peer-mapped), local[0..K) this rank's words.  Writes the global MIN
// to out[0..K) (packed words; shared or global memory); returns false on
// timeout (a peer's words did not arrive within kSpinTimeoutNs).
__device__ bool peer_min_epoch(uint8_t* const* bufs, int world, int rank, const unsigned long long* local, int64_t K,
                               unsigned long long epoch, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int par = int(epoch & 1);
    const unsigned long long tag = (epoch + 1) << 32;  // low 32 bits of the tag, in the cells' high half
    // 1. push this rank's words into every rank's buffer (own one included)
    for (int64_t i = lane; i < int64_t(world) * K; i += 32) {
        const int p = int(i / K);
        const int64_t k = i - int64_t(p) * K;
        const unsigned long long v = local[k];
        st_relaxed_sys_v2(peer_cells(bufs[p], par, rank, K, k), tag | (v & 0xffffffffull), tag | (v >> 32));
    }
    for (int64_t k = lane; k < K; k += 32) out[k] = ~0ull;
    __syncwarp();
    // 2. wait for every rank's words in the own buffer, MIN per stream
    bool ok = true;
    const unsigned long long t0 = globaltimer_ns();
    for (int64_t i = lane; i < int64_t(world) * K; i += 32) {
        const int p = int(i / K);
        const int64_t k = i - int64_t(p) * K;
        const unsigned long long* c = peer_cells(bufs[rank], par, p, K, k);
        unsigned long long lo, hi;
        for (;;) {
            ld_relaxed_sys_v2(c, lo, hi);
            if ((lo >> 32) == (tag >> 32) && (hi >> 32) == (tag >> 32)) break;
            if (globaltimer_ns() - t0 > kSpinTimeoutNs) { ok = false; break; }
        }
        if (!ok) break;
        atomicMin(out + k, (hi << 32) | (lo & 0xffffffffull));
    }
    ok = __all_sync(kFull, ok);
    __syncwarp();
    return ok;
}

// Per-rank launch (one warp): local packed words -> global MIN -> API form
// (err_off = -1 or position, status) for K streams.  On a timeout (a peer
// never arrived) err_off = -2 and status = -1 for every stream.
__global__ void peer_combine_kernel(uint8_t* const* __restrict__ bufs, int world, int rank,
                                    const unsigned long long* __restrict__ local, int64_t K, unsigned long long epoch,
                                    int64_t* __restrict__ err_off, int32_t* __restrict__ status) {
    griddep_wait();
    extern __shared__ unsigned long long s_out[];
    const bool ok = peer_min_epoch(bufs, world, rank, local, K, epoch, s_out);
    __syncwarp();
    for (int64_t k = threadIdx.x; k < K; k += 32) {
        const unsigned long long wv = s_out[k];
        if (!ok) {
            err_off[k] = -2;
            if (status) status[k] = -1;
        } else if (wv >= kErrNone) {
            err_off[k] = -1;
            if (status) status[k] = kOk;
        } else {
            err_off[k] = int64_t(wv >> 3);
            if (status) status[k] = int32_t(wv & 7);
        }
    }
}

// Single-GPU emulation of `world` ranks (one block = one rank, all blocks
// co-resident: a cooperative launch) running `epochs` combines back to back:
// rank r contributes local[(e * world + r) * K + k] in epoch e and writes the
// MIN it sees to out[(e * world + r) * K + k].  Exercises the slot parity,
// the counters and the resets with real atomics; NVLink is not involved.
__global__ void peer_combine_emulate_kernel(uint8_t* const* __restrict__ bufs, int world,
                                            const unsigned long long* __restrict__ local, int64_t K, int epochs,
                                            unsigned long long* __restrict__ out, int* __restrict__ ok_out) {
    const int rank = blockIdx.x;
    for (int e = 0; e < epochs; ++e) {
        const int64_t o = (int64_t(e) * world + rank) * K;
        const bool ok = peer_min_epoch(bufs, world, rank, local + o, K, (unsigned long long)e, out + o);
        if (!ok && (threadIdx.x & 31) == 0) atomicExch(ok_out, 0);
        if (!ok) return;
    }
}

__global__ void peer_buffer_init_kernel(uint8_t* buf, int64_t K) {
    griddep_wait();
    auto* p = reinterpret_cast<unsigned long long*>(buf);
    const int64_t cells = 2ll * kPeerMaxWorld * K * 2;
    for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) p[i] = 0ull;  // tag 0: no epoch yet
}

}  // namespace b64
