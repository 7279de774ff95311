// peer.cu -- one-sided cross-GPU first-error combine over peer memory
// (DESIGN.md "Multi-GPU").
//
// The multi-GPU decode's only exchange is a MIN over ranks of K packed error
// words (pos << 3 | kind).  Instead of an NCCL all_reduce, every rank writes
// its words straight into every rank's buffer with system-scope atomicMin
// over NVLink (peer pointers from CUDA IPC), then signals arrival on every
// rank's counter; a rank whose counter shows all arrivals of this epoch holds
// the global MIN in its own buffer.  One tiny kernel, no NCCL launch.
//
// Per-rank buffer (b64_peer_combine_bytes): two slots of K words + an arrival
// counter.  Epoch e uses slot e & 1; after reading its slot a rank resets it
// for epoch e + 2.  Safe because a peer can only write that slot in epoch
// e + 2 after passing the barrier of epoch e + 1, which needs this rank's
// arrival in e + 1, issued after the reset.  Counters only grow (epoch e is
// complete when the counter reaches (e + 1) * world).
#include "b64_device.cuh"

namespace b64 {

constexpr int64_t kPeerCounterOff = 0;  // uint64 arrival counter, then the two slots (64-byte aligned)
constexpr int64_t kPeerSlotsOff = 64;
constexpr unsigned long long kSpinTimeoutNs = 5ull * 1000 * 1000 * 1000;  // 5 s: a peer never arrived

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// One rank's side of epoch `epoch`, executed by one warp.  bufs[p] is rank p's
// buffer (peer-mapped), local[0..K) this rank's words.  Writes the global MIN
// to out[0..K) (packed words); returns false on timeout.
__device__ bool peer_min_epoch(uint8_t* const* bufs, int world, int rank, const unsigned long long* local, int64_t K,
                               unsigned long long epoch, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int64_t slot = int64_t(epoch & 1) * K;
    // 1. contribute to every rank's slot (system-scope atomics over NVLink)
    for (int64_t i = lane; i < int64_t(world) * K; i += 32) {
        const int p = int(i / K);
        const int64_t k = i - int64_t(p) * K;
        auto* cells = reinterpret_cast<unsigned long long*>(bufs[p] + kPeerSlotsOff);
        atomicMin_system(cells + slot + k, local[k]);
    }
    __threadfence_system();
    __syncwarp();
    // 2. arrive on every rank's counter
    if (lane < world) atomicAdd_system(reinterpret_cast<unsigned long long*>(bufs[lane] + kPeerCounterOff), 1ull);
    // 3. wait for all arrivals of this epoch on the own counter
    const auto* ctr = reinterpret_cast<const unsigned long long*>(bufs[rank] + kPeerCounterOff);
    const unsigned long long want = (epoch + 1) * (unsigned long long)world;
    bool ok = true;
    if (lane == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(ctr) < want) {
            if (globaltimer_ns() - t0 > kSpinTimeoutNs) { ok = false; break; }
            __nanosleep(64);
        }
    }
    ok = __shfl_sync(kFull, ok ? 1 : 0, 0) != 0;
    __syncwarp();
    // 4. the own slot now holds the MIN over all ranks; 5. reset it for epoch + 2
    auto* mine = reinterpret_cast<unsigned long long*>(bufs[rank] + kPeerSlotsOff) + slot;
    for (int64_t k = lane; k < K; k += 32) {
        out[k] = ok ? atomicMax_system(mine + k, 0ull) : 0ull;  // atomic read at system scope
        mine[k] = kErrNone;
    }
    __threadfence_system();
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
    const int64_t words = (kPeerSlotsOff / 8) + 2 * K;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) p[i] = (i < kPeerSlotsOff / 8) ? 0ull : kErrNone;
}

}  // namespace b64
