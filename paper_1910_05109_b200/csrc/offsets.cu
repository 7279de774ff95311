// offsets.cu -- output offsets of a batch, computed on the device
// (b64_encode_batch_offsets / b64_decode_batch_offsets).
//
// out_off[i] = sum over j < i of len_out(in_off[j+1] - in_off[j]), i = 0..count,
// with len_out the encode length law 4*ceil(L/3) or the decode
// capacity 3*floor(L/4).  Three launches and no
// workspace: out_off itself holds the per-tile partial sums between them.
//   1. off_tile_sum_kernel: tile k (kScanTile strings) writes its sum to the
//      slot out_off[min((k+1)*T, count)] -- a cell that only tile k+1 (or
//      nobody: out_off[count]) later writes.
//   2. off_tile_scan_kernel (one CTA): the slots become inclusive prefix sums
//      over tiles, i.e. slot k = the exclusive prefix of tile k+1, and
//      out_off[count] = the total.
//   3. off_fill_kernel: tile k reads its prefix from slot k-1 = out_off[k*T]
//      (0 for k = 0) and writes out_off[k*T .. (k+1)*T) -- its own range, so
//      no tile reads a cell another tile writes.
#include "b64_device.cuh"

namespace b64 {

constexpr int kScanItems = 8;
constexpr int64_t kScanTile = int64_t(kThreads) * kScanItems;  // strings per tile

template <int LAW>  // 0: encode 4*ceil(L/3); 1: decode 3*floor(L/4)
__device__ __forceinline__ int64_t out_len_of(int64_t L) {
    return LAW == 0 ? 4 * ((L + 2) / 3) : 3 * (L >> 2);
}

// Block-wide exclusive scan of one int64 per thread (kThreads threads); *total = the sum.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* s_warp, int64_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    int64_t wpre = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const int64_t t = s_warp[w];
        if (w < wid) wpre += t;
        all += t;
    }
    __syncthreads();
    *total = all;
    return wpre + x - v;
}

template <int LAW>
__global__ void __launch_bounds__(kThreads) off_tile_sum_kernel(const int64_t* __restrict__ in_off, int64_t count,
                                                                int64_t* __restrict__ out_off) {
    __shared__ int64_t s_warp[kThreads / 32];
    griddep_wait();
    const int64_t ntile = (count + kScanTile - 1) / kScanTile;
    for (int64_t k = blockIdx.x; k < ntile; k += gridDim.x) {
        const int64_t i0 = k * kScanTile + int64_t(threadIdx.x) * kScanItems;
        int64_t sum = 0;
        if (i0 < count) {
            int64_t prev = in_off[i0];
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) {
                if (i0 + j < count) {
                    const int64_t nx = in_off[i0 + j + 1];
                    sum += out_len_of<LAW>(nx - prev);
                    prev = nx;
                }
            }
        }
        int64_t total;
        block_exclusive_scan(sum, s_warp, &total);
        if (threadIdx.x == 0) out_off[min((k + 1) * kScanTile, count)] = total;
    }
}

__global__ void __launch_bounds__(1024) off_tile_scan_kernel(int64_t* __restrict__ out_off, int64_t count) {
    __shared__ int64_t s_warp[32];
    griddep_wait();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ntile = (count + kScanTile - 1) / kScanTile;
    int64_t carry = 0;
    for (int64_t k0 = 0; k0 < ntile; k0 += 1024) {
        const int64_t k = k0 + threadIdx.x;
        int64_t* slot = out_off + min((k + 1) * kScanTile, count);
        const int64_t v = k < ntile ? *slot : 0;
        int64_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        int64_t wpre = 0, all = 0;
        for (int w = 0; w < 32; ++w) {
            const int64_t t = s_warp[w];
            if (w < wid) wpre += t;
            all += t;
        }
        if (k < ntile) *slot = carry + wpre + x;  // inclusive over tiles 0..k
        carry += all;
        __syncthreads();
    }
    if (threadIdx.x == 0) out_off[0] = 0;
}

template <int LAW>
__global__ void __launch_bounds__(kThreads) off_fill_kernel(const int64_t* __restrict__ in_off, int64_t count,
                                                            int64_t* __restrict__ out_off) {
    __shared__ int64_t s_warp[kThreads / 32];
    griddep_wait();
    const int64_t ntile = (count + kScanTile - 1) / kScanTile;
    for (int64_t k = blockIdx.x; k < ntile; k += gridDim.x) {
        const int64_t prefix = out_off[k * kScanTile];  // slot of tile k-1 (out_off[0] = 0 for k = 0)
        __syncthreads();  // every thread has read the prefix before thread 0 overwrites the cell
        const int64_t i0 = k * kScanTile + int64_t(threadIdx.x) * kScanItems;
        int64_t len[kScanItems];
        int64_t sum = 0;
        if (i0 < count) {
            int64_t prev = in_off[i0];
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) {
                len[j] = 0;
                if (i0 + j < count) {
                    const int64_t nx = in_off[i0 + j + 1];
                    len[j] = out_len_of<LAW>(nx - prev);
                    prev = nx;
                }
                sum += len[j];
            }
        }
        int64_t total;
        int64_t run = prefix + block_exclusive_scan(sum, s_warp, &total);
        if (i0 < count) {
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) {
                if (i0 + j < count) out_off[i0 + j] = run;
                run += len[j];
            }
        }
    }
}

}  // namespace b64
