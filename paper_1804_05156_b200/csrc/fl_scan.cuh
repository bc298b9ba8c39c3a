// fl_scan.cuh -- single-pass exclusive scan with decoupled look-back.
//
// Used for the node -> incidence offsets (inc_ptr), the free-node ranks of
// partition_boundary, and (inside the column kernel) the CSC offsets.  Tiles
// take ids from an atomic ticket so a tile only ever waits on tiles that are
// already resident: forward progress without a grid barrier.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fl {

// status word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive prefix), [61:0] value.
// Flag and value travel in ONE 64-bit word, so relaxed (not acquire/release)
// accesses suffice: no other data is published through it.  ld.acquire.gpu
// compiles to CCTL.IVALL (a full L1 invalidation per poll) on sm_100a, which
// wiped every CTA's L1 working set while a tile waited (profiles/ v2 notes).
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// Called by ONE thread of the tile.  Publishes `aggregate` and returns the
// exclusive prefix of all earlier tiles.
__device__ __forceinline__ uint64_t lookback(uint64_t* status, int64_t tile, uint64_t aggregate) {
    if (tile == 0) {
        st_status(&status[0], kFlagInc | aggregate);
        return 0;
    }
    st_status(&status[tile], kFlagAgg | aggregate);
    uint64_t excl = 0;
    int64_t pred = tile - 1;
    while (true) {
        const uint64_t v = ld_status(&status[pred]);
        const uint64_t flag = v >> 62;
        if (flag == 0) continue;
        excl += v & kValMask;
        if (flag == 2) break;
        --pred;
    }
    st_status(&status[tile], kFlagInc | (excl + aggregate));
    return excl;
}

// Warp-wide variant (call with all 32 lanes of ONE warp; every lane returns the
// exclusive prefix).  Each round inspects 32 predecessors at once: the walk over
// tiles that have only published aggregates costs one L2 round trip per 32
// tiles instead of one per tile.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t* status, int64_t tile,
                                                  uint64_t aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_status(&status[0], kFlagInc | aggregate);
        return 0;
    }
    if (lane == 0) st_status(&status[tile], kFlagAgg | aggregate);
    uint64_t excl = 0;
    int64_t hi = tile - 1;  // window covers predecessors hi, hi-1, ..., hi-31
    while (true) {
        const int64_t idx = hi - lane;
        uint64_t v = idx >= 0 ? ld_status(&status[idx]) : (kFlagInc | 0ull);
        uint32_t flag = (uint32_t)(v >> 62);
        // the nearest inclusive prefix in the window
        const unsigned inc_mask = __ballot_sync(0xffffffffu, flag == 2);
        const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
        // lanes up to the inclusive one must all have published something
        const unsigned empty = __ballot_sync(0xffffffffu, flag == 0 && lane <= first_inc);
        if (empty) continue;  // re-read the same window
        uint64_t part = (lane <= first_inc) ? (v & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (first_inc < 32) break;
        hi -= 32;
    }
    if (lane == 0) st_status(&status[tile], kFlagInc | (excl + aggregate));
    return excl;
}

template <int BLOCK>
__device__ __forceinline__ int64_t block_exclusive_sum(int64_t x, int64_t* warp_sums,
                                                       int64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int64_t w = (lane < BLOCK / 32) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < BLOCK / 32) warp_sums[lane] = w;
    }
    __syncthreads();
    total = warp_sums[BLOCK / 32 - 1];
    const int64_t before = (warp > 0) ? warp_sums[warp - 1] : 0;
    __syncthreads();
    return before + incl - x;
}

// out[i] = sum_{k<i} f(k) for i in [0, n); out[n] = total (out has n+1 slots).
template <int BLOCK, int ITEMS, class OutT, class F>
__global__ void __launch_bounds__(BLOCK) k_scan(int64_t n, F f, OutT* out, uint64_t* status,
                                                unsigned int* ticket) {
    __shared__ int64_t warp_sums[BLOCK / 32];
    __shared__ int64_t s_tile, s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * (int64_t)BLOCK * ITEMS + (int64_t)threadIdx.x * ITEMS;
    int64_t v[ITEMS];
    int64_t local = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t i = base + k;
        v[k] = (i < n) ? (int64_t)f(i) : 0;
        local += v[k];
    }
    int64_t total;
    int64_t excl = block_exclusive_sum<BLOCK>(local, warp_sums, total);
    if (threadIdx.x < 32) {
        const uint64_t e = warp_lookback(status, tile, (uint64_t)total);
        if (threadIdx.x == 0) s_excl = (int64_t)e;
    }
    __syncthreads();
    excl += s_excl;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t i = base + k;
        if (i < n) out[i] = (OutT)excl;
        excl += v[k];
    }
    if (base <= n - 1 && base + ITEMS >= n) out[n] = (OutT)excl;  // the thread holding n-1
    if (n == 0 && tile == 0 && threadIdx.x == 0) out[0] = 0;
}

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;

// Host helper: exclusive scan of f over [0, n) into out[0..n].  `ws` must hold
// at least scan_ws_bytes(n) bytes; zeroed here on the stream.
inline size_t scan_ws_bytes(int64_t n) {
    const int64_t tiles = (n + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems);
    return sizeof(uint64_t) * (size_t)(tiles + 1) + 64;
}

template <class OutT, class F>
cudaError_t launch_scan(int64_t n, F f, OutT* out, void* ws, cudaStream_t s) {
    const int64_t tiles = (n + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems);
    const size_t bytes = scan_ws_bytes(n);
    cudaError_t e = cudaMemsetAsync(ws, 0, bytes, s);
    if (e != cudaSuccess) return e;
    uint64_t* status = static_cast<uint64_t*>(ws);
    unsigned int* ticket = reinterpret_cast<unsigned int*>(status + tiles);
    const int grid = tiles > 0 ? (int)tiles : 1;
    k_scan<kScanBlock, kScanItems, OutT, F><<<grid, kScanBlock, 0, s>>>(n, f, out, status, ticket);
    return cudaGetLastError();
}

}  // namespace fl
