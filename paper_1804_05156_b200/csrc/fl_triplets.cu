// fl_triplets.cu -- generic from_triplets on the GPU.
//
// from_triplets (sparse.hpp:61-115): validate, two stable counting sorts (row,
// then column) so the triplets are in (column, row, original position) order,
// sum each duplicate group sequentially from its first value, drop sums equal
// to 0.0, count columns.  Here: one stable LSD radix sort of the 64-bit keys
// (column << 32 | row) carrying the original positions -- stability keeps the
// original order inside each (column, row) group -- then one thread per group
// sums it in that order (bitwise the reference), a scan compacts the non-zero
// sums, and a column histogram + scan gives col_ptr.
#include <cuda_runtime.h>

#include <cstdint>

#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

namespace {

constexpr int kRB = 256;            // threads per radix block
constexpr int kRItems = 8;          // rounds per tile
constexpr int kRTile = kRB * kRItems;
constexpr int kRWarps = kRB / 32;

__global__ void k_trip_keys(int64_t nz, int32_t m, int32_t n, const int32_t* __restrict__ ii,
                            const int32_t* __restrict__ jj, uint64_t* __restrict__ key,
                            uint32_t* __restrict__ idx, uint32_t* __restrict__ err) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = ii[k], c = jj[k];
        if (r < 0 || r >= m || c < 0 || c >= n) atomicOr(err, DERR_INDEX);
        key[k] = ((uint64_t)(uint32_t)c << 32) | (uint32_t)r;
        idx[k] = (uint32_t)k;
    }
}

__device__ __forceinline__ int digit_of(uint64_t key, int shift) { return (int)((key >> shift) & 0xFF); }

// per-tile digit histograms, digit-major: hist[d * nblocks + block]
__global__ void __launch_bounds__(kRB) k_radix_hist(int64_t nz, int shift, const uint64_t* __restrict__ key,
                                                    int32_t* __restrict__ hist, int nblocks) {
    __shared__ int32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRTile;
    for (int r = 0; r < kRItems; ++r) {
        const int64_t e = base + r * kRB + threadIdx.x;
        if (e < nz) atomicAdd(&h[digit_of(key[e], shift)], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: element order inside a tile is (round, warp, lane)
__global__ void __launch_bounds__(kRB) k_radix_scatter(int64_t nz, int shift, int nblocks,
                                                       const uint64_t* __restrict__ key_in,
                                                       const uint32_t* __restrict__ idx_in,
                                                       const int32_t* __restrict__ off,
                                                       uint64_t* __restrict__ key_out,
                                                       uint32_t* __restrict__ idx_out) {
    __shared__ int32_t wcnt[kRWarps][256];
    __shared__ int32_t woff[kRWarps][256];
    __shared__ int32_t run[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lower = (1u << lane) - 1;
    run[threadIdx.x] = off[(int64_t)threadIdx.x * nblocks + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kRTile;
    for (int r = 0; r < kRItems; ++r) {
        for (int q = threadIdx.x; q < kRWarps * 256; q += kRB) (&wcnt[0][0])[q] = 0;
        __syncthreads();
        const int64_t e = base + r * kRB + threadIdx.x;
        const bool valid = e < nz;
        uint64_t k = 0;
        uint32_t x = 0;
        int d = 256 + lane;  // invalid lanes never match a digit
        if (valid) {
            k = key_in[e];
            x = idx_in[e];
            d = digit_of(k, shift);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lower);
        if (valid && rank == 0) wcnt[w][d] = __popc(peers);
        __syncthreads();
        {
            const int dd = threadIdx.x;  // one thread per digit: prefix over warps
            int32_t o = run[dd];
            for (int q = 0; q < kRWarps; ++q) {
                woff[q][dd] = o;
                o += wcnt[q][dd];
            }
            run[dd] = o;
        }
        __syncthreads();
        if (valid) {
            const int32_t pos = woff[w][d] + rank;
            key_out[pos] = k;
            idx_out[pos] = x;
        }
        __syncthreads();
    }
}

__global__ void k_group_heads(int64_t nz, const uint64_t* __restrict__ key, int32_t* __restrict__ head) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nz;
         k += (int64_t)gridDim.x * blockDim.x)
        head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

// one thread per group: sequential sum from the first value (sparse.hpp:98-104)
__global__ void k_group_sum(int64_t nz, const uint64_t* __restrict__ key, const uint32_t* __restrict__ idx,
                            const int32_t* __restrict__ head_pos, const double* __restrict__ s,
                            double* __restrict__ gsum, uint64_t* __restrict__ gkey,
                            int32_t* __restrict__ keep) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nz;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (!(k == 0 || key[k] != key[k - 1])) continue;
        double sum = s[idx[k]];
        int64_t q = k + 1;
        while (q < nz && key[q] == key[k]) sum = __dadd_rn(sum, s[idx[q++]]);
        const int32_t g = head_pos[k];
        gsum[g] = sum;
        gkey[g] = key[k];
        keep[g] = sum != 0.0 ? 1 : 0;  // sparse.hpp:105
    }
}

__global__ void k_group_emit(int32_t ng, const uint64_t* __restrict__ gkey, const double* __restrict__ gsum,
                             const int32_t* __restrict__ keep, const int32_t* __restrict__ kpos,
                             int32_t* __restrict__ row_idx, double* __restrict__ values,
                             int32_t* __restrict__ ccount) {
    for (int32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        if (!keep[g]) continue;
        const int32_t o = kpos[g];
        row_idx[o] = (int32_t)(gkey[g] & 0xFFFFFFFFull);
        values[o] = gsum[g];
        atomicAdd(ccount + (int32_t)(gkey[g] >> 32), 1);
    }
}

}  // namespace

int launch_from_triplets(fl_ctx* ctx, int32_t m, int32_t n, int64_t nz, const int32_t* ii,
                         const int32_t* jj, const double* ss, fl_result* res) {
    const cudaStream_t s = ctx->stream;
    res->what = FL_OUT_STIFFNESS;
    res->n = n;
    res->m = m;
    res->col_begin = 0;
    res->sizes_valid = false;
    FL_TRY(res->counters.ensure(sizeof(uint32_t) * CNT_WORDS));
    uint32_t* counters = res->counters.as<uint32_t>();
    FL_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * CNT_WORDS, s));
    const size_t nz1 = (size_t)std::max<int64_t>(nz, 1);
    DevBuf k0, k1, i0, i1, aux, gsum, gkey, keep, kpos, hist;
    auto release = [&]() {
        DevBuf* all[] = {&k0, &k1, &i0, &i1, &aux, &gsum, &gkey, &keep, &kpos, &hist};
        for (DevBuf* d : all) d->release();
    };
    auto run = [&]() -> int {
        FL_TRY(k0.ensure(8 * nz1));
        FL_TRY(k1.ensure(8 * nz1));
        FL_TRY(i0.ensure(4 * nz1));
        FL_TRY(i1.ensure(4 * nz1));
        FL_TRY(aux.ensure(4 * (nz1 + 1)));
        const int grid = (int)std::min<int64_t>(std::max<int64_t>(div_up(nz, 256), 1), (int64_t)ctx->sm_count * 16);
        if (nz > 0) {
            k_trip_keys<<<grid, 256, 0, s>>>(nz, m, n, ii, jj, k0.as<uint64_t>(), i0.as<uint32_t>(),
                                             counters + CNT_ERR);
            count_launch(ctx);
        }
        uint32_t* h = static_cast<uint32_t*>(ctx->pinned);
        FL_CUDA(cudaMemcpyAsync(h, counters + CNT_ERR, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        if (h[0] & DERR_INDEX) return set_error(FL_E_INDEX_OUT_OF_RANGE, "triplet index outside the matrix");
        // stable LSD radix sort over the digits the indices use
        int rbits = 0, cbits = 0;
        while (rbits < 31 && ((int64_t)1 << rbits) < m) ++rbits;
        while (cbits < 31 && ((int64_t)1 << cbits) < n) ++cbits;
        const int nblocks = (int)std::max<int64_t>(1, (nz + kRTile - 1) / kRTile);
        FL_TRY(hist.ensure(sizeof(int32_t) * (256 * (size_t)nblocks + 1)));
        FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(256 * (int64_t)nblocks)));
        uint64_t* kin = k0.as<uint64_t>();
        uint64_t* kout = k1.as<uint64_t>();
        uint32_t* xin = i0.as<uint32_t>();
        uint32_t* xout = i1.as<uint32_t>();
        int shifts[8], np = 0;
        for (int sh = 0; sh < rbits; sh += 8) shifts[np++] = sh;
        for (int sh = 0; sh < cbits; sh += 8) shifts[np++] = 32 + sh;
        for (int pidx = 0; pidx < np && nz > 0; ++pidx) {
            const int sh = shifts[pidx];
            k_radix_hist<<<nblocks, kRB, 0, s>>>(nz, sh, kin, hist.as<int32_t>(), nblocks);
            const int32_t* hp = hist.as<int32_t>();
            FL_CUDA(launch_scan<int32_t>(256 * (int64_t)nblocks,
                                         [hp] __device__(int64_t i) { return (int64_t)hp[i]; },
                                         aux.as<int32_t>(), ctx->scan_ws.p, s));
            k_radix_scatter<<<nblocks, kRB, 0, s>>>(nz, sh, nblocks, kin, xin, aux.as<int32_t>(), kout, xout);
            count_launch(ctx, 3);
            std::swap(kin, kout);
            std::swap(xin, xout);
        }
        // duplicate groups
        int32_t* head = aux.as<int32_t>();
        FL_TRY(kpos.ensure(4 * (nz1 + 1)));
        if (nz > 0) {
            k_group_heads<<<grid, 256, 0, s>>>(nz, kin, head);
            count_launch(ctx);
        }
        FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(nz)));
        const int32_t* hd = head;
        FL_CUDA(launch_scan<int32_t>(nz, [hd] __device__(int64_t i) { return (int64_t)hd[i]; },
                                     kpos.as<int32_t>(), ctx->scan_ws.p, s));
        count_launch(ctx);
        FL_CUDA(cudaMemcpyAsync(h, kpos.as<int32_t>() + nz, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        const int32_t ng = (int32_t)h[0];
        const size_t ng1 = (size_t)std::max(ng, 1);
        FL_TRY(gsum.ensure(8 * ng1));
        FL_TRY(gkey.ensure(8 * ng1));
        FL_TRY(keep.ensure(4 * (ng1 + 1)));
        if (nz > 0) {
            k_group_sum<<<grid, 256, 0, s>>>(nz, kin, xin, kpos.as<int32_t>(), ss, gsum.as<double>(),
                                             gkey.as<uint64_t>(), keep.as<int32_t>());
            count_launch(ctx);
        }
        // compaction of the non-zero sums; column counts -> col_ptr
        int32_t* kp2 = head;  // reuse
        const int32_t* kk = keep.as<int32_t>();
        FL_CUDA(launch_scan<int32_t>(ng, [kk] __device__(int64_t i) { return (int64_t)kk[i]; }, kp2,
                                     ctx->scan_ws.p, s));
        count_launch(ctx);
        FL_CUDA(cudaMemcpyAsync(h, kp2 + ng, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        const int64_t nnz = (int32_t)h[0];
        FL_TRY(res->arr[FL_A_ROW_IDX].ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1)));
        FL_TRY(res->arr[FL_A_VALUES].ensure(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1)));
        FL_TRY(res->arr[FL_A_COL_PTR].ensure(sizeof(int32_t) * ((size_t)n + 1)));
        int32_t* ccount = kpos.as<int32_t>();  // reuse (groups summed already)
        FL_TRY(kpos.ensure(4 * ((size_t)std::max<int64_t>(nz, n) + 1)));
        ccount = kpos.as<int32_t>();
        FL_CUDA(cudaMemsetAsync(ccount, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        if (ng > 0) {
            k_group_emit<<<std::min(div_up(ng, 256), ctx->sm_count * 16), 256, 0, s>>>(
                ng, gkey.as<uint64_t>(), gsum.as<double>(), keep.as<int32_t>(), kp2,
                res->arr[FL_A_ROW_IDX].as<int32_t>(), res->arr[FL_A_VALUES].as<double>(), ccount);
            count_launch(ctx);
        }
        const int32_t* cct = ccount;
        FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(n)));
        FL_CUDA(launch_scan<int32_t>(n, [cct] __device__(int64_t i) { return (int64_t)cct[i]; },
                                     res->arr[FL_A_COL_PTR].as<int32_t>(), ctx->scan_ws.p, s));
        count_launch(ctx);
        FL_CUDA(cudaGetLastError());
        return FL_OK;
    };
    const int rc = run();
    cudaStreamSynchronize(s);
    release();
    return rc;
}

}  // namespace fl
