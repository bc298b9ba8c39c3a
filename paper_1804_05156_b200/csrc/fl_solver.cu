// fl_solver.cu -- conjugate gradient on the free-node system.
//
// cg_solve (solver.hpp:63-136): x0 = 0, r = b, optional Jacobi (auto for
// n >= 1024, inv_diag = 1 / A(c,c) where stored and nonzero), p = z,
// alpha = rz / (p.Ap), x += alpha p, r -= alpha q, stop at |r| <= rel_tol |b|
// keeping the best iterate, beta = rz' / rz.  The matrix arrives as the
// reference's CSC; it is transposed once to CSR (rows sorted by column) so
// q = A p is one thread per row summing A(r, c) p[c] over ascending c from 0.0
// -- the reference's matvec order (sparse.hpp:129-141), bitwise.  Dot products
// are deterministic fixed-order block reductions (run-to-run identical; not the
// reference's sequential order, so CG iterates agree to rounding, not bits).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

namespace {

constexpr int kRed = 256;        // threads per reduction block
constexpr int kRedBlocks = 592;  // 4 per SM

__global__ void k_csr_count(int32_t n, const int32_t* __restrict__ col_ptr,
                            const int32_t* __restrict__ row_idx, int32_t* __restrict__ cnt) {
    const int64_t nnz = col_ptr[n];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + row_idx[k], 1);
}

__global__ void k_csr_fill(int32_t n, const int32_t* __restrict__ col_ptr,
                           const int32_t* __restrict__ row_idx, const double* __restrict__ val,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ col,
                           double* __restrict__ cval) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
        for (int32_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
            const int32_t pos = atomicAdd(cursor + row_idx[k], 1);
            col[pos] = c;
            cval[pos] = val[k];
        }
}

// rows ascending by column (insertion sort; rows are short)
__global__ void k_csr_sort(int32_t n, const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                           double* __restrict__ cval) {
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int32_t a = row_ptr[r], b = row_ptr[r + 1];
        for (int32_t i = a + 1; i < b; ++i) {
            const int32_t kc = col[i];
            const double kv = cval[i];
            int32_t j = i - 1;
            while (j >= a && col[j] > kc) {
                col[j + 1] = col[j];
                cval[j + 1] = cval[j];
                --j;
            }
            col[j + 1] = kc;
            cval[j + 1] = kv;
        }
    }
}

// inv_diag[c] = 1 / A(c,c) if stored and nonzero, else 1 (solver.hpp:80-86)
__global__ void k_inv_diag(int32_t n, const int32_t* __restrict__ col_ptr,
                           const int32_t* __restrict__ row_idx, const double* __restrict__ val,
                           double* __restrict__ inv) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        double d = 1.0;
        for (int32_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k)
            if (row_idx[k] == c && val[k] != 0.0) d = __ddiv_rn(1.0, val[k]);
        inv[c] = d;
    }
}

// q = A p, row-sequential in ascending column order (matvec's order)
__global__ void k_spmv(int32_t n, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                       const double* __restrict__ cval, const double* __restrict__ x,
                       double* __restrict__ y) {
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int32_t k = __ldg(row_ptr + r); k < __ldg(row_ptr + r + 1); ++k)
            s = __dadd_rn(s, __dmul_rn(__ldg(cval + k), __ldg(x + __ldg(col + k))));
        y[r] = s;
    }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    // fixed-order tree: deterministic for a fixed launch shape
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int q = 0; q < kRed / 32; ++q) t = __dadd_rn(t, sh[q]);
    __syncthreads();
    return t;
}

// partial[block] = sum a[k] * b[k] over the block's grid-stride share
__global__ void __launch_bounds__(kRed) k_dot_partial(int32_t n, const double* __restrict__ a,
                                                      const double* __restrict__ b,
                                                      double* __restrict__ partial) {
    __shared__ double sh[kRed / 32];
    double v = 0.0;
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        v = __dadd_rn(v, __dmul_rn(a[k], b[k]));
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// z = inv .* r (or r); partials of r.z and r.r
__global__ void __launch_bounds__(kRed) k_precond(int32_t n, const double* __restrict__ inv,
                                                  const double* __restrict__ r, double* __restrict__ z,
                                                  double* __restrict__ prz, double* __restrict__ prr) {
    __shared__ double sh[kRed / 32];
    double vz = 0.0, vr = 0.0;
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const double rk = r[k];
        const double zk = inv ? __dmul_rn(inv[k], rk) : rk;
        z[k] = zk;
        vz = __dadd_rn(vz, __dmul_rn(rk, zk));
        vr = __dadd_rn(vr, __dmul_rn(rk, rk));
    }
    const double tz = block_sum(vz, sh);
    const double tr = block_sum(vr, sh);
    if (threadIdx.x == 0) {
        prz[blockIdx.x] = tz;
        prr[blockIdx.x] = tr;
    }
}

// scalars s[]: 0 rz, 1 pq, 2 alpha, 3 rr, 4 rz_next, 5 beta
__global__ void k_finish(int nb, const double* __restrict__ partial, double* __restrict__ out) {
    double t = 0.0;
    for (int q = 0; q < nb; ++q) t = __dadd_rn(t, partial[q]);
    *out = t;
}

// x += alpha p; r -= alpha q (alpha = rz / pq on the device)
__global__ void k_update_xr(int32_t n, const double* __restrict__ s, const double* __restrict__ p,
                            const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r) {
    const double alpha = __ddiv_rn(s[0], s[1]);
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        x[k] = __dadd_rn(x[k], __dmul_rn(alpha, p[k]));
        r[k] = __dsub_rn(r[k], __dmul_rn(alpha, q[k]));
    }
}

// p = z + beta p, beta = rz_next / rz; then rz = rz_next
__global__ void k_update_p(int32_t n, double* __restrict__ s, const double* __restrict__ z,
                           double* __restrict__ p) {
    const double beta = __ddiv_rn(s[4], s[0]);
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        p[k] = __dadd_rn(z[k], __dmul_rn(beta, p[k]));
}

__global__ void k_roll_rz(double* s) { s[0] = s[4]; }

// u = u0 with u[free[k]] = x[k] (solve_poisson's scatter, solver.hpp:243-245)
__global__ void k_scatter_free(int32_t nf, const int32_t* __restrict__ free_nodes,
                               const double* __restrict__ x, double* __restrict__ u) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x)
        u[free_nodes[k]] = x[k];
}

}  // namespace

struct CgWork {
    DevBuf row_ptr, col, cval, inv, x, best, r, z, p, q, partial, s;
};

// CSR (rows sorted by column) of an m x n CSC matrix into row_ptr / col / cval;
// `cnt` is scratch for m + 1 int32
static int build_csr(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                     const double* values, int64_t nnz, int32_t* cnt, DevBuf& row_ptr, DevBuf& col,
                     DevBuf& cval) {
    const cudaStream_t s = ctx->stream;
    FL_TRY(row_ptr.ensure(sizeof(int32_t) * ((size_t)m + 1)));
    FL_TRY(col.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1)));
    FL_TRY(cval.ensure(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1)));
    FL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)m + 1), s));
    if (nnz > 0) {
        k_csr_count<<<(int)std::min<int64_t>(div_up(nnz, 256), ctx->sm_count * 16), 256, 0, s>>>(
            n, col_ptr, row_idx, cnt);
        count_launch(ctx);
    }
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(m)));
    const int32_t* cc = cnt;
    FL_CUDA(launch_scan<int32_t>(m, [cc] __device__(int64_t i) { return (int64_t)cc[i]; },
                                 row_ptr.as<int32_t>(), ctx->scan_ws.p, s));
    count_launch(ctx);
    FL_CUDA(cudaMemcpyAsync(cnt, row_ptr.p, sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToDevice, s));
    const int gn = std::max(1, std::min(div_up(n, 256), ctx->sm_count * 8));
    const int gm = std::max(1, std::min(div_up(m, 256), ctx->sm_count * 8));
    k_csr_fill<<<gn, 256, 0, s>>>(n, col_ptr, row_idx, values, cnt, col.as<int32_t>(), cval.as<double>());
    k_csr_sort<<<gm, 256, 0, s>>>(m, row_ptr.as<int32_t>(), col.as<int32_t>(), cval.as<double>());
    count_launch(ctx, 2);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// y = A x with the reference's matvec order (sparse.hpp:129-141), bitwise
int matvec_device(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                  const double* values, const double* x, double* y) {
    const cudaStream_t s = ctx->stream;
    int32_t* h = reinterpret_cast<int32_t*>(static_cast<double*>(ctx->pinned) + 8);
    FL_CUDA(cudaMemcpyAsync(h, col_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    const int64_t nnz = h[0];
    DevBuf row_ptr, col, cval, cnt;
    int rc = cnt.ensure(sizeof(int32_t) * ((size_t)m + 1));
    if (!rc) rc = build_csr(ctx, m, n, col_ptr, row_idx, values, nnz, cnt.as<int32_t>(), row_ptr, col, cval);
    if (!rc && m > 0) {
        k_spmv<<<std::min(div_up(m, 256), ctx->sm_count * 8), 256, 0, s>>>(
            m, row_ptr.as<int32_t>(), col.as<int32_t>(), cval.as<double>(), x, y);
        count_launch(ctx);
        if (cudaGetLastError() != cudaSuccess) rc = set_error(FL_ERR_CUDA, "k_spmv launch");
    }
    cudaStreamSynchronize(s);
    row_ptr.release();
    col.release();
    cval.release();
    cnt.release();
    return rc;
}

int cg_solve_device(fl_ctx* ctx, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                    const double* values, const double* b, double rel_tol, int64_t max_iter,
                    int precond, double* x_out, int64_t* iterations, double* relres, int32_t* converged) {
    const cudaStream_t s = ctx->stream;
    *iterations = 0;
    *relres = 0.0;
    *converged = 1;
    if (n == 0) return FL_OK;
    CgWork w;
    auto cleanup = [&]() {
        DevBuf* all[] = {&w.row_ptr, &w.col, &w.cval, &w.inv, &w.x, &w.best, &w.r, &w.z, &w.p, &w.q,
                         &w.partial, &w.s};
        for (DevBuf* d : all) d->release();
    };
    auto run = [&]() -> int {
        double* h = static_cast<double*>(ctx->pinned);
        int32_t* hi = reinterpret_cast<int32_t*>(h + 8);
        FL_CUDA(cudaMemcpyAsync(hi, col_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        const int64_t nnz = hi[0];
        const size_t nd = sizeof(double) * (size_t)n;
        for (DevBuf* d : {&w.inv, &w.x, &w.best, &w.r, &w.z, &w.p, &w.q}) FL_TRY(d->ensure(nd));
        FL_TRY(w.partial.ensure(sizeof(double) * 2 * kRedBlocks));
        FL_TRY(w.s.ensure(sizeof(double) * 8));
        double* S = w.s.as<double>();
        double* part = w.partial.as<double>();
        const int grid = std::min(div_up(n, 256), ctx->sm_count * 8);
        const int rblocks = std::min(kRedBlocks, std::max(1, div_up(n, kRed)));
        // CSR of A (rows sorted by column); q is scratch until the loop
        FL_TRY(build_csr(ctx, n, n, col_ptr, row_idx, values, nnz, w.q.as<int32_t>(), w.row_ptr,
                         w.col, w.cval));
        const bool jacobi = precond == 1 || (precond == 2 && n >= 1024);  // solver.hpp:44-48
        const double* inv = nullptr;
        if (jacobi) {
            k_inv_diag<<<grid, 256, 0, s>>>(n, col_ptr, row_idx, values, w.inv.as<double>());
            count_launch(ctx);
            inv = w.inv.as<double>();
        }
        double* x = w.x.as<double>();
        double* r = w.r.as<double>();
        double* z = w.z.as<double>();
        double* p = w.p.as<double>();
        double* q = w.q.as<double>();
        FL_CUDA(cudaMemsetAsync(x, 0, nd, s));
        FL_CUDA(cudaMemcpyAsync(r, b, nd, cudaMemcpyDeviceToDevice, s));
        // bnorm, z = M r, rz
        k_precond<<<rblocks, kRed, 0, s>>>(n, inv, r, z, part, part + kRedBlocks);
        k_finish<<<1, 1, 0, s>>>(rblocks, part, S + 0);
        k_finish<<<1, 1, 0, s>>>(rblocks, part + kRedBlocks, S + 3);
        count_launch(ctx, 3);
        FL_CUDA(cudaMemcpyAsync(h, S, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        const double bnorm = std::sqrt(h[3]);
        if (bnorm == 0.0) {  // b = 0 short-circuits to x = 0
            FL_CUDA(cudaMemcpyAsync(x_out, x, nd, cudaMemcpyDeviceToDevice, s));
            return FL_OK;
        }
        FL_CUDA(cudaMemcpyAsync(p, z, nd, cudaMemcpyDeviceToDevice, s));
        FL_CUDA(cudaMemcpyAsync(w.best.p, x, nd, cudaMemcpyDeviceToDevice, s));
        const int64_t cap = max_iter > 0 ? max_iter : 10 * (int64_t)n;
        double best_relres = 1.0;
        for (int64_t it = 1; it <= cap; ++it) {
            k_spmv<<<grid, 256, 0, s>>>(n, w.row_ptr.as<int32_t>(), w.col.as<int32_t>(), w.cval.as<double>(), p, q);
            k_dot_partial<<<rblocks, kRed, 0, s>>>(n, p, q, part);
            k_finish<<<1, 1, 0, s>>>(rblocks, part, S + 1);
            k_update_xr<<<grid, 256, 0, s>>>(n, S, p, q, x, r);
            k_precond<<<rblocks, kRed, 0, s>>>(n, inv, r, z, part, part + kRedBlocks);
            k_finish<<<1, 1, 0, s>>>(rblocks, part, S + 4);
            k_finish<<<1, 1, 0, s>>>(rblocks, part + kRedBlocks, S + 3);
            count_launch(ctx, 7);
            FL_CUDA(cudaMemcpyAsync(h, S, sizeof(double) * 5, cudaMemcpyDeviceToHost, s));
            FL_CUDA(cudaStreamSynchronize(s));
            if (!(h[1] > 0.0))
                return set_error(FL_E_NOT_POSITIVE_DEFINITE, "cg_solve: non-positive curvature encountered");
            const double rel = std::sqrt(h[3]) / bnorm;
            if (rel < best_relres) {
                best_relres = rel;
                FL_CUDA(cudaMemcpyAsync(w.best.p, x, nd, cudaMemcpyDeviceToDevice, s));
            }
            *iterations = it;
            if (rel <= rel_tol) {
                *relres = rel;
                FL_CUDA(cudaMemcpyAsync(x_out, x, nd, cudaMemcpyDeviceToDevice, s));
                return FL_OK;
            }
            k_update_p<<<grid, 256, 0, s>>>(n, S, z, p);
            k_roll_rz<<<1, 1, 0, s>>>(S);
            count_launch(ctx, 2);
        }
        *relres = best_relres;
        *converged = 0;
        FL_CUDA(cudaMemcpyAsync(x_out, w.best.p, nd, cudaMemcpyDeviceToDevice, s));
        return FL_OK;
    };
    const int rc = run();
    cudaStreamSynchronize(s);
    cleanup();
    return rc;
}

namespace {

// A with row and column `pin` removed (indices above pin shift down by one)
__global__ void k_drop_count(int32_t n, int32_t pin, const int32_t* __restrict__ col_ptr,
                             const int32_t* __restrict__ row_idx, int32_t* __restrict__ cnt) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        if (c == pin) continue;
        int32_t k = 0;
        for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) k += row_idx[e] != pin;
        cnt[c < pin ? c : c - 1] = k;
    }
}

__global__ void k_drop_fill(int32_t n, int32_t pin, const int32_t* __restrict__ col_ptr,
                            const int32_t* __restrict__ row_idx, const double* __restrict__ val,
                            const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_row,
                            double* __restrict__ out_val) {
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        if (c == pin) continue;
        int32_t o = out_ptr[c < pin ? c : c - 1];
        for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
            const int32_t r = row_idx[e];
            if (r == pin) continue;
            out_row[o] = r < pin ? r : r - 1;
            out_val[o] = val[e];
            ++o;
        }
    }
}

// b_r = (b - mean) without entry pin (enforce_compatibility, system.hpp:205-212)
__global__ void k_drop_rhs(int32_t n, int32_t pin, const double* __restrict__ mean,
                           const double* __restrict__ b, double* __restrict__ br) {
    const double mu = *mean;
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        if (k != pin) br[k < pin ? k : k - 1] = __dsub_rn(b[k], mu);
}

// partial sums of b (the mean)
__global__ void __launch_bounds__(kRed) k_sum_partial(int32_t n, const double* __restrict__ a,
                                                      double* __restrict__ partial) {
    __shared__ double sh[kRed / 32];
    double v = 0.0;
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        v = __dadd_rn(v, a[k]);
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void k_mean(int nb, const double* __restrict__ partial, double n, double* __restrict__ out) {
    double t = 0.0;
    for (int q = 0; q < nb; ++q) t = __dadd_rn(t, partial[q]);
    *out = __ddiv_rn(t, n);
}

// u = x with 0 at pin
__global__ void k_insert_pin(int32_t n, int32_t pin, const double* __restrict__ x, double* __restrict__ u) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        u[k] = k == pin ? 0.0 : x[k < pin ? k : k - 1];
}

// zero_average_shift (system.hpp:217-234): partials of sum avg(u)|t| and sum |t|
template <int D>
__global__ void __launch_bounds__(kRed) k_shift_partial(int32_t nt, const double* __restrict__ nodes,
                                                        const int32_t* __restrict__ elems,
                                                        const double* __restrict__ u,
                                                        double* __restrict__ pw, double* __restrict__ pt) {
    __shared__ double sh[kRed / 32];
    double w = 0.0, tot = 0.0;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        int32_t v[D + 1];
        for (int k = 0; k <= D; ++k) v[k] = elems[(size_t)t * (D + 1) + k];
        double meas;
        if (D == 2) {  // mesh.hpp:34-38
            const double* a = nodes + (size_t)v[0] * 2;
            const double* b = nodes + (size_t)v[1] * 2;
            const double* c = nodes + (size_t)v[2] * 2;
            meas = fabs(__dmul_rn(0.5, __dsub_rn(__dmul_rn(__dsub_rn(b[0], a[0]), __dsub_rn(c[1], a[1])),
                                                 __dmul_rn(__dsub_rn(c[0], a[0]), __dsub_rn(b[1], a[1])))));
        } else {  // mesh.hpp:42-51
            const double* a = nodes + (size_t)v[0] * 3;
            double e[3][3];
            for (int k = 0; k < 3; ++k)
                for (int x = 0; x < 3; ++x) e[k][x] = __dsub_rn(nodes[(size_t)v[k + 1] * 3 + x], a[x]);
            const double cx = __dsub_rn(__dmul_rn(e[0][1], e[1][2]), __dmul_rn(e[0][2], e[1][1]));
            const double cy = __dsub_rn(__dmul_rn(e[0][2], e[1][0]), __dmul_rn(e[0][0], e[1][2]));
            const double cz = __dsub_rn(__dmul_rn(e[0][0], e[1][1]), __dmul_rn(e[0][1], e[1][0]));
            meas = fabs(__ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, e[2][0]), __dmul_rn(cy, e[2][1])),
                                            __dmul_rn(cz, e[2][2])), 6.0));
        }
        double avg = 0.0;
        for (int k = 0; k <= D; ++k) avg = __dadd_rn(avg, u[v[k]]);
        avg = __ddiv_rn(avg, (double)(D + 1));
        w = __dadd_rn(w, __dmul_rn(avg, meas));
        tot = __dadd_rn(tot, meas);
    }
    const double a = block_sum(w, sh);
    const double b = block_sum(tot, sh);
    if (threadIdx.x == 0) {
        pw[blockIdx.x] = a;
        pt[blockIdx.x] = b;
    }
}

__global__ void k_shift(int32_t n, int nb, const double* __restrict__ pw, const double* __restrict__ pt,
                        double* __restrict__ u) {
    double w = 0.0, t = 0.0;
    for (int q = 0; q < nb; ++q) {
        w = __dadd_rn(w, pw[q]);
        t = __dadd_rn(t, pt[q]);
    }
    const double c = __ddiv_rn(w, t);
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        u[k] = __dsub_rn(u[k], c);
}

}  // namespace

// solve_poisson's pure-Neumann path (solver.hpp:254-276) on device arrays
int solve_neumann_device(fl_ctx* ctx, int dim, int32_t n, int32_t nt, const double* nodes,
                         const int32_t* elems, const int32_t* col_ptr, const int32_t* row_idx,
                         const double* values, const double* b, int32_t pin, double rel_tol,
                         int64_t max_iter, int precond, double* u, int64_t* iterations, double* relres,
                         int32_t* converged) {
    const cudaStream_t s = ctx->stream;
    if (pin < 0 || pin >= n) return set_error(FL_E_INDEX_OUT_OF_RANGE, "pin_node out of range");
    DevBuf cnt, ptr, row, val, br, x, part;
    auto release = [&]() {
        DevBuf* all[] = {&cnt, &ptr, &row, &val, &br, &x, &part};
        for (DevBuf* d : all) d->release();
    };
    auto run = [&]() -> int {
        const int32_t nr = n - 1;
        const int g = std::max(1, std::min(div_up(n, 256), ctx->sm_count * 8));
        FL_TRY(part.ensure(sizeof(double) * (2 * kRedBlocks + 2)));
        double* pp = part.as<double>();
        double* mean = pp + 2 * kRedBlocks;
        const int rb = std::min(kRedBlocks, std::max(1, div_up(n, kRed)));
        k_sum_partial<<<rb, kRed, 0, s>>>(n, b, pp);
        k_mean<<<1, 1, 0, s>>>(rb, pp, (double)n, mean);
        FL_TRY(cnt.ensure(sizeof(int32_t) * ((size_t)nr + 1)));
        FL_TRY(ptr.ensure(sizeof(int32_t) * ((size_t)nr + 2)));
        FL_TRY(br.ensure(sizeof(double) * (size_t)std::max(nr, 1)));
        FL_TRY(x.ensure(sizeof(double) * (size_t)std::max(nr, 1)));
        k_drop_count<<<g, 256, 0, s>>>(n, pin, col_ptr, row_idx, cnt.as<int32_t>());
        k_drop_rhs<<<g, 256, 0, s>>>(n, pin, mean, b, br.as<double>());
        count_launch(ctx, 4);
        FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(nr)));
        const int32_t* cc = cnt.as<int32_t>();
        FL_CUDA(launch_scan<int32_t>(nr, [cc] __device__(int64_t i) { return (int64_t)cc[i]; },
                                     ptr.as<int32_t>(), ctx->scan_ws.p, s));
        count_launch(ctx);
        int32_t* h = reinterpret_cast<int32_t*>(static_cast<double*>(ctx->pinned) + 8);
        FL_CUDA(cudaMemcpyAsync(h, ptr.as<int32_t>() + nr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FL_CUDA(cudaStreamSynchronize(s));
        const int64_t nnz = h[0];
        FL_TRY(row.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1)));
        FL_TRY(val.ensure(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1)));
        k_drop_fill<<<g, 256, 0, s>>>(n, pin, col_ptr, row_idx, values, ptr.as<int32_t>(), row.as<int32_t>(),
                                      val.as<double>());
        count_launch(ctx);
        FL_TRY(cg_solve_device(ctx, nr, ptr.as<int32_t>(), row.as<int32_t>(), val.as<double>(),
                               br.as<double>(), rel_tol, max_iter, precond, x.as<double>(), iterations,
                               relres, converged));
        k_insert_pin<<<g, 256, 0, s>>>(n, pin, x.as<double>(), u);
        const int rt = std::min(kRedBlocks, std::max(1, div_up(nt, kRed)));
        if (dim == 2) k_shift_partial<2><<<rt, kRed, 0, s>>>(nt, nodes, elems, u, pp, pp + kRedBlocks);
        else k_shift_partial<3><<<rt, kRed, 0, s>>>(nt, nodes, elems, u, pp, pp + kRedBlocks);
        k_shift<<<g, 256, 0, s>>>(n, rt, pp, pp + kRedBlocks, u);
        count_launch(ctx, 3);
        FL_CUDA(cudaGetLastError());
        return FL_OK;
    };
    const int rc = run();
    cudaStreamSynchronize(s);
    release();
    return rc;
}

int scatter_free(fl_ctx* ctx, int32_t nf, const int32_t* free_nodes, const double* x, double* u) {
    if (nf > 0) {
        k_scatter_free<<<std::min(div_up(nf, 256), ctx->sm_count * 8), 256, 0, ctx->stream>>>(nf, free_nodes,
                                                                                             x, u);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

}  // namespace fl
