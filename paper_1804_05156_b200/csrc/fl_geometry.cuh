// fl_geometry.cuh -- per-element arithmetic of the reference, FMA-free.
//
// Every expression keeps the reference's operand order so the rounded result
// is bitwise the reference's (the translation unit is compiled -fmad=false;
// divisions go through fl::div_by, which is the correctly rounded quotient).
// Citations: /root/reference/proj/include/femlite/<file>:<line>.
#pragma once

#include "fl_internal.cuh"

namespace fl {

// quadrature.hpp:65-71 (tet4)
constexpr double kTet4A = 0.58541019662496845;
constexpr double kTet4B = 0.13819660112501051;
constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi

struct FieldDesc {
    int kind;
    double value;
    const double* samples;
};

// built-in fields at a point (z = 0 in 2-D, mesh.hpp:72-77)
__device__ __forceinline__ double eval_point(const FieldDesc& f, double x, double y, double z) {
    switch (f.kind) {
    case FL_FIELD_CONST: return f.value;
    case FL_FIELD_X: return x;
    case FL_FIELD_XYZ: return x + y + z;
    case FL_FIELD_SINSIN: return sin(kPi * x) * sin(kPi * y);
    default: return 0.0;
    }
}

// Column j of the local stiffness (s_ij, i = 0..D) and the load contribution
// of local vertex j, for element t.  `vx` holds the D+1 vertex coordinates.
template <int D>
struct ElemCol;

// ---------------------------------------------------------------------------
// 2-D: assembly.hpp:133-151 (edge vectors, area, rotated normals),
//      assembly.hpp:283-292 (s = n_i.n_j / (4 area)), system.hpp:80-96 (load)
// ---------------------------------------------------------------------------
template <>
struct ElemCol<2> {
    double x[3], y[3];

    __device__ __forceinline__ void load(const double* __restrict__ nodes, const int32_t* v) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double2 p = __ldg(reinterpret_cast<const double2*>(nodes) + v[k]);
            x[k] = p.x;
            y[k] = p.y;
        }
    }

    // s[i] = s_ij for i = 0..2; returns the unsigned area (0 = degenerate)
    __device__ __forceinline__ double stiffness_col(int j, double s[3]) const {
        // e_i = v[kTriFaces[i][1]] - v[kTriFaces[i][0]]: e0 = v2-v1, e1 = v0-v2, e2 = v1-v0
        const double ex[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
        const double ey[3] = {y[2] - y[1], y[0] - y[2], y[1] - y[0]};
        const double area = 0.5 * fabs(-ex[2] * ey[1] + ey[2] * ex[1]);
        const Recip R = recip(4.0 * area);
        // normals n_i = (-e_iy, e_ix, 0)
        const double njx = (j == 0) ? -ey[0] : (j == 1) ? -ey[1] : -ey[2];
        const double njy = (j == 0) ? ex[0] : (j == 1) ? ex[1] : ex[2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double dot = (-ey[i]) * njx + ex[i] * njy + 0.0 * 0.0;
            s[i] = div_by(dot, R);
        }
        return area;
    }

    // the whole local matrix at once (element-first path): s_ij for all i, j with
    // exactly stiffness_col's operations; the dot product is symmetric in (i, j)
    // operand for operand, so s_ij == s_ji bitwise and only i <= j is computed
    __device__ __forceinline__ double stiffness_all(double s[3][3]) const {
        const double ex[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
        const double ey[3] = {y[2] - y[1], y[0] - y[2], y[1] - y[0]};
        const double area = 0.5 * fabs(-ex[2] * ey[1] + ey[2] * ex[1]);
        const Recip R = recip(4.0 * area);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i <= j; ++i) {
                const double dot = (-ey[i]) * (-ey[j]) + ex[i] * ex[j] + 0.0 * 0.0;
                s[i][j] = s[j][i] = div_by(dot, R);
            }
        return area;
    }

    // system.hpp:83-95: contrib_j = area * (f(mid_{j+1}) + f(mid_{j+2})) / 6
    __device__ __forceinline__ double load_col(int j, int32_t t, const FieldDesc& f,
                                               const Recip& R6) const {
        if (f.kind == FL_FIELD_NONE) return 0.0;
        const double ex1 = x[0] - x[2], ey1 = y[0] - y[2];
        const double ex2 = x[1] - x[0], ey2 = y[1] - y[0];
        const double area = fabs(0.5 * (-ex2 * ey1 + ey2 * ex1));  // mesh.hpp:34-38
        const int i1 = (j + 1) % 3, i2 = (j + 2) % 3;
        double fa, fb;
        if (f.kind == FL_FIELD_SAMPLES) {
            fa = __ldg(f.samples + (size_t)t * 3 + i1);
            fb = __ldg(f.samples + (size_t)t * 3 + i2);
        } else if (f.kind == FL_FIELD_CONST) {
            fa = fb = f.value;
        } else {
            fa = mid_field(i1, f);
            fb = mid_field(i2, f);
        }
        return div_by(area * (fa + fb), R6);
    }

    // mid of face i: kTriFaces = {1,2},{2,0},{0,1}; (va + vb) / 2.0
    __device__ __forceinline__ double mid_field(int i, const FieldDesc& f) const {
        const int a = (i == 0) ? 1 : (i == 1) ? 2 : 0;
        const int b = (i == 0) ? 2 : (i == 1) ? 0 : 1;
        return eval_point(f, (x[a] + x[b]) * 0.5, (y[a] + y[b]) * 0.5, 0.0);
    }

    // SURVEY.md §8 a11 for d = 2: xbar = ((x0 + x1) + x2) / 3
    __device__ __forceinline__ double coef_c5(const Recip& R3) const {
        const double xbar = div_by((x[0] + x[1]) + x[2], R3);
        return 1.0 + 0.5 * sin((2.0 * kPi) * xbar);
    }

    __device__ __forceinline__ double face_share(int lf, const FieldDesc& g, const Recip& R3,
                                                 int32_t t) const {
        // system.hpp:138-148: face lf = {kTriFaces[lf][0], kTriFaces[lf][1]}
        const int a = (lf == 0) ? 1 : (lf == 1) ? 2 : 0;
        const int b = (lf == 0) ? 2 : (lf == 1) ? 0 : 1;
        const double ex = x[b] - x[a], ey = y[b] - y[a];
        const double length = __dsqrt_rn(ex * ex + ey * ey);
        double gv;
        if (g.kind == FL_FIELD_SAMPLES) gv = __ldg(g.samples + (size_t)t * 3 + lf);
        else gv = eval_point(g, (x[a] + x[b]) * 0.5, (y[a] + y[b]) * 0.5, 0.0);
        (void)R3;
        return (length * gv) * 0.5;
    }
};

// ---------------------------------------------------------------------------
// 3-D: assembly.hpp:152-169 (face normals by cross products, volume),
//      assembly.hpp:283-292 (s = n_i.n_j / (36 vol)), system.hpp:97-111 (tet4 load)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cross3(double ux, double uy, double uz, double vx, double vy,
                                       double vz, double& ox, double& oy, double& oz) {
    // assembly.hpp:76-80
    ox = uy * vz - uz * vy;
    oy = uz * vx - ux * vz;
    oz = ux * vy - uy * vx;
}

template <>
struct ElemCol<3> {
    double x[4], y[4], z[4];

    __device__ __forceinline__ void load(const double* __restrict__ nodes, const int32_t* v) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double* p = nodes + (size_t)v[k] * 3;
            x[k] = __ldg(p);
            y[k] = __ldg(p + 1);
            z[k] = __ldg(p + 2);
        }
    }

    // normals of the four faces, kTetFaces = {1,3,2},{0,2,3},{0,3,1},{0,1,2}
    __device__ __forceinline__ void normals(double n[4][3]) const {
        const int f0[4] = {1, 0, 0, 0}, f1[4] = {3, 2, 3, 1}, f2[4] = {2, 3, 1, 2};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double ux = x[f1[i]] - x[f0[i]], uy = y[f1[i]] - y[f0[i]], uz = z[f1[i]] - z[f0[i]];
            const double vx = x[f2[i]] - x[f0[i]], vy = y[f2[i]] - y[f0[i]], vz = z[f2[i]] - z[f0[i]];
            cross3(ux, uy, uz, vx, vy, vz, n[i][0], n[i][1], n[i][2]);
        }
    }

    // |cr . v14| / 6 with cr = n_3 (same inputs as assembly.hpp:166), v14 = v3 - v0
    __device__ __forceinline__ double volume(const double n3[3], const Recip& R6) const {
        const double d = n3[0] * (x[3] - x[0]) + n3[1] * (y[3] - y[0]) + n3[2] * (z[3] - z[0]);
        return div_by(fabs(d), R6);
    }

    __device__ __forceinline__ double stiffness_col(int j, double s[4], const Recip& R6) const {
        double n[4][3];
        normals(n);
        const double vol = volume(n[3], R6);
        const Recip R = recip(36.0 * vol);
        double nj[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            nj[c] = (j == 0) ? n[0][c] : (j == 1) ? n[1][c] : (j == 2) ? n[2][c] : n[3][c];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double dot = n[i][0] * nj[0] + n[i][1] * nj[1] + n[i][2] * nj[2];
            s[i] = div_by(dot, R);
        }
        return vol;
    }

    // the whole local matrix at once (element-first path), stiffness_col's
    // operations; n_i . n_j is symmetric operand for operand (s_ij == s_ji)
    __device__ __forceinline__ double stiffness_all(double s[4][4], const Recip& R6) const {
        double n[4][3];
        normals(n);
        const double vol = volume(n[3], R6);
        const Recip R = recip(36.0 * vol);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i <= j; ++i) {
                const double dot = n[i][0] * n[j][0] + n[i][1] * n[j][1] + n[i][2] * n[j][2];
                s[i][j] = s[j][i] = div_by(dot, R);
            }
        return vol;
    }

    // load_col for every j at once: the quadrature weights w_q are shared
    __device__ __forceinline__ void load_all(int32_t t, double vol, const FieldDesc& f,
                                             double out[4]) const {
        double w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double fx;
            if (f.kind == FL_FIELD_SAMPLES) {
                fx = __ldg(f.samples + (size_t)t * 4 + q);
            } else if (f.kind == FL_FIELD_CONST) {
                fx = f.value;
            } else {
                double px = 0.0, py = 0.0, pz = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double lam = (k == q) ? kTet4A : kTet4B;
                    px += lam * x[k];
                    py += lam * y[k];
                    pz += lam * z[k];
                }
                fx = eval_point(f, px, py, pz);
            }
            w[q] = vol * 0.25 * fx;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc += w[q] * ((q == j) ? kTet4A : kTet4B);
            out[j] = f.kind == FL_FIELD_NONE ? 0.0 : acc;
        }
    }

    // system.hpp:97-111: w_q = vol * 0.25 * f(x_q); contrib_j = sum_q w_q * lambda_qj
    __device__ __forceinline__ double load_col(int j, int32_t t, double vol,
                                               const FieldDesc& f) const {
        if (f.kind == FL_FIELD_NONE) return 0.0;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double fx;
            if (f.kind == FL_FIELD_SAMPLES) {
                fx = __ldg(f.samples + (size_t)t * 4 + q);
            } else if (f.kind == FL_FIELD_CONST) {
                fx = f.value;
            } else {
                double px = 0.0, py = 0.0, pz = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double lam = (k == q) ? kTet4A : kTet4B;
                    px += lam * x[k];
                    py += lam * y[k];
                    pz += lam * z[k];
                }
                fx = eval_point(f, px, py, pz);
            }
            const double w = vol * 0.25 * fx;
            acc += w * ((q == j) ? kTet4A : kTet4B);
        }
        return acc;
    }

    // xbar = (((x0 + x1) + x2) + x3) / 4
    __device__ __forceinline__ double coef_c5(const Recip&) const {
        const double xbar = (((x[0] + x[1]) + x[2]) + x[3]) * 0.25;
        return 1.0 + 0.5 * sin((2.0 * kPi) * xbar);
    }

    // system.hpp:149-166: area * g(barycentre) / 3 for face lf
    __device__ __forceinline__ double face_share(int lf, const FieldDesc& g, const Recip& R3,
                                                 int32_t t) const {
        const int f0 = (lf == 0) ? 1 : 0;
        const int f1 = (lf == 0) ? 3 : (lf == 1) ? 2 : (lf == 2) ? 3 : 1;
        const int f2 = (lf == 0) ? 2 : (lf == 1) ? 3 : (lf == 2) ? 1 : 2;
        double cx, cy, cz;
        cross3(x[f1] - x[f0], y[f1] - y[f0], z[f1] - z[f0], x[f2] - x[f0], y[f2] - y[f0],
               z[f2] - z[f0], cx, cy, cz);
        const double area = 0.5 * __dsqrt_rn(cx * cx + cy * cy + cz * cz);
        double gv;
        if (g.kind == FL_FIELD_SAMPLES) {
            gv = __ldg(g.samples + (size_t)t * 4 + lf);
        } else {
            const double bx = div_by(x[f0] + x[f1] + x[f2], R3);
            const double by = div_by(y[f0] + y[f1] + y[f2], R3);
            const double bz = div_by(z[f0] + z[f1] + z[f2], R3);
            gv = eval_point(g, bx, by, bz);
        }
        return div_by(area * gv, R3);
    }
};

}  // namespace fl
