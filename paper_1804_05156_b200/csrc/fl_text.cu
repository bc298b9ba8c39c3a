// fl_text.cu -- the reference's text writers on the GPU.
//
//   write_matrix_market(CscMatrix, ostream)   matrix_market.hpp:15-24
//       "%%MatrixMarket matrix coordinate real general\n", "m n nnz\n", then per
//       column c ascending, per stored entry k: "<row+1> <c+1> <%.17g value>\n"
//   write_mesh(Mesh, ostream)                 mesh_io.hpp:125-142
//       "d N NT\n", N lines of d coordinates (detail::format_real = "%.17g",
//       mesh_io.hpp:56-60), NT lines of d+1 one-based vertex ids, NT lines of
//       d+1 flags (int), single spaces between fields
//
// %.17g is glibc's: the value rounded to 17 significant decimal digits with
// exact (correctly rounded, ties-to-even) arithmetic, then C's %g style rules
// (f style when -4 <= X < 17 else e style with a sign and >= 2 exponent digits,
// trailing zeros and a bare point removed; "inf", "nan" with sign).  Exact on
// the device:
//   fast path   N = round(|v| * 10^(16-X)) from the 181-bit product of the
//               53-bit significand and a 128-bit truncated 10^k (fl_pow10.cuh,
//               tools/gen_pow10.py).  The truncation error is below the
//               significand m (< 2^53) in units of the product, so the rounding
//               decision is certain unless the remainder lies within m of one
//               half; when 10^k is exact in 128 bits (0 <= k <= 55) it is exact;
//   exact path  otherwise a big-integer comparison of 2|v|10^k against 2N+1
//               (<= 16 64-bit limbs) decides, ties to even.
// Lines are formatted by one thread each (two per thread), measured, placed by
// a block scan into shared memory and stored coalesced at the tile's offset from
// a decoupled look-back over tiles: one pass, one write of every output byte.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "fl_internal.cuh"
#include "fl_pow10.cuh"
#include "fl_scan.cuh"

struct fl_text {
    fl_ctx* ctx = nullptr;
    fl::DevBuf buf;     // the text
    fl::DevBuf total;   // int64: bytes of text (device)
    fl::DevBuf ws;      // look-back status + tickets
    fl::DevBuf stage[3];
    int64_t bytes = -1;  // host copy after fl_text_size
};

namespace fl {

// ---------------------------------------------------------------------------
// %.17g
// ---------------------------------------------------------------------------
enum : int { G_NUM = 0, G_ZERO = 1, G_INF = 2, G_NAN = 3 };

struct G17 {
    uint32_t h, l;  // the 17 significant digits: h = first 9, l = last 8
    int32_t x;      // decimal exponent of the first digit
    int16_t nd;     // significant digits left after stripping trailing zeros (1..17)
    int8_t kind;  // G_*
    int8_t neg;
};

struct Big {  // little-endian 64-bit limbs
    static constexpr int L = 16;
    uint64_t w[L];
    __device__ void set(uint64_t v) {
        w[0] = v;
#pragma unroll
        for (int i = 1; i < L; ++i) w[i] = 0;
    }
    __device__ void mul(uint64_t f) {
        uint64_t carry = 0;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            const uint64_t lo = w[i] * f;
            const uint64_t hi = __umul64hi(w[i], f);
            const uint64_t s = lo + carry;
            carry = hi + (s < lo);
            w[i] = s;
        }
    }
    __device__ void mul_pow5(int a) {
        constexpr uint64_t P27 = 7450580596923828125ull;  // 5^27
        for (; a >= 27; a -= 27) mul(P27);
        uint64_t f = 1;
        for (; a > 0; --a) f *= 5;
        mul(f);
    }
    __device__ void shl(int d) {
        const int ws = d >> 6, bs = d & 63;
        for (int i = L - 1; i >= 0; --i) {
            const int s = i - ws;
            uint64_t v = 0;
            if (s >= 0) {
                v = w[s] << bs;
                if (bs && s > 0) v |= w[s - 1] >> (64 - bs);
            }
            w[i] = v;
        }
    }
};

__device__ int big_cmp(const Big& a, const Big& b) {
    for (int i = Big::L - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

// sign of 2|v|10^k - b, |v| = m * 2^e  (exact)
__device__ __noinline__ int exact_cmp2(uint64_t m, int e, int k, uint64_t b) {
    Big l, r;
    l.set(m);
    r.set(b);
    if (k >= 0) l.mul_pow5(k);
    else r.mul_pow5(-k);
    const int d = e + 1 + k;  // 2|v|10^k = m 5^k 2^(e+1+k)
    if (d >= 0) l.shl(d);
    else r.shl(-d);
    return big_cmp(l, r);
}
// sign of |v| * 10^k - (nf + 1/2)
__device__ __forceinline__ int exact_vs_half(uint64_t m, int e, int k, uint64_t nf) {
    return exact_cmp2(m, e, k, 2 * nf + 1);
}

struct U192 {
    uint64_t w0, w1, w2;
};

__device__ __forceinline__ uint64_t bits64_at(const U192& p, int s) {  // (p >> s) mod 2^64
    const uint64_t w[4] = {p.w0, p.w1, p.w2, 0};
    const int i = s >> 6, b = s & 63;
    uint64_t v = w[i] >> b;
    if (b) v |= w[i + 1] << (64 - b);
    return v;
}
__device__ __forceinline__ bool bit_at(const U192& p, int s) {
    const uint64_t w = s < 64 ? p.w0 : s < 128 ? p.w1 : p.w2;
    return (w >> (s & 63)) & 1;
}
__device__ __forceinline__ U192 low_bits(const U192& p, int s) {  // p mod 2^s, 0 <= s < 192
    U192 r = p;
    if (s < 64) {
        r.w0 &= s ? (~0ull >> (64 - s)) : 0;
        r.w1 = r.w2 = 0;
    } else if (s < 128) {
        r.w1 &= (s - 64) ? (~0ull >> (128 - s)) : 0;
        r.w2 = 0;
    } else {
        r.w2 &= (s - 128) ? (~0ull >> (192 - s)) : 0;
    }
    return r;
}
__device__ __forceinline__ bool is_zero(const U192& p) { return (p.w0 | p.w1 | p.w2) == 0; }

// N = |v| * 10^k rounded to nearest, ties to even; requires the result < 2^64.
// nf_out: floor of the truncated product (the true floor, or one less when the
// true value sits within m / 2^s below the next integer)
__device__ uint64_t scaled_round(uint64_t m, int e, int k, bool force_exact, uint64_t& nf_out) {
    const Pow10 P = kPow10[k - kPow10Min];
    U192 p;
    {
        const uint64_t a0 = P.lo * m, a1 = __umul64hi(P.lo, m);
        const uint64_t b0 = P.hi * m, b1 = __umul64hi(P.hi, m);
        p.w0 = a0;
        p.w1 = a1 + b0;
        p.w2 = b1 + (p.w1 < a1);
    }
    const int s = -(e + P.q);  // value = p / 2^s (+ error < m / 2^s when inexact)
    const uint64_t nf = bits64_at(p, s);
    nf_out = nf;
    const bool half_bit = bit_at(p, s - 1);
    const U192 below = low_bits(p, s - 1);
    if (P.exact && !force_exact) {
        if (!half_bit) return nf;
        if (!is_zero(below)) return nf + 1;
        return nf + (nf & 1);  // exact tie
    }
    if (!force_exact) {
        if (half_bit) return nf + 1;  // true remainder >= computed > ... >= half, and > half
        // remainder + m <= half: the true remainder is below one half
        U192 t = below;
        t.w0 += m;
        const uint64_t c0 = t.w0 < m;
        t.w1 += c0;
        t.w2 += (c0 && t.w1 == 0);
        if (!bit_at(t, s - 1) || is_zero(low_bits(t, s - 1))) return nf;
    }
    // exact decision: |v|10^k lies in [nf, nf + 1 + m/2^s); compare it with
    // nf + 1/2 and, above that, with nf + 3/2
    const int c = exact_vs_half(m, e, k, nf);
    if (c < 0) return nf;
    if (c == 0) return nf + (nf & 1);
    const int c2 = exact_vs_half(m, e, k, nf + 1);
    if (c2 < 0) return nf + 1;
    if (c2 == 0) return (nf + 1) + ((nf + 1) & 1);
    return nf + 2;
}

__device__ G17 g17(double v, bool force_exact) {
    G17 g;
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    g.neg = (int8_t)(bits >> 63);
    const int eb = (int)((bits >> 52) & 0x7ff);
    const uint64_t frac = bits & ((1ull << 52) - 1);
    g.h = g.l = 0;
    g.x = 0;
    g.nd = 1;
    if (eb == 0x7ff) {
        g.kind = frac ? G_NAN : G_INF;
        return g;
    }
    if (eb == 0 && frac == 0) {
        g.kind = G_ZERO;
        return g;
    }
    g.kind = G_NUM;
    const uint64_t m = eb ? (frac | (1ull << 52)) : frac;
    const int e = eb ? eb - 1075 : -1074;
    // floor(log10 |v|) or one less: floor((bit length - 1 + e) log10 2)
    int x = ((63 - __clzll((long long)m) + e) * 1262611) >> 22;
    constexpr uint64_t E16 = 10000000000000000ull, E17 = 100000000000000000ull;
    uint64_t n = 0;
    // X is right when 10^16 <= |v| 10^(16-X) < 10^17 for the TRUE value (before
    // rounding); a rounding carry to 10^17 then moves to the next decade
    for (int guard = 0; guard < 4; ++guard) {
        uint64_t nf;
        n = scaled_round(m, e, 16 - x, force_exact, nf);
        if (nf >= E17) {
            x += 1;
            continue;
        }
        if (nf < E16 && !(nf == E16 - 1 && exact_cmp2(m, e, 16 - x, 2 * E16) >= 0)) {
            x -= 1;
            continue;
        }
        if (n == E17) {
            n = E16;
            x += 1;
        }
        break;
    }
    const uint32_t h = (uint32_t)(n / 100000000ull);
    const uint32_t l = (uint32_t)(n - (uint64_t)h * 100000000ull);
    int nd = 17;
    uint32_t t = l;
    if (t == 0) {
        nd = 9;
        t = h;
    }
    while (t % 10 == 0) {
        t /= 10;
        --nd;
    }
    g.h = h;
    g.l = l;
    g.x = x;
    g.nd = (int16_t)nd;
    return g;
}

__device__ __forceinline__ int g17_len(const G17& g) {
    int len = g.neg;
    if (g.kind == G_ZERO) return len + 1;
    if (g.kind != G_NUM) return len + 3;
    const int x = g.x, nd = g.nd;
    if (x >= -4 && x < 17) {
        if (x >= 0) len += (x + 1) + (nd > x + 1 ? 1 + nd - (x + 1) : 0);
        else len += 2 + (-x - 1) + nd;
    } else {
        len += (nd > 1 ? nd + 1 : 1) + 2 + ((x >= 100 || x <= -100) ? 3 : 2);
    }
    return len;
}

__device__ __forceinline__ int g17_emit(const G17& g, char* d) {
    char* p = d;
    if (g.neg) *p++ = '-';
    if (g.kind == G_ZERO) {
        *p++ = '0';
        return (int)(p - d);
    }
    if (g.kind == G_INF || g.kind == G_NAN) {
        const char* s = g.kind == G_INF ? "inf" : "nan";
        p[0] = s[0];
        p[1] = s[1];
        p[2] = s[2];
        return (int)(p + 3 - d);
    }
    char dg[17];
    {
        uint32_t a = g.h, b = g.l;
#pragma unroll
        for (int i = 16; i >= 9; --i) {
            dg[i] = (char)('0' + b % 10);
            b /= 10;
        }
#pragma unroll
        for (int i = 8; i >= 0; --i) {
            dg[i] = (char)('0' + a % 10);
            a /= 10;
        }
    }
    const int x = g.x, nd = g.nd;
    if (x >= -4 && x < 17) {
        if (x >= 0) {
            for (int i = 0; i <= x; ++i) *p++ = i < nd ? dg[i] : '0';
            if (nd > x + 1) {
                *p++ = '.';
                for (int i = x + 1; i < nd; ++i) *p++ = dg[i];
            }
        } else {
            *p++ = '0';
            *p++ = '.';
            for (int i = 0; i < -x - 1; ++i) *p++ = '0';
            for (int i = 0; i < nd; ++i) *p++ = dg[i];
        }
    } else {
        *p++ = dg[0];
        if (nd > 1) {
            *p++ = '.';
            for (int i = 1; i < nd; ++i) *p++ = dg[i];
        }
        *p++ = 'e';
        int ax = x;
        if (x < 0) {
            *p++ = '-';
            ax = -x;
        } else {
            *p++ = '+';
        }
        if (ax >= 100) {
            *p++ = (char)('0' + ax / 100);
            ax %= 100;
        }
        *p++ = (char)('0' + ax / 10);
        *p++ = (char)('0' + ax % 10);
    }
    return (int)(p - d);
}

// signed decimal integer (operator<< on an int / long long)
__device__ __forceinline__ int int_len(int64_t v) {
    int len = v < 0 ? 1 : 0;
    uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    int nd = 1;
    while (u >= 10) {
        u /= 10;
        ++nd;
    }
    return len + nd;
}
__device__ __forceinline__ int int_emit(int64_t v, char* d) {
    char* p = d;
    uint64_t u = (uint64_t)v;
    if (v < 0) {
        *p++ = '-';
        u = (uint64_t)(-(v + 1)) + 1;
    }
    int nd = 1;
    for (uint64_t t = u; t >= 10; t /= 10) ++nd;
    for (int i = nd - 1; i >= 0; --i) {
        p[i] = (char)('0' + u % 10);
        u /= 10;
    }
    return (int)(p + nd - d);
}

// ---------------------------------------------------------------------------
// line sources
// ---------------------------------------------------------------------------
constexpr int kTextBlock = 256, kTextLPT = 2, kTextTile = kTextBlock * kTextLPT;
constexpr int kColWin = 1024;  // CSC columns one tile can stage

// "%.17g\n" per value (test / format_real)
struct RealsSrc {
    static constexpr int MAXLINE = 25;
    const double* v;
    bool force_exact;
    struct Line {
        G17 g;
    };
    __device__ void setup(int64_t, int, int32_t*) const {}
    __device__ Line get(int64_t i, const int32_t*) const { return {g17(v[i], force_exact)}; }
    __device__ int len(const Line& l) const { return g17_len(l.g) + 1; }
    __device__ void emit(const Line& l, char* d) const {
        const int n = g17_emit(l.g, d);
        d[n] = '\n';
    }
};

// "<row+1> <col+1> <%.17g>\n" over the CSC entries in column order
struct MatrixMarketSrc {
    static constexpr int MAXLINE = 11 + 11 + 25;
    const int32_t* col_ptr;
    const int32_t* row_idx;
    const double* values;
    int32_t n;
    struct Line {
        G17 g;
        int32_t r, c;
    };
    // the tile's first column and, when the tile spans at most kColWin columns,
    // their col_ptr in shared memory: aux[0] = c0, aux[1] = count, aux[2..]
    __device__ void setup(int64_t k0, int cnt, int32_t* aux) const {
        if (threadIdx.x == 0) {
            // last column with col_ptr[c] <= k (columns may be empty)
            auto find = [&](int64_t k) {
                int32_t lo = 0, hi = n - 1;
                while (lo < hi) {
                    const int32_t mid = (int32_t)(((int64_t)lo + hi + 1) >> 1);
                    if ((int64_t)__ldg(col_ptr + mid) <= k) lo = mid;
                    else hi = mid - 1;
                }
                return lo;
            };
            const int32_t c0 = find(k0), c1 = find(k0 + cnt - 1);
            aux[0] = c0;
            aux[1] = c1 - c0 + 2 <= kColWin ? c1 - c0 + 2 : -(c1 - c0 + 1);
        }
        __syncthreads();
        const int32_t c0 = aux[0], w = aux[1];
        for (int i = threadIdx.x; i < w; i += blockDim.x) aux[2 + i] = __ldg(col_ptr + c0 + i);
        __syncthreads();
    }
    __device__ Line get(int64_t k, const int32_t* aux) const {
        const int32_t c0 = aux[0], w = aux[1];
        int32_t c;
        if (w > 0) {
            int lo = 0, hi = w - 2;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int64_t)aux[2 + mid] <= k) lo = mid;
                else hi = mid - 1;
            }
            c = c0 + lo;
        } else {
            int32_t lo = c0, hi = c0 - w;
            while (lo < hi) {
                const int32_t mid = (int32_t)(((int64_t)lo + hi + 1) >> 1);
                if ((int64_t)__ldg(col_ptr + mid) <= k) lo = mid;
                else hi = mid - 1;
            }
            c = lo;
        }
        return {g17(__ldg(values + k), false), __ldg(row_idx + k), c};
    }
    __device__ int len(const Line& l) const {
        return int_len((int64_t)l.r + 1) + 1 + int_len((int64_t)l.c + 1) + 1 + g17_len(l.g) + 1;
    }
    __device__ void emit(const Line& l, char* d) const {
        char* p = d;
        p += int_emit((int64_t)l.r + 1, p);
        *p++ = ' ';
        p += int_emit((int64_t)l.c + 1, p);
        *p++ = ' ';
        p += g17_emit(l.g, p);
        *p = '\n';
    }
};

// write_mesh node lines: d coordinates
template <int D>
struct NodeSrc {
    static constexpr int MAXLINE = 25 * D;
    const double* nodes;
    struct Line {
        G17 g[D];
    };
    __device__ void setup(int64_t, int, int32_t*) const {}
    __device__ Line get(int64_t k, const int32_t*) const {
        Line l;
#pragma unroll
        for (int c = 0; c < D; ++c) l.g[c] = g17(__ldg(nodes + k * D + c), false);
        return l;
    }
    __device__ int len(const Line& l) const {
        int s = D;  // D - 1 spaces + '\n'
#pragma unroll
        for (int c = 0; c < D; ++c) s += g17_len(l.g[c]);
        return s;
    }
    __device__ void emit(const Line& l, char* d) const {
        char* p = d;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            if (c) *p++ = ' ';
            p += g17_emit(l.g[c], p);
        }
        *p = '\n';
    }
};

// write_mesh element lines (one-based ids) or flag lines (int)
template <int NV, bool FLAGS>
struct IntRowSrc {
    static constexpr int MAXLINE = 12 * NV;
    const int32_t* elems;
    const int8_t* flags;
    struct Line {
        int32_t v[NV];
    };
    __device__ void setup(int64_t, int, int32_t*) const {}
    __device__ Line get(int64_t t, const int32_t*) const {
        Line l;
#pragma unroll
        for (int c = 0; c < NV; ++c)
            l.v[c] = FLAGS ? (flags ? (int32_t)flags[t * NV + c] : 0) : __ldg(elems + t * NV + c) + 1;
        return l;
    }
    __device__ int len(const Line& l) const {
        int s = NV;
#pragma unroll
        for (int c = 0; c < NV; ++c) s += int_len(l.v[c]);
        return s;
    }
    __device__ void emit(const Line& l, char* d) const {
        char* p = d;
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            if (c) *p++ = ' ';
            p += int_emit(l.v[c], p);
        }
        *p = '\n';
    }
};

// ---------------------------------------------------------------------------
// the text kernel: one tile = kTextTile consecutive lines
// ---------------------------------------------------------------------------
template <class Src>
__global__ void __launch_bounds__(kTextBlock) k_text(Src src, int64_t n_lines, char* __restrict__ out,
                                                     const int64_t* __restrict__ base,
                                                     uint64_t* status, unsigned* ticket,
                                                     int64_t* __restrict__ total_out) {
    __shared__ __align__(16) char text[kTextTile * Src::MAXLINE + 16];
    __shared__ int32_t aux[2 + kColWin];
    __shared__ int64_t warp_sums[kTextBlock / 32];
    __shared__ int64_t s_tile, s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t k0 = tile * kTextTile;
    const int cnt = (int)min((int64_t)kTextTile, n_lines - k0);
    src.setup(k0, cnt, aux);
    typename Src::Line ln[kTextLPT];
    int lens[kTextLPT];
    int64_t mine = 0;
#pragma unroll
    for (int r = 0; r < kTextLPT; ++r) {
        const int q = threadIdx.x * kTextLPT + r;
        lens[r] = 0;
        if (q < cnt) {
            ln[r] = src.get(k0 + q, aux);
            lens[r] = src.len(ln[r]);
        }
        mine += lens[r];
    }
    int64_t total;
    int64_t off = block_exclusive_sum<kTextBlock>(mine, warp_sums, total);
#pragma unroll
    for (int r = 0; r < kTextLPT; ++r) {
        if (lens[r]) src.emit(ln[r], text + off);
        off += lens[r];
    }
    if (threadIdx.x < 32) {
        const uint64_t e = warp_lookback(status, tile, (uint64_t)total);
        if (threadIdx.x == 0) s_excl = (int64_t)e;
    }
    __syncthreads();
    const int64_t start = *base + s_excl;
    if (k0 + cnt == n_lines && threadIdx.x == 0) *total_out = start + total;
    // coalesced store: head bytes up to 4-byte alignment, aligned words assembled
    // from the shared text with funnel shifts, tail bytes
    char* dst = out + start;
    const int T = (int)total;
    const int head = min((int)((4 - ((uintptr_t)dst & 3)) & 3), T);
    if ((int)threadIdx.x < head) dst[threadIdx.x] = text[threadIdx.x];
    const int nw = (T - head) >> 2;
    const uint32_t* t32 = reinterpret_cast<const uint32_t*>(text);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
    const int sh = (head & 3) * 8;
    for (int w = threadIdx.x; w < nw; w += kTextBlock) {
        const int si = (head >> 2) + w;
        const uint32_t lo = t32[si], hi = t32[si + 1];
        d32[w] = sh ? __funnelshift_r(lo, hi, sh) : lo;
    }
    const int tail0 = head + nw * 4;
    if ((int)threadIdx.x < T - tail0) dst[tail0 + threadIdx.x] = text[tail0 + threadIdx.x];
}

template <class Src>
static int launch_text(fl_ctx* ctx, fl_text* tx, const Src& src, int64_t n_lines, const int64_t* base,
                       int64_t* total_out, size_t ws_off) {
    if (n_lines <= 0) {
        FL_CUDA(cudaMemcpyAsync(total_out, base, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        return FL_OK;
    }
    const int64_t tiles = (n_lines + kTextTile - 1) / kTextTile;
    uint64_t* status = reinterpret_cast<uint64_t*>(tx->ws.as<char>() + ws_off);
    unsigned* ticket = reinterpret_cast<unsigned*>(status + tiles + 1);
    FL_CUDA(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (size_t)(tiles + 2), ctx->stream));
    k_text<Src><<<(unsigned)tiles, kTextBlock, 0, ctx->stream>>>(src, n_lines, tx->buf.as<char>(), base,
                                                                  status, ticket, total_out);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

static size_t ws_bytes(int64_t n_lines) {
    const int64_t tiles = (n_lines + kTextTile - 1) / kTextTile;
    return sizeof(uint64_t) * (size_t)(tiles + 2) + 64;
}

// header written on the host into the front of the device buffer; the kernels
// start at its length (device word `base`)
static int put_header(fl_ctx* ctx, fl_text* tx, const std::string& h, size_t body_bound, int sections) {
    FL_TRY(tx->buf.ensure(h.size() + body_bound + 16));
    FL_TRY(tx->total.ensure(sizeof(int64_t) * (size_t)(sections + 1)));
    // pageable sources: the copies have consumed them when the calls return
    const int64_t hl = (int64_t)h.size();
    if (hl > 0)
        FL_CUDA(cudaMemcpyAsync(tx->buf.p, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
    FL_CUDA(cudaMemcpyAsync(tx->total.p, &hl, sizeof hl, cudaMemcpyHostToDevice, ctx->stream));
    tx->bytes = -1;
    return FL_OK;
}

static int stage_in(fl_ctx* ctx, fl::DevBuf& b, const void* src, size_t bytes, int mem, const void** out) {
    if (mem == FL_MEM_DEVICE || bytes == 0) {
        *out = src;
        return FL_OK;
    }
    FL_TRY(b.ensure(bytes));
    FL_CUDA(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *out = b.p;
    return FL_OK;
}

}  // namespace fl

using namespace fl;

extern "C" {

FL_API int fl_text_create(fl_ctx* ctx, fl_text** out) {
    if (!ctx || !out) return set_error(FL_ERR_ARGUMENT, "null argument");
    *out = new fl_text();
    (*out)->ctx = ctx;
    return FL_OK;
}

FL_API int fl_text_destroy(fl_text* tx) {
    if (!tx) return FL_OK;
    cudaSetDevice(tx->ctx->device);
    cudaStreamSynchronize(tx->ctx->stream);
    tx->buf.release();
    tx->total.release();
    tx->ws.release();
    for (auto& s : tx->stage) s.release();
    delete tx;
    return FL_OK;
}

FL_API int fl_text_size(fl_text* tx, int64_t* bytes) {
    if (!tx || !bytes) return set_error(FL_ERR_ARGUMENT, "null argument");
    if (tx->bytes < 0) {
        fl_ctx* ctx = tx->ctx;
        FL_CUDA(cudaSetDevice(ctx->device));
        int64_t* h = reinterpret_cast<int64_t*>(static_cast<char*>(ctx->pinned) + 2048);
        FL_CUDA(cudaMemcpyAsync(h, tx->total.p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        FL_CUDA(cudaStreamSynchronize(ctx->stream));
        tx->bytes = *h;
    }
    *bytes = tx->bytes;
    return FL_OK;
}

FL_API int fl_text_copy(fl_text* tx, char* dst, int64_t capacity, int mem) {
    int64_t n = 0;
    FL_TRY(fl_text_size(tx, &n));
    if (!dst && n > 0) return set_error(FL_ERR_ARGUMENT, "null destination");
    if (capacity < n) return set_error(FL_ERR_ARGUMENT, "destination smaller than the text");
    fl_ctx* ctx = tx->ctx;
    if (n > 0) {
        FL_CUDA(cudaMemcpyAsync(dst, tx->buf.p, (size_t)n,
                                mem == FL_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                ctx->stream));
        FL_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return FL_OK;
}

FL_API int fl_text_device_ptr(fl_text* tx, const char** ptr, int64_t* bytes) {
    if (!ptr) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_TRY(fl_text_size(tx, bytes));
    *ptr = tx->buf.as<const char>();
    return FL_OK;
}

FL_API int fl_format_reals(fl_ctx* ctx, int64_t n, const double* v, int mem, uint32_t flags,
                           fl_text* out) {
    if (!ctx || !out || n < 0 || (n > 0 && !v)) return set_error(FL_ERR_ARGUMENT, "bad argument");
    FL_CUDA(cudaSetDevice(ctx->device));
    const void* dv = nullptr;
    FL_TRY(stage_in(ctx, out->stage[0], v, sizeof(double) * (size_t)n, mem, &dv));
    FL_TRY(put_header(ctx, out, std::string(), (size_t)n * RealsSrc::MAXLINE, 1));
    FL_TRY(out->ws.ensure(ws_bytes(n)));
    RealsSrc src{static_cast<const double*>(dv), (flags & 1u) != 0};
    int64_t* tot = out->total.as<int64_t>();
    FL_TRY(launch_text(ctx, out, src, n, tot, tot + 1, 0));
    FL_CUDA(cudaMemcpyAsync(tot, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    return FL_OK;
}

FL_API int fl_write_matrix_market(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr,
                                  const int32_t* row_idx, const double* values, int mem,
                                  fl_text* out) {
    if (!ctx || !out || !col_ptr || m < 0 || n < 0) return set_error(FL_ERR_ARGUMENT, "bad argument");
    FL_CUDA(cudaSetDevice(ctx->device));
    int32_t nnz = 0;
    if (mem == FL_MEM_DEVICE) {
        FL_CUDA(cudaMemcpyAsync(ctx->pinned, col_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                ctx->stream));
        FL_CUDA(cudaStreamSynchronize(ctx->stream));
        std::memcpy(&nnz, ctx->pinned, sizeof nnz);
    } else {
        nnz = col_ptr[n];
    }
    if (nnz < 0) return set_error(FL_E_SHAPE_MISMATCH, "col_ptr[n] < 0");
    if (nnz > 0 && (!row_idx || !values)) return set_error(FL_ERR_ARGUMENT, "null entries");
    const void *dc = nullptr, *dr = nullptr, *dv = nullptr;
    FL_TRY(stage_in(ctx, out->stage[0], col_ptr, sizeof(int32_t) * ((size_t)n + 1), mem, &dc));
    FL_TRY(stage_in(ctx, out->stage[1], row_idx, sizeof(int32_t) * (size_t)nnz, mem, &dr));
    FL_TRY(stage_in(ctx, out->stage[2], values, sizeof(double) * (size_t)nnz, mem, &dv));
    // write_matrix_market's header (matrix_market.hpp:16-17)
    const std::string h = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(m) + " " +
                          std::to_string(n) + " " + std::to_string(nnz) + "\n";
    FL_TRY(put_header(ctx, out, h, (size_t)nnz * MatrixMarketSrc::MAXLINE, 1));
    FL_TRY(out->ws.ensure(ws_bytes(nnz)));
    MatrixMarketSrc src{static_cast<const int32_t*>(dc), static_cast<const int32_t*>(dr),
                        static_cast<const double*>(dv), n};
    int64_t* tot = out->total.as<int64_t>();
    if (n == 0) return launch_text(ctx, out, src, 0, tot, tot, 0);
    FL_TRY(launch_text(ctx, out, src, nnz, tot, tot + 1, 0));
    FL_CUDA(cudaMemcpyAsync(tot, tot + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    return FL_OK;
}

FL_API int fl_write_mesh(fl_ctx* ctx, fl_mesh* mesh, fl_text* out) {
    if (!ctx || !mesh || !out) return set_error(FL_ERR_ARGUMENT, "null argument");
    FL_CUDA(cudaSetDevice(ctx->device));
    const int d = mesh->dim, nv = d + 1;
    const int64_t N = mesh->n_nodes, NT = mesh->n_elems;
    const std::string h = std::to_string(d) + " " + std::to_string(N) + " " + std::to_string(NT) + "\n";
    const size_t bound = (size_t)N * 25 * d + (size_t)NT * 12 * nv * 2;
    FL_TRY(put_header(ctx, out, h, bound, 3));
    const size_t w1 = ws_bytes(N), w2 = ws_bytes(NT);
    FL_TRY(out->ws.ensure(w1 + 2 * w2 + 64));
    int64_t* tot = out->total.as<int64_t>();  // [0] running end, [1..3] section ends
    const double* nodes = mesh->nodes.as<double>();
    const int32_t* elems = mesh->elems.as<int32_t>();
    const int8_t* flags = mesh->has_flags ? mesh->flags.as<int8_t>() : nullptr;
    // sections in order: nodes, elements, flags (mesh_io.hpp:127-141)
    if (d == 2) {
        FL_TRY(launch_text(ctx, out, NodeSrc<2>{nodes}, N, tot, tot + 1, 0));
        FL_TRY(launch_text(ctx, out, IntRowSrc<3, false>{elems, nullptr}, NT, tot + 1, tot + 2, w1));
        FL_TRY(launch_text(ctx, out, IntRowSrc<3, true>{nullptr, flags}, NT, tot + 2, tot + 3, w1 + w2));
    } else {
        FL_TRY(launch_text(ctx, out, NodeSrc<3>{nodes}, N, tot, tot + 1, 0));
        FL_TRY(launch_text(ctx, out, IntRowSrc<4, false>{elems, nullptr}, NT, tot + 1, tot + 2, w1));
        FL_TRY(launch_text(ctx, out, IntRowSrc<4, true>{nullptr, flags}, NT, tot + 2, tot + 3, w1 + w2));
    }
    FL_CUDA(cudaMemcpyAsync(tot, tot + 3, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    return FL_OK;
}

}  // extern "C"
