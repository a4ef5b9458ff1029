// apo_device.cuh -- APO ("all-pairs offers" without the mean stream) device helpers
// shared by the two merge-loop kernels (hseg_kernels.cu: the generic loop, which
// still carries the first APO variant; apo_loop.cu: the APO loop proper).
//
// Reference semantics: every value these helpers bound or evaluate is the
// reference's fp64 sqrt-BSMSE (dissim.py:33-42, _kernels.py:31-115 op order).
#pragma once

#include "rhseg_device.cuh"

namespace rhseg {

// D entries: an exact value is a non-negative double (sign bit clear); an interval
// (APO sections only, see the APO section below) is [sign=1 | centre c with its low 6
// mantissa bits replaced by k] = c (1 -/+ 2^(k-46)).
constexpr double kU64 = 1.1102230246251565e-16;
constexpr int kApoKMax = 45;  // widest encodable interval: c (1 -/+ 1/2)
__device__ __forceinline__ bool d_is_interval(double v) { return __double_as_longlong(v) < 0; }
__device__ __forceinline__ void d_decode(double c, int k, double& lo, double& hi) {
    const double rho = __longlong_as_double((long long)(k - 46 + 1023) << 52);
    lo = __dmul_rd(c, 1.0 - rho);  // 1 -/+ rho are exact for 2^-46 <= rho <= 1/2
    hi = __dmul_ru(c, 1.0 + rho);
}
__device__ __forceinline__ void d_unpack(double v, double& lo, double& hi) {
    const long long b = __double_as_longlong(v);
    if (b < 0) d_decode(__longlong_as_double(b & 0x7fffffffffffffc0LL), (int)(b & 63), lo, hi);
    else lo = hi = v;
}
// encode [lo, hi] (0 < lo <= hi < inf); false when the interval is too wide to encode
__device__ __forceinline__ bool d_pack_interval(double lo, double hi, double& out) {
    if (lo == hi) { out = lo; return true; }
    if (!(lo > 0.0) || !(hi < kInf)) return false;
    const long long cb = __double_as_longlong(0.5 * lo + 0.5 * hi) & 0x7fffffffffffffc0LL;
    const double c = __longlong_as_double(cb);  // truncated centre
    // first guess from the exponents of the half-width and the centre, then verify
    // with the decoder itself (rarely more than one extra iteration)
    const double w = fmax(hi - c, c - lo);
    const int ew = (int)((__double_as_longlong(w) >> 52) & 0x7ff), ec = (int)((cb >> 52) & 0x7ff);
    int k = max(0, ew - ec + 47);
    for (; k <= kApoKMax; ++k) {
        double l2, h2;
        d_decode(c, k, l2, h2);
        if (l2 <= lo && h2 >= hi) break;
    }
    if (k > kApoKMax) return false;
    out = __longlong_as_double((long long)(0x8000000000000000ULL | (unsigned long long)cb | (unsigned long long)k));
    return true;
}

// ---- APO: row a' without the mean stream (w > 0, BSMSE/Euclidean, one CTA per section)
// After merging b into a, the new mean is m' = lam m_a + (1 - lam) m_b + e (lam = n_a/n,
// e = the rounding of the new sums / count), and for every region j the parallelogram
// identity gives, exactly in real arithmetic,
//     || lam m_a + (1-lam) m_b - m_j ||^2 = lam T_aj + (1-lam) T_bj - lam (1-lam) T_ab
// with T_xy = ||m_x - m_y||^2. D already holds d(a, j), d(b, j) and d(a, b), and the
// reference value satisfies d^2 = C T (1 + eps) with |eps| <= E = (B + 8) u (C = n_x n_y /
// (n_x + n_y) for BSMSE, 1 for Euclidean: ascending-band sum of B rounded squares, the
// coefficient product, sqrt). So two D rows (16 bytes per column instead of the 8B + 16
// bytes of a mean column) give a rigorous interval around the reference's d(a', j):
// directed-rounding arithmetic throughout, ||e|| <= 3.01 u max ||m|| (max over the
// section's initial means, which bound every later mean). Entries the interval cannot
// settle are evaluated exactly (warp_exact) -- offers that may beat a row's cached best
// (0.3 per step on a C4 leaf), a's best when several columns tie within their intervals,
// argmin winners, multi-candidate rescans -- so every dissimilarity the merge sequence
// and the log see is the reference's exact fp64 value.
//
// D entries: an exact value is a non-negative double (sign bit clear). An interval is
// [sign=1 | centre c with its low 6 mantissa bits replaced by k] = c (1 -/+ 2^(k-46)),
// decoded with directed multiplies (single DMUL.RM/.RP instructions).
//
// The interval arithmetic itself is round-to-nearest with explicit slack (directed
// division/sqrt are long software sequences): with u = 2^-53, every quantity below is
// within a few u of its real value, and each bound is widened by at least twice the
// worst-case accumulated error:
//   A = d(a,j)^2 (1/n_a + 1/n_j) = T_aj (1 + eps) (1 +- 5u)        (d^2 = C T (1 + eps))
//   V = lam A + (1-lam) B - lam(1-lam) T_ab,  |V - V_true| <= (E + 12u) S,  S = sum of |terms|
//   ||v|| in [sqrt(V_lo - 2(E+16u)S), sqrt(V_hi + 2(E+16u)S)]   (the rounding of the
//        subtraction and sqrt is covered by the doubled slack; ||v|| <= 2 max||m||)
//   sqrt(T') in [||v|| -+ ee], ee = 10u max||m|| (>= 3.02u max||m|| for e, + sqrt/sub rounding)
//   d(a',j) = sqrt(C') sqrt(T') sqrt(1 + eps'),  widened by 2 (E/2 + 8u) relative.
// Per-step constants of the row-a' pass (identical in every thread).
struct ApoStep {
    double lam, mu, kt_lo, kt_hi;  // na/nn, nb/nn, lam mu T_ab (d(a, b) may be an interval)
    double rna, rnb, rnn;
    double vslack, ee, mrel;
};
template <int M>
__device__ __forceinline__ ApoStep apo_step(double na, double nb, double dab, double E, double ee) {
    ApoStep p;
    const double nn = na + nb;
    p.lam = na / nn;
    p.mu = nb / nn;
    p.rna = M == kBsmse ? 1.0 / na : 0.0;
    p.rnb = M == kBsmse ? 1.0 / nb : 0.0;
    p.rnn = M == kBsmse ? 1.0 / nn : 0.0;
    double dl, dh;
    d_unpack(dab, dl, dh);
    const double cab = M == kBsmse ? p.rna + p.rnb : 1.0;
    p.kt_lo = p.lam * p.mu * (dl * dl * cab);
    p.kt_hi = p.lam * p.mu * (dh * dh * cab);
    p.vslack = 2.0 * (E + 16.0 * kU64);
    p.ee = ee;
    p.mrel = 2.0 * (0.5 * E + 8.0 * kU64);
    return p;
}
// interval around the reference's d(a', j) from the raw D entries d(a, j), d(b, j)
template <int M>
__device__ __forceinline__ void apo_interval(const ApoStep& p, double rA, double rB, double nj, double& dlo,
                                             double& dhi) {
    double al, ah, bl, bh;
    d_unpack(rA, al, ah);
    d_unpack(rB, bl, bh);
    const double rj = M == kBsmse ? 1.0 / nj : 0.0;
    const double ca = M == kBsmse ? p.rna + rj : 1.0, cb = M == kBsmse ? p.rnb + rj : 1.0;
    const double Al = al * al * ca, Ah = ah * ah * ca, Bl = bl * bl * cb, Bh = bh * bh * cb;
    const double Vl = p.lam * Al + p.mu * Bl - p.kt_hi;
    const double Vh = p.lam * Ah + p.mu * Bh - p.kt_lo;
    const double dv = p.vslack * (p.lam * Ah + p.mu * Bh + p.kt_hi);
    const double nlo = fmax(0.0, sqrt(fmax(0.0, Vl - dv)) - p.ee);
    const double nhi = sqrt(fmax(0.0, Vh + dv)) + p.ee;
    const double sc = M == kBsmse ? sqrt(1.0 / (p.rnn + rj)) : 1.0;  // sqrt(C')
    dlo = nlo * sc * (1.0 - p.mrel);
    dhi = nhi * sc * (1.0 + p.mrel);
}

// Exact d(i, j) by one warp (all lanes return it) from two fp64 mean vectors
// (shared or global memory; APO keeps a region-major copy of the exact cached means):
// every lane loads its bands up front, the per-band terms are independent, and only
// the ascending-band sum is a serial chain, fed by shuffles issued ahead of it.
template <int M>
__device__ __noinline__ double warp_exact(const double* mi, const double* mj, double ci, double cj, int B,
                                             int lane) {
    double s = 0.0;
    for (int k0 = 0; k0 < B; k0 += 256) {
        double term[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 32 * u + lane;
            const double vi = k < B ? mi[k] : 0.0, vj = k < B ? __ldcg(mj + k) : 0.0;
            if (M == kSam) {
                term[u] = __dmul_rn(vi, vj);
            } else {
                const double t = __dsub_rn(vi, vj);
                term[u] = __dmul_rn(t, t);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int kn = min(32, B - (k0 + 32 * u));
            if (kn <= 0) break;
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
                const double tk = __shfl_sync(0xffffffffu, term[u], kk);
                if (kk < kn) s = __dadd_rn(s, tk);
            }
        }
    }
    return pair_finish<M>(ci, cj, s, 0.0, 0.0);
}

// The same value through a per-warp shared-memory staging row: the lanes write the
// per-band terms, lane 0 runs the ascending-band sum from shared memory (a shuffle-fed
// chain stalls every lane of the warp on every one of its B additions), all lanes get
// the result. stg: B doubles owned by the calling warp.
template <int M>
__device__ __noinline__ double warp_exact_stg(const double* mi, const double* mj, double ci, double cj, int B,
                                              int lane, double* stg) {
    for (int k0 = 0; k0 < B; k0 += 256) {
        double term[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 32 * u + lane;
            const double vi = k < B ? mi[k] : 0.0, vj = k < B ? __ldcg(mj + k) : 0.0;
            if (M == kSam) {
                term[u] = __dmul_rn(vi, vj);
            } else {
                const double t = __dsub_rn(vi, vj);
                term[u] = __dmul_rn(t, t);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 32 * u + lane;
            if (k < B) stg[k] = term[u];
        }
    }
    __syncwarp();
    double s = 0.0;
    if (lane == 0) {
        int k = 0;
        for (; k + 8 <= B; k += 8) {
            double t[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) t[q] = stg[k + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) s = __dadd_rn(s, t[q]);
        }
        for (; k < B; ++k) s = __dadd_rn(s, stg[k]);
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    __syncwarp();  // the staging row may be rewritten by the warp's next call
    return pair_finish<M>(ci, cj, s, 0.0, 0.0);
}

// APO: a's best when its single candidate may be an interval (nothing to compare)
__device__ __forceinline__ void rb_offer_iv(RowBest& b, double v, int j) {
    if (__double_as_longlong(v) < 0) { b.d = v; b.j = j; }
    else rb_offer(b, v, j);
}

}  // namespace rhseg
