// cf_physics.cuh — per-element / per-facet / per-node physics of the castfem
// explicit step, as sm_100a device code.
//
// Every expression keeps the reference's operation order (paths relative to
// /root/reference/proj/include/castfem/) so that, compiled with -fmad=false
// (no FMA contraction; fp64 '/' and sqrt are IEEE round-to-nearest on sm_100a
// as on x86), results are bitwise equal to the reference built with
// -ffp-contract=off:
//   PiecewiseLinear::operator()  material.hpp:30-38
//   MaterialTable::enthalpy      material.hpp:89-102 (melt_fraction :69-72)
//   apparent_heat_capacity       fem.hpp:26-45 (Lemmon)
//   element_accumulate           fem.hpp:57-70
//   facet_flux_accumulate        fem.hpp:74-79 (+ interface branch blocked.hpp:485-490)
//   element_stable_dt            fem.hpp:83-85
#pragma once

#include <cstdint>

#include "cf_internal.hpp"

namespace cfb {

__device__ __forceinline__ double dev_pl_eval(const DevParams* __restrict__ P, DevTable t, double x) {
    const double* xs = P->pool + t.off;
    const double* ys = xs + t.n;
    if (t.n <= 1) return ys[0];
    if (x <= xs[0]) return ys[0];
    if (x >= xs[t.n - 1]) return ys[t.n - 1];
    int i = 0;
    while (i + 1 < t.n && xs[i + 1] <= x) ++i;
    const double f = (x - xs[i]) / (xs[i + 1] - xs[i]);
    return ys[i] + f * (ys[i + 1] - ys[i]);
}

template <bool TDEP>
__device__ __forceinline__ double dev_c(const DevParams* __restrict__ P, const DevMaterial& m, double T) {
    if (!TDEP || m.c.n <= 1) return m.c0;
    return dev_pl_eval(P, m.c, T);
}
template <bool TDEP>
__device__ __forceinline__ double dev_k(const DevParams* __restrict__ P, const DevMaterial& m, double T) {
    if (!TDEP || m.k.n <= 1) return m.k0;
    return dev_pl_eval(P, m.k, T);
}

// MaterialTable::enthalpy material.hpp:89-102
template <bool TDEP>
__device__ __forceinline__ double dev_enthalpy(const DevParams* __restrict__ P, const DevMaterial& m, double T) {
    double sensible;
    if (!TDEP || m.c.n <= 1) {
        sensible = m.c0 * (T - m.ref);
    } else {
        const double* xs = P->pool + m.c.off;
        const double* ys = xs + m.c.n;
        const int n = m.c.n;
        const double Tc = T < xs[0] ? xs[0] : (xs[n - 1] < T ? xs[n - 1] : T);
        int ub = 0;
        while (ub < n && xs[ub] <= Tc) ++ub;
        const int i = (ub < n - 1 ? ub : n - 1) - 1;
        sensible = P->pool[m.cum_off + i] + 0.5 * (ys[i] + dev_pl_eval(P, m.c, Tc)) * (Tc - xs[i]);
    }
    // melt_fraction material.hpp:69-72: clamp((T - Ts)/(Tl - Ts), 0, 1). Outside the mushy range
    // the clamp decides without the IEEE division (T <= Ts gives v <= 0, T >= Tl gives v >= 1:
    // the correctly rounded quotient is monotone), so only mushy nodes divide; NaN falls through
    double mf = 0.0;
    if (m.has_phase) {
        if (T >= m.liquidus) {
            mf = 1.0;
        } else if (!(T <= m.solidus)) {
            const double v = (T - m.solidus) / (m.liquidus - m.solidus);
            mf = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
        }
    }
    return sensible + m.latent * mf;
}

// Element gradients and volume from the oriented corner coordinates: the
// operation sequence of the host tet_geometry (cf_mesh.cpp; geometry.hpp:50-79):
// e_k = p_k - p0, c = e2 x e3, det = e1.c, vol = det/6, g1 = (e2 x e3)/det,
// g2 = (e3 x e1)/det, g3 = (e1 x e2)/det (as products with inv = 1/det),
// g0 = ((g1+g2)+g3)*-1. With -fmad=false and IEEE '/', bitwise equal to the
// stored ElementGeom.
__device__ __forceinline__ void dev_tet_grads(const double (&p)[4][3], double (&g)[4][3], double& vol) {
    double e1[3], e2[3], e3[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        e1[k] = p[1][k] - p[0][k];
        e2[k] = p[2][k] - p[0][k];
        e3[k] = p[3][k] - p[0][k];
    }
    const double c0 = e2[1] * e3[2] - e2[2] * e3[1];
    const double c1 = e2[2] * e3[0] - e2[0] * e3[2];
    const double c2 = e2[0] * e3[1] - e2[1] * e3[0];
    const double det = e1[0] * c0 + e1[1] * c1 + e1[2] * c2;
    vol = det / 6.0;
    const double inv = 1.0 / det;
    g[1][0] = c0 * inv;
    g[1][1] = c1 * inv;
    g[1][2] = c2 * inv;
    g[2][0] = (e3[1] * e1[2] - e3[2] * e1[1]) * inv;
    g[2][1] = (e3[2] * e1[0] - e3[0] * e1[2]) * inv;
    g[2][2] = (e3[0] * e1[1] - e3[1] * e1[0]) * inv;
    g[3][0] = (e1[1] * e2[2] - e1[2] * e2[1]) * inv;
    g[3][1] = (e1[2] * e2[0] - e1[0] * e2[2]) * inv;
    g[3][2] = (e1[0] * e2[1] - e1[1] * e2[0]) * inv;
#pragma unroll
    for (int k = 0; k < 3; ++k) g[0][k] = ((g[1][k] + g[2][k]) + g[3][k]) * -1.0;
}

// tet_geometry (cf_mesh.cpp / geometry.hpp:48-77) on the device: edges first (min/max of the six
// lengths, first pair (0,1) seeding both, as std::min/std::max), then the gradients and volume.
__device__ __forceinline__ void dev_tet_geometry(const double (&p)[4][3], double (&g)[4][3], double& vol,
                                                 double& min_edge, double& max_edge) {
    double d0 = p[1][0] - p[0][0], d1 = p[1][1] - p[0][1], d2 = p[1][2] - p[0][2];
    min_edge = max_edge = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a + 1; b < 4; ++b) {
            d0 = p[b][0] - p[a][0];
            d1 = p[b][1] - p[a][1];
            d2 = p[b][2] - p[a][2];
            const double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            min_edge = len < min_edge ? len : min_edge;
            max_edge = max_edge < len ? len : max_edge;
        }
    dev_tet_grads(p, g, vol);
}

// One element: lumped capacitance share `lump` (added to each of the 4
// nodes) and the 4 conduction residual terms rc[a] (subtracted).
// g1..g3 are the stored gradients; g0 = (g1+g2+g3)*-1.0 (geometry.hpp:75).
// Bitwise equal to the reference's apparent_heat_capacity + element_accumulate:
//  - T[hi]-T[lo] equals fmax(..)-fmin(..) exactly (same extreme values); the
//    lo/hi indices are only needed by the rare secant branch;
//  - the degeneracy test gt2 < 1e-14*scale*scale (scale = range/max_edge) is
//    decided without the division whenever gt2*max_edge^2 clears 1e-14*range^2
//    by a 1e-6 relative margin (far above the ~1e-15 rounding of either form);
//    otherwise the reference expression is evaluated verbatim.
//  - LB (stored layout, which does not stream max_edge): max_edge >= 1/|g_1| (the height
//    from vertex 1, 1/|grad N_1|, is at most the longest edge), so gt2 > 1000*rhs*|g_1|^2
//    implies the margin test above with a factor-1000 allowance for the rounding of the stored
//    g_1 (relative error <= ~1e-4 even for the flattest tet finalize_mesh accepts,
//    V > 1e-12 max_edge^3). Exactly: gt2*max_edge^2 >= range^2 >> 1e-14 range^2, so the test
//    passes for all but near-uniform (round-off) gradients and extreme slivers; only then is the
//    exact max_edge fetched (max_edge_fn(): a global load) and the original test evaluated.
template <bool TDEP, bool LB, class MaxEdge>
__device__ __forceinline__ void dev_element(const DevParams* __restrict__ P, const DevMaterial& m,
                                            const double (&g)[4][3], double vol, MaxEdge&& max_edge_fn,
                                            const double (&T)[4], const double (&H)[4], double& lump,
                                            double (&rc)[4], bool probe_no_divsqrt = false) {
    // grad T (fem.hpp:36-40 and :64-65 compute the same sums; shared here). The reference
    // starts each sum at 0.0; starting at the first product differs only in the sign of an
    // all-zero sum, which every consumer erases (squares in gt2/gh2; kv*(g.gradT) enters r
    // only through r - rc with r starting at +0.0), so every output stays bitwise equal.
    double gtx = g[0][0] * T[0], gty = g[0][1] * T[0], gtz = g[0][2] * T[0];
#pragma unroll
    for (int a = 1; a < 4; ++a) {
        gtx = gtx + g[a][0] * T[a];
        gty = gty + g[a][1] * T[a];
        gtz = gtz + g[a][2] * T[a];
    }
    const double t_bar = 0.25 * (((T[0] + T[1]) + T[2]) + T[3]);
    // compare-selects (finite T): same extreme values as the reference's index scan
    const double l01 = T[1] < T[0] ? T[1] : T[0], l23 = T[3] < T[2] ? T[3] : T[2];
    const double h01 = T[1] > T[0] ? T[1] : T[0], h23 = T[3] > T[2] ? T[3] : T[2];
    const double Tlo = l23 < l01 ? l23 : l01;
    const double Thi = h23 > h01 ? h23 : h01;
    const double range = Thi - Tlo;
    double capp;
    if (range <= 0) {
        capp = dev_c<TDEP>(P, m, t_bar);
    } else {
        double ghx = g[0][0] * H[0], ghy = g[0][1] * H[0], ghz = g[0][2] * H[0];
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            ghx = ghx + g[a][0] * H[a];
            ghy = ghy + g[a][1] * H[a];
            ghz = ghz + g[a][2] * H[a];
        }
        const double gt2 = gtx * gtx + gty * gty + gtz * gtz;
        bool degenerate = false;
        const double rhs = 1e-14 * (range * range);
        const double g1sq = g[1][0] * g[1][0] + g[1][1] * g[1][1] + g[1][2] * g[1][2];
        if (!LB || !(gt2 > (rhs * 1000.0) * g1sq)) {
            const double max_edge = max_edge_fn();
            const double lhs = gt2 * (max_edge * max_edge);
            if (!(lhs > rhs * 1.000001)) {
                const double scale = range / max_edge;
                degenerate = gt2 < 1e-14 * scale * scale;
            }
        }
        if (degenerate) {
            // secant (H_hi - H_lo)/range with the reference's first-index tie rule
            double tl = T[0], th = T[0], hl = H[0], hh = H[0];
#pragma unroll
            for (int a = 1; a < 4; ++a) {
                if (T[a] < tl) { tl = T[a]; hl = H[a]; }
                if (T[a] > th) { th = T[a]; hh = H[a]; }
            }
            capp = (hh - hl) / range;
        } else {
            const double gh2 = ghx * ghx + ghy * ghy + ghz * ghz;
            capp = probe_no_divsqrt ? gh2 + gt2 : sqrt(gh2 / gt2);  // (diagnostics probe only)
        }
    }
    // element_accumulate fem.hpp:60-69
    lump = m.rho * capp * vol * 0.25;
    const double kv = dev_k<TDEP>(P, m, t_bar) * vol;
#pragma unroll
    for (int a = 0; a < 4; ++a) rc[a] = kv * (g[a][0] * gtx + g[a][1] * gty + g[a][2] * gtz);
}

// element_stable_dt fem.hpp:83-85 at the element mean temperature
template <bool TDEP>
__device__ __forceinline__ double dev_stable_bound(const DevParams* __restrict__ P, const DevMaterial& m,
                                                  double min_edge, const double (&T)[4]) {
    const double t_bar = 0.25 * (((T[0] + T[1]) + T[2]) + T[3]);
    return m.rho * dev_c<TDEP>(P, m, t_bar) * min_edge * min_edge / dev_k<TDEP>(P, m, t_bar);
}

}  // namespace cfb
