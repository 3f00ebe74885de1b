// precompute.cpp — host pre-calculating step of the product path
// (§II l.191-246: "implemented by the CPU", l.265), double precision.
//
// Computed ONCE for pitch 0 and reused for every pitch by the periodicity of
// PAPER.md l.174-185 / l.222-231 (λ_{i,o}(x + kP e_z) = λ_{i,o}(x) + 2kπ;
// v*, α*, w* invariant under (λ + 2kπ, z + kP)).  Written independently of the
// oracle: PI-lines by safeguarded Newton (not bisection), ψ̂ by scan +
// Illinois regula falsi (not bisection).  Index rules follow DESIGN.md
// reading A12 so integer tables are reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "plan.hpp"

namespace kats {

namespace {

struct Geo {
    double R, D, P, lam0, z0, dlam, h, r_fov, dw, da, aoff, dx, dy, dz;
    int nr, nc, nx, ny, nz, vt;
    bool flat;                      // KATS_FLAG_FLAT: column coordinate u [mm] on the plane at distance D
};

Geo derive(const katsevich_geometry &g)
{
    Geo o;
    o.R = g.R; o.D = g.D; o.P = g.pitch; o.lam0 = g.lambda0; o.z0 = g.z0;
    o.vt = g.views_per_turn;
    o.dlam = 2.0 * kPi / g.views_per_turn;
    o.h = g.pitch / (2.0 * kPi);
    double hx = 0.5 * g.nx * g.dx, hy = 0.5 * g.ny * g.dy;
    o.r_fov = g.r_fov > 0.0 ? g.r_fov : std::hypot(hx, hy) * (1.0 + 1e-9);
    o.dw = g.d_w; o.da = g.d_alpha; o.aoff = g.alpha_offset;
    o.dx = g.dx; o.dy = g.dy; o.dz = g.pitch / g.nz_per_pitch;
    o.nr = g.n_rows; o.nc = g.n_cols; o.nx = g.nx; o.ny = g.ny; o.nz = g.nz_per_pitch;
    o.flat = (g.flags & KATS_FLAG_FLAT) != 0;
    return o;
}

// Detector column position (fractional column index) and row scale (rows per unit of z - z_src) of
// the ray from the source through (x, y) at view angle (c, s): curved α* = atan2(u, v*), w* =
// D (z - z_src)/sqrt(u² + v*²) (P:l.161-170); flat (reading A27) u* = D u / v*, w* = D (z - z_src)/v*.
inline void ray_col_scale(const Geo &o, double x, double y, double c, double s, double &col, double &sc)
{
    const double vs = o.R - x * c - y * s, us = -x * s + y * c;
    const double a = o.flat ? o.D * us / vs : std::atan2(us, vs);
    col = a / o.da + 0.5 * (o.nc - 1) - o.aoff;
    sc = o.D / (o.flat ? vs : std::hypot(us, vs)) / o.dw;
}

// A12 canonical snapping: an argument within 1e-9 of an integer is that integer.
inline double snap9(double a)
{
    double r = std::round(a);
    return std::fabs(a - r) < 1e-9 ? r : a;
}

// Linear index on n nodes: (idx, frac) with idx in [0, n-2]; false outside [0, n-1].
inline bool node_index(double pos, int n, int32_t &idx, double &frac)
{
    double a = snap9(pos);
    if (a < 0.0 || a > (double)(n - 1) || std::isnan(a)) return false;
    double fl = std::floor(a);
    int32_t i = (int32_t)fl;
    if (i > n - 2) i = n - 2;
    idx = i;
    frac = a - (double)i;
    return true;
}

// PI-line of (x, y, z).  The chord a(σ-δ)a(σ+δ)
// through x: with A = (x cos(σ+λ0) + y sin(σ+λ0))/R, B = (-x sin + y cos)/R
// one has δ = acos A and the chord position u = B / sin δ; σ is the root of
// F(σ) = σ + u δ - (z - z0)/h on [ζ-π, ζ+π].  Safeguarded Newton: the
// analytic F' is used while the iterate stays in the shrinking bracket,
// bisection otherwise.
bool pi_line_newton(const Geo &o, double x, double y, double z, double &li, double &lo)
{
    const double zeta = (z - o.z0) / o.h;
    double a = zeta - kPi, b = zeta + kPi;
    double s = zeta;
    auto eval = [&](double sg, double &F, double &dF, double &del) {
        double c = std::cos(sg + o.lam0), sn = std::sin(sg + o.lam0);
        double A = (x * c + y * sn) / o.R, B = (-x * sn + y * c) / o.R;
        A = std::min(1.0, std::max(-1.0, A));
        double sd = std::sqrt(std::max(1e-300, 1.0 - A * A));
        del = std::acos(A);
        double u = B / sd;
        double ddel = -B / sd;
        double du = (-A * sd + B * B * A / sd) / (sd * sd);
        F = sg + u * del - zeta;
        dF = 1.0 + du * del + u * ddel;
    };
    double F, dF, del;
    bool ok = false;
    for (int it = 0; it < 100; ++it) {
        eval(s, F, dF, del);
        if (F == 0.0) { ok = true; break; }
        if (F < 0.0) a = s; else b = s;
        double sn = s - F / dF;
        if (!(sn > a && sn < b) || !std::isfinite(sn)) sn = 0.5 * (a + b);
        if (std::fabs(sn - s) <= 2e-16 * std::max(1.0, std::fabs(s)) || b - a <= 4e-16 * std::max(1.0, std::fabs(s))) {
            s = sn; ok = true; break;
        }
        s = sn;
    }
    eval(s, F, dF, del);
    li = s - del;
    lo = s + del;
    return ok && std::fabs(F) < 1e-9;
}

// Eq. (11): w_κ(α, ψ) = (DP/2πR)(ψ cos α + (ψ/tan ψ) sin α); flat (reading A27): the same κ-plane on
// the plane at distance D, (DP/2πR)(ψ + (ψ/tan ψ) u/D).
inline double kappa_height(const Geo &o, double kappa, double alpha, double psi)
{
    double q = std::fabs(psi) < 1e-6 ? 1.0 - psi * psi / 3.0 - psi * psi * psi * psi / 45.0
                                     : psi * std::cos(psi) / std::sin(psi);
    if (o.flat) return kappa * (psi + q * alpha / o.D);
    return kappa * (psi * std::cos(alpha) + q * std::sin(alpha));
}

// ψ̂(α, w) (Eq. 14, P:l.147): the root of smallest |ψ| met moving outward
// from ψ = 0 (reading A8) within [-ψmax, ψmax].  Outward scan with
// 8192 steps, then Illinois regula falsi on the first bracketing step.
bool kappa_root(const Geo &o, double kappa, double psi_max, double alpha, double w, double &psi)
{
    auto f = [&](double p) { return kappa_height(o, kappa, alpha, p) - w; };
    double f0 = f(0.0);
    if (f0 == 0.0) { psi = 0.0; return true; }
    const double sgn = f0 < 0.0 ? 1.0 : -1.0;
    const int N = 8192;
    double pa = 0.0, fa = f0;
    for (int k = 1; k <= N; ++k) {
        double pb = sgn * psi_max * (double)k / N;
        double fb = f(pb);
        if (fb == 0.0) { psi = pb; return true; }
        if ((fa < 0.0) != (fb < 0.0)) {
            int side = 0;
            for (int it = 0; it < 200; ++it) {
                double pc = (pa * fb - pb * fa) / (fb - fa);
                if (!(pc > std::min(pa, pb) && pc < std::max(pa, pb))) pc = 0.5 * (pa + pb);
                double fc = f(pc);
                if (fc == 0.0) { pa = pb = pc; break; }
                if ((fc < 0.0) == (fb < 0.0)) {
                    pb = pc; fb = fc;
                    if (side == -1) fa *= 0.5;
                    side = -1;
                } else {
                    pa = pc; fa = fc;
                    if (side == 1) fb *= 0.5;
                    side = 1;
                }
                if (std::fabs(pb - pa) <= 1e-16 * std::max(1.0, std::fabs(pa))) break;
            }
            psi = 0.5 * (pa + pb);
            return true;
        }
        pa = pb; fa = fb;
    }
    return false;
}

}  // namespace

int validate(const katsevich_geometry &g, std::string &detail)
{
    char buf[256];
    auto bad = [&](const char *what) {
        std::snprintf(buf, sizeof buf, "invalid geometry: %s", what);
        detail = buf;
        return KATS_ERR_INVALID_GEOMETRY;
    };
    if (!(g.R > 0)) return bad("R <= 0");
    if (!(g.D > 0)) return bad("D <= 0");
    if (!(g.pitch > 0)) return bad("pitch <= 0");
    if (g.views_per_turn < 3) return bad("views_per_turn < 3");
    if (g.n_rows < 2) return bad("n_rows < 2");
    if (g.n_cols < 2) return bad("n_cols < 2");
    if (!(g.d_w > 0) || !(g.d_alpha > 0)) return bad("detector spacing <= 0");
    if (g.nx < 1 || g.ny < 1 || g.nz_per_pitch < 1) return bad("empty voxel grid");
    if (!(g.dx > 0) || !(g.dy > 0)) return bad("voxel spacing <= 0");
    if (g.n_psi != 0 && g.n_psi < 2) return bad("n_psi must be 0 or >= 2");
    if (g.flags & ~(KATS_FLAG_HALF_SAMPLE | KATS_FLAG_HANN | KATS_FLAG_FLAT)) return bad("unknown flags");
    if ((g.flags & KATS_FLAG_FLAT) && (g.flags & KATS_FLAG_HALF_SAMPLE))
        return bad("the half-sample derivative is not supported with the flat detector");
    if ((g.flags & KATS_FLAG_HALF_SAMPLE) && (g.n_rows < 3 || g.n_cols < 3))
        return bad("the half-sample derivative needs n_rows >= 3 and n_cols >= 3");
    if ((g.flags & KATS_FLAG_HALF_SAMPLE) && g.n_rows > 65) return bad("the half-sample derivative needs n_rows <= 65");
    if (!std::isfinite(g.lambda0) || !std::isfinite(g.z0) || !std::isfinite(g.alpha_offset)) return bad("non-finite parameter");
    double half_fan = (0.5 * (g.n_cols - 1) + std::fabs(g.alpha_offset)) * g.d_alpha;
    if (!(g.flags & KATS_FLAG_FLAT) && !(half_fan < 0.5 * kPi)) return bad("detector fan reaches |alpha| >= pi/2");
    Geo o = derive(g);
    if (g.r_fov < 0 || !(o.r_fov < g.R)) return bad("r_fov >= R (FOV cylinder must lie inside the helix)");
    return KATS_OK;
}

// Noo's half-sample derivative (NEXT-4; reading A25) produces g1 at (λ_{k+½}, α_{l+½},
// w_{m+½}): the samples of a detector with one row and one column fewer (same spacings and α offset)
// on the same helix parametrised from λ0 + Δλ/2, z0 + h Δλ/2 (a(λ_{k+½}) = a'(λ_k), Eq. 1).  Steps
// 2-7 and every table use that grid; the voxel grid and the FOV are unchanged.
katsevich_geometry half_sample_geometry(const katsevich_geometry &g)
{
    katsevich_geometry e = g;
    const double dlam = 2.0 * kPi / g.views_per_turn;
    e.n_rows = g.n_rows - 1;
    e.n_cols = g.n_cols - 1;
    e.lambda0 = g.lambda0 + 0.5 * dlam;
    e.z0 = g.z0 + g.pitch / (2.0 * kPi) * 0.5 * dlam;
    e.flags = g.flags & ~KATS_FLAG_HALF_SAMPLE;    // other variants carry over to the shifted grid
    return e;
}

int compute_host_tables(const katsevich_geometry &g, HostTables &t, std::string &detail)
{
    const Geo o = derive(g);
    t.dlam = o.dlam;
    t.h = o.h;
    t.r_fov = o.r_fov;
    t.alpha_m = std::asin(o.r_fov / o.R);                 // α_m = arcsin(r/R), P:l.133
    t.psi_max = 0.5 * kPi + t.alpha_m;                    // ψ ∈ [-π/2-α_m, π/2+α_m], P:l.132
    t.n_psi = g.n_psi > 0 ? g.n_psi : 2 * g.n_rows + 1;
    t.dpsi = 2.0 * t.psi_max / (t.n_psi - 1);
    t.kappa = o.D * o.P / (2.0 * kPi * o.R);              // DP/(2πR), Eq. (11)
    const int nr = o.nr, nc = o.nc, np = t.n_psi;
    auto alpha_of = [&](int l) { return ((double)l - 0.5 * (nc - 1) + o.aoff) * o.da; };
    auto w_of = [&](int m) { return ((double)m - 0.5 * (nr - 1)) * o.dw; };

    // ---- T_fr: forward height rebin (Eqs. 10-11) ----
    t.fr_idx.assign((size_t)np * nc, -1);
    t.fr_frac.assign((size_t)np * nc, 0.0);
    for (int i = 0; i < np; ++i) {
        double psi = -t.psi_max + (double)i * t.dpsi;
        for (int l = 0; l < nc; ++l) {
            double pos = kappa_height(o, t.kappa, alpha_of(l), psi) / o.dw + 0.5 * (nr - 1);
            int32_t m; double f;
            if (node_index(pos, nr, m, f)) { t.fr_idx[(size_t)i * nc + l] = m; t.fr_frac[(size_t)i * nc + l] = f; }
        }
    }
    // ---- T_br: backward height rebin (Eqs. 13-14) ----
    t.br_idx.assign((size_t)nr * nc, -1);
    t.br_frac.assign((size_t)nr * nc, 0.0);
    int root_fail = 0;
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:root_fail)
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            double psi;
            if (!kappa_root(o, t.kappa, t.psi_max, alpha_of(l), w_of(m), psi)) continue;   // no root: zero
            int32_t i; double f;
            if (node_index((psi + t.psi_max) / t.dpsi, np, i, f)) {
                t.br_idx[(size_t)m * nc + l] = i; t.br_frac[(size_t)m * nc + l] = f;
            }
        }

    // K4^T writes each κ-line of a column once, walking the rows, when T_br's index never decreases
    // down a column (rows without a root are skipped)
    t.br_monotone = true;
    for (int l = 0; l < nc && t.br_monotone; ++l) {
        int32_t prev = -1;
        for (int m = 0; m < nr; ++m) {
            const int32_t i = t.br_idx[(size_t)m * nc + l];
            if (i < 0) continue;
            if (i < prev) { t.br_monotone = false; break; }
            prev = i;
        }
    }

    // ---- T_pi: PI-line limits per voxel of pitch 0 (P:l.194-202) ----
    const size_t nvox = (size_t)o.nx * o.ny * o.nz;
    t.pi_first.assign(nvox, 0);
    t.pi_last.assign(nvox, -1);
    t.w_first.assign(nvox, 0.0);
    t.w_last.assign(nvox, 0.0);
    const double r2 = o.r_fov * o.r_fov;
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    double wL = 0.0;
    int pi_fail = 0;
    #pragma omp parallel for collapse(2) schedule(dynamic, 2) reduction(min:lo) reduction(max:hi, wL) reduction(+:pi_fail)
    for (int j = 0; j < o.nz; ++j)
        for (int iy = 0; iy < o.ny; ++iy) {
            double y = ((double)iy - 0.5 * o.ny) * o.dy;
            double z = (double)j * o.dz;
            for (int ix = 0; ix < o.nx; ++ix) {
                double x = ((double)ix - 0.5 * o.nx) * o.dx;
                if (!(x * x + y * y < r2)) continue;           // outside U (P:l.96): empty window -> 0
                double li, lo_;
                if (!pi_line_newton(o, x, y, z, li, lo_)) { ++pi_fail; continue; }
                double ti = li / o.dlam, to = lo_ / o.dlam;
                int64_t kf = (int64_t)std::floor(snap9(ti + 0.5));
                int64_t kl = (int64_t)std::ceil(snap9(to - 0.5));
                auto cell = [&](int64_t k) {
                    double a = std::max((double)k - 0.5, ti), b = std::min((double)k + 0.5, to);
                    return b > a ? b - a : 0.0;
                };
                size_t id = ((size_t)j * o.ny + iy) * o.nx + ix;
                t.pi_first[id] = (int32_t)kf;
                t.pi_last[id] = (int32_t)kl;
                t.w_first[id] = cell(kf);
                t.w_last[id] = cell(kl);
                lo = std::min(lo, kf);
                hi = std::max(hi, kl);
                // w_L (P:l.336): |w*| at the first/last grid view inside [λ_i, λ_o]
                for (int e = 0; e < 2; ++e) {
                    double k = e == 0 ? std::ceil(ti) : std::floor(to);
                    double lam = k * o.dlam;
                    double c = std::cos(lam + o.lam0), s = std::sin(lam + o.lam0);
                    double col, sc;
                    ray_col_scale(o, x, y, c, s, col, sc);
                    double wst = sc * o.dw * (z - o.z0 - o.h * lam);
                    wL = std::max(wL, std::fabs(wst));
                }
            }
        }
    if (pi_fail) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "PI-line solver did not converge for %d voxels", pi_fail);
        detail = buf;
        return KATS_ERR_PI_NONCONVERGENCE;
    }
    if (lo > hi) { lo = 0; hi = -1; }
    t.bp_lo = lo;
    t.bp_hi = hi;
    t.w_L = wL;
    t.td_covered = wL <= 0.5 * (nr - 1) * o.dw * (1.0 + 1e-9);
    // Interior views (k_first < k < k_last) sample inside [λ_i, λ_o], so |w*| <= w_L and
    // |α*| <= α_m; with a relative margin well above fp32 rounding the kernel may skip the
    // per-sample detector test.
    // (flat: |u*| <= D tan α_m over the FOV cylinder)
    const double a_lo = (-0.5 * (nc - 1) + o.aoff) * o.da, a_hi = (0.5 * (nc - 1) + o.aoff) * o.da;
    const double a_m = o.flat ? o.D * std::tan(t.alpha_m) : t.alpha_m;
    t.interior_in_detector = wL <= 0.5 * (nr - 1) * o.dw * (1.0 - 1e-5) &&
                             a_lo <= -a_m - 1e-5 * o.da && a_hi >= a_m + 1e-5 * o.da;
    (void)root_fail;

    // ---- footprint box of one CTA (kTileX x kTileY columns, kChunkZ slices) on one
    // interior view: columns/quad rows spanned by the tile's corner rays (the
    // extreme α* and |r| over a square are at its corners), over every tile, chunk
    // and interior view; +margins for the kernel's fp32 arithmetic.
    {
        const int ntx = (o.nx + kTileX - 1) / kTileX, nty = (o.ny + kTileY - 1) / kTileY;
        const int nch = (o.nz + kChunkZ - 1) / kChunkZ;
        int bw = 0, bh = 0;
        #pragma omp parallel for collapse(2) schedule(dynamic, 1) reduction(max:bw, bh)
        for (int ty = 0; ty < nty; ++ty)
            for (int tx = 0; tx < ntx; ++tx)
                for (int ch = 0; ch < nch; ++ch) {
                    int64_t k0 = INT64_MAX, k1 = INT64_MIN;
                    for (int j = ch * kChunkZ; j < std::min(o.nz, (ch + 1) * kChunkZ); ++j)
                        for (int iy = ty * kTileY; iy < std::min(o.ny, (ty + 1) * kTileY); ++iy)
                            for (int ix = tx * kTileX; ix < std::min(o.nx, (tx + 1) * kTileX); ++ix) {
                                size_t id = ((size_t)j * o.ny + iy) * o.nx + ix;
                                if (t.pi_first[id] + 1 <= t.pi_last[id] - 1) {
                                    k0 = std::min<int64_t>(k0, t.pi_first[id] + 1);
                                    k1 = std::max<int64_t>(k1, t.pi_last[id] - 1);
                                }
                            }
                    const double xa = ((double)tx * kTileX - 0.5 * o.nx) * o.dx, xb = xa + (kTileX - 1) * o.dx;
                    const double ya = ((double)ty * kTileY - 0.5 * o.ny) * o.dy, yb = ya + (kTileY - 1) * o.dy;
                    const double zb = (double)ch * kChunkZ * o.dz;
                    for (int64_t k = k0; k <= k1; ++k) {
                        const double lam = (double)k * o.dlam;
                        const double c = std::cos(lam + o.lam0), s = std::sin(lam + o.lam0);
                        const double zc = o.z0 + o.h * lam;
                        double cmin = 1e300, cmax = -1e300, pmin = 1e300, pmax = -1e300;
                        const double cx[4] = {xa, xb, xa, xb}, cy[4] = {ya, ya, yb, yb};
                        for (int q = 0; q < 4; ++q) {
                            double col, sc;
                            ray_col_scale(o, cx[q], cy[q], c, s, col, sc);
                            const double p0 = sc * (zb - zc) + 0.5 * (nr - 1) + 1.5;
                            const double p1 = p0 + sc * (kChunkZ - 1) * o.dz;
                            cmin = std::min(cmin, col); cmax = std::max(cmax, col);
                            pmin = std::min(pmin, std::min(p0, p1)); pmax = std::max(pmax, std::max(p0, p1));
                        }
                        bw = std::max(bw, (int)(std::floor(cmax) - std::floor(cmin)) + 3);
                        bh = std::max(bh, (int)(std::floor(pmax) - std::floor(pmin)) + 4);
                    }
                }
        t.fp_cols = std::min(bw, nc);
        t.fp_rows = std::min(bh, nr + 2);
    }
    // ---- sliding-window backprojection prerequisites (backproject.cu k_bp_window):
    // per column, interior windows [k_first+1, k_last-1] non-empty and nondecreasing in z,
    // and the largest number of slices whose interior windows contain a common view.
    {
        bool mono = true;
        int mact = 0;
        #pragma omp parallel for schedule(static) reduction(&&:mono) reduction(max:mact)
        for (int iy = 0; iy < o.ny; ++iy)
            for (int ix = 0; ix < o.nx; ++ix) {
                const size_t c = (size_t)iy * o.nx + ix, plane = (size_t)o.nx * o.ny;
                if (t.pi_last[c] < t.pi_first[c]) continue;            // outside U: whole column empty
                int lo = 0;
                for (int j = 0; j < o.nz; ++j) {
                    const int a = t.pi_first[c + j * plane] + 1, b = t.pi_last[c + j * plane] - 1;
                    if (a > b) mono = false;
                    if (j > 0 && (a < t.pi_first[c + (j - 1) * plane] + 1 || b < t.pi_last[c + (j - 1) * plane] - 1))
                        mono = false;
                    // slices active at view a (the newest): those with b_j' >= a
                    while (lo < j && t.pi_last[c + lo * plane] - 1 < a) ++lo;
                    mact = std::max(mact, j - lo + 1);
                }
            }
        t.windows_monotone = mono;
        t.max_active = mact;
        // full-column tile footprint: column span only (rows = the whole detector)
        const int ntx = (o.nx + kTileX - 1) / kTileX, nty = (o.ny + kTileY - 1) / kTileY;
        int bw = 0;
        #pragma omp parallel for collapse(2) schedule(dynamic, 1) reduction(max:bw)
        for (int ty = 0; ty < nty; ++ty)
            for (int tx = 0; tx < ntx; ++tx) {
                int64_t k0 = INT64_MAX, k1 = INT64_MIN;
                for (int iy = ty * kTileY; iy < std::min(o.ny, (ty + 1) * kTileY); ++iy)
                    for (int ix = tx * kTileX; ix < std::min(o.nx, (tx + 1) * kTileX); ++ix) {
                        const size_t c = (size_t)iy * o.nx + ix, plane = (size_t)o.nx * o.ny;
                        if (t.pi_last[c] < t.pi_first[c]) continue;
                        k0 = std::min<int64_t>(k0, t.pi_first[c] + 1);
                        k1 = std::max<int64_t>(k1, t.pi_last[c + (o.nz - 1) * plane] - 1);
                    }
                const double xa = ((double)tx * kTileX - 0.5 * o.nx) * o.dx, xb = xa + (kTileX - 1) * o.dx;
                const double ya = ((double)ty * kTileY - 0.5 * o.ny) * o.dy, yb = ya + (kTileY - 1) * o.dy;
                for (int64_t k = k0; k <= k1; ++k) {
                    const double lam = (double)k * o.dlam;
                    const double c = std::cos(lam + o.lam0), s = std::sin(lam + o.lam0);
                    double cmin = 1e300, cmax = -1e300;
                    const double cx[4] = {xa, xb, xa, xb}, cy[4] = {ya, ya, yb, yb};
                    for (int q = 0; q < 4; ++q) {
                        double col, sc;
                        ray_col_scale(o, cx[q], cy[q], c, s, col, sc);
                        cmin = std::min(cmin, col); cmax = std::max(cmax, col);
                    }
                    bw = std::max(bw, (int)(std::floor(cmax) - std::floor(cmin)) + 3);
                }
            }
        t.fp_cols_column = std::min(bw, nc);

        // TMEM-window kernel: per warp (8x4 columns), the span of slices between the oldest slice
        // not closed by every lane (warp-uniform flush point) and the newest slice open in any lane
        int span = 0, span2 = 0;
        if (t.windows_monotone) {
            const int nwx = (o.nx + 7) / 8, nwy = (o.ny + 3) / 4;
            #pragma omp parallel for collapse(2) schedule(dynamic, 4) reduction(max:span, span2)
            for (int wy = 0; wy < nwy; ++wy)
                for (int wx = 0; wx < nwx; ++wx) {
                    std::vector<size_t> cols;
                    for (int ly = 0; ly < 4; ++ly)
                        for (int lx = 0; lx < 8; ++lx) {
                            const int ix = wx * 8 + lx, iy = wy * 4 + ly;
                            if (ix >= o.nx || iy >= o.ny) continue;
                            const size_t c = (size_t)iy * o.nx + ix;
                            if (t.pi_last[c] >= t.pi_first[c]) cols.push_back(c);
                        }
                    if (cols.empty()) continue;
                    const size_t plane = (size_t)o.nx * o.ny;
                    int64_t kmin = INT64_MAX, kmax = INT64_MIN;
                    for (size_t c : cols) {
                        kmin = std::min<int64_t>(kmin, t.pi_first[c] + 1);
                        kmax = std::max<int64_t>(kmax, t.pi_last[c + (o.nz - 1) * plane]);
                    }
                    std::vector<int> lo(cols.size(), 0), hi(cols.size(), -1);
                    int tf_prev = INT32_MAX;
                    for (int64_t k = kmin; k <= kmax; ++k) {
                        int tf = INT32_MAX, th = -1;
                        for (size_t q = 0; q < cols.size(); ++q) {
                            const size_t c = cols[q];
                            while (hi[q] + 1 < o.nz && t.pi_first[c + (hi[q] + 1) * plane] + 1 <= k) ++hi[q];
                            while (lo[q] <= hi[q] && t.pi_last[c + lo[q] * plane] <= k) ++lo[q];   // closes at k_last
                            tf = std::min(tf, lo[q]);
                            th = std::max(th, hi[q]);
                        }
                        if (th >= tf) span = std::max(span, th - tf + 1);
                        // views k-1, k in one pass: flushed up to the k-1 point, open up to k
                        const int tf2 = std::min(tf, tf_prev);
                        if (th >= tf2) span2 = std::max(span2, th - tf2 + 1);
                        tf_prev = tf;
                    }
                }
        }
        t.warp_span = span;
        t.warp_span2 = std::max(span, span2);
    }
    return t.td_covered ? KATS_OK : KATS_WARN_TD_NOT_COVERED;
}

}  // namespace kats
