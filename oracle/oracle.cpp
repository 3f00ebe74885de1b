/*
 * oracle.cpp — TEST INFRASTRUCTURE ONLY.  Plain, slow, double-precision CPU
 * Katsevich reconstruction for helical cone-beam CT with a curved detector,
 * written directly from arXiv 2201.02309 §II.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code with the
 * CUDA product path (paper_2201_02309_b200/): its own geometry struct, its own
 * PI-line solver (bisection), its own ψ̂ root finder (scan + bisection), its
 * own filter (direct-sum Hilbert) and backprojection.
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".
 *
 * NEXT-4 flat-detector variant (ora_geom.flat = 1; reading A27): the same seven steps in
 * flat-detector coordinates (u, w) on the plane at distance D (Noo et al. 2003, the implementation
 * PAPER.md l.115 cites): derivative at constant ray direction (∂_λ + (u²+D²)/D ∂_u + uw/D ∂_w),
 * length weight D/√(D²+u²+w²), κ-lines w_κ(u,ψ) = DP/(2πR)(ψ + (ψ/tanψ) u/D) (Eq. 11 divided by
 * cos α, u = D tan α), Hilbert kernel 1/(π(u−u')) along u, no post-cosine (the flat g^F equals the
 * curved g^F of the same ray), backprojection at u* = D x·e_t/v*, w* = D (z − z_src)/v*.
 * Every function cites the passage it follows; readings of silent / ambiguous
 * points follow SURVEY.md §8(c) A1-A21 and are listed in DESIGN.md.
 *
 * Unlike the product (which uses pitch-periodic tables, P:l.174-185), the
 * oracle evaluates PI-lines, v*, α*, w* and the BP weights at ABSOLUTE
 * coordinates (z_j + kP, λ = v·Δλ) for every pitch k, solving afresh — the
 * plain definition, so periodicity is a checked property, not an assumption.
 */
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <omp.h>

extern "C" {

/* Oracle-private geometry description (mirrors the problem statement of
 * PAPER.md l.87-98, l.117, l.189, l.311-349).  Not shared with the product. */
typedef struct {
    double R, D, P, lambda0, z0, r_fov;      /* helix radius, src-det distance, pitch, start angle/height, FOV radius */
    int32_t n_rows; double d_w;              /* w_m = (m-(n_rows-1)/2) d_w   (P:l.340) */
    int32_t n_cols; double d_alpha, alpha_offset; /* α_l = (l-(n_cols-1)/2+off) d_alpha (P:l.328) */
    int32_t views_per_turn;                  /* Δλ = 2π / views_per_turn */
    int32_t nx, ny; double dx, dy;           /* x_i = (i - nx/2) dx  (P:l.316) */
    int32_t nz;                              /* slices per pitch: z_j = j P / nz (P:l.357, l.740) */
    int32_t n_psi;                           /* κ-lines (0 -> 2 n_rows + 1) */
    int32_t apod;                            /* NEXT-4: 1 = Hann-apodised Hilbert filter (reading A26) */
    int32_t flat;                            /* NEXT-4: 1 = flat detector: columns u_l = (l-(n_cols-1)/2+off) d_alpha
                                                [mm on the plane at distance D] (reading A27) */
} ora_geom;

}  // extern "C"

namespace {

const double PI = 3.14159265358979323846;

struct G {
    ora_geom g;
    double dlam, h, r_fov, alpha_m, psi_max, dpsi, kappa_scale;
    int n_psi;
};

G make(const ora_geom *in)
{
    G o; o.g = *in;
    o.dlam = 2.0 * PI / in->views_per_turn;
    o.h = in->P / (2.0 * PI);                               /* h = P/2π */
    double hx = 0.5 * in->nx * in->dx, hy = 0.5 * in->ny * in->dy;
    o.r_fov = in->r_fov > 0 ? in->r_fov : std::sqrt(hx * hx + hy * hy) * (1.0 + 1e-9);  /* A17 */
    o.alpha_m = std::asin(o.r_fov / in->R);                 /* α_m = arcsin(r/R), P:l.133 */
    o.psi_max = PI / 2 + o.alpha_m;                         /* ψ ∈ [-π/2-α_m, π/2+α_m], P:l.132 */
    o.n_psi = in->n_psi > 0 ? in->n_psi : 2 * in->n_rows + 1;   /* A6 */
    o.dpsi = 2.0 * o.psi_max / (o.n_psi - 1);
    o.kappa_scale = in->D * in->P / (2.0 * PI * in->R);     /* DP/(2πR), Eq. (11) P:l.135 */
    return o;
}

/* detector column coordinate: α_l (curved, rad) or u_l (flat, mm) */
inline double alpha_l(const G &o, int l) { return (l - 0.5 * (o.g.n_cols - 1) + o.g.alpha_offset) * o.g.d_alpha; }
inline double w_m(const G &o, int m) { return (m - 0.5 * (o.g.n_rows - 1)) * o.g.d_w; }
inline double psi_i(const G &o, int i) { return -o.psi_max + i * o.dpsi; }
inline double x_i(const G &o, int i) { return (i - 0.5 * o.g.nx) * o.g.dx; }
inline double y_i(const G &o, int i) { return (i - 0.5 * o.g.ny) * o.g.dy; }
inline double z_j(const G &o, int j, int pitch) { return j * o.g.P / o.g.nz + pitch * o.g.P; }
inline bool in_fov(const G &o, double x, double y) { return x * x + y * y < o.r_fov * o.r_fov; }  /* U, A17 */

/* A12: snap a floor/ceil argument to the nearest integer when within 1e-9. */
inline double snap(double a)
{
    double r = std::nearbyint(a);
    return std::fabs(a - r) < 1e-9 ? r : a;
}

/* Linear-interpolation index rule of A9/A12 on a grid of n nodes: returns
 * false when pos lies outside [0, n-1] (zero contribution). */
inline bool lin_index(double pos, int n, int *idx, double *frac)
{
    double a = snap(pos);
    if (!(a >= 0.0 && a <= n - 1)) return false;
    int m = (int)std::floor(a);
    if (m >= n - 1) m = n - 2;
    if (m < 0) m = 0;          /* n == 1 degenerate */
    *idx = m; *frac = a - m;
    return true;
}

/* ---------- PI-line (P:l.104, l.194) ----------
 * The PI-line of x is the chord a(σ-δ)a(σ+δ) through x with 0 < 2δ < 2π.
 * Chord points: xy = R cosδ e_r(σ) + u R sinδ e_t(σ), z = z0 + h(σ + uδ),
 * e_r = (cos(σ+λ0), sin(σ+λ0)), e_t = (-sin(σ+λ0), cos(σ+λ0)), u ∈ [-1,1].
 * Given σ, x fixes δ = arccos((x·e_r)/R) and u = (x·e_t)/(R sinδ); σ solves
 * F(σ) = σ + u δ - (z - z0)/h = 0, bracketed by [ζ-π, ζ+π], ζ = (z-z0)/h.
 * Solved by plain bisection to machine precision. */
void pi_line(const G &o, double x, double y, double z, double *li, double *lo)
{
    const double R = o.g.R, lam0 = o.g.lambda0;
    const double zeta = (z - o.g.z0) / o.h;
    auto F = [&](double s, double *dd) {
        double c = std::cos(s + lam0), sn = std::sin(s + lam0);
        double cr = (x * c + y * sn) / R;
        cr = std::max(-1.0, std::min(1.0, cr));
        double d = std::acos(cr);
        double u = (-x * sn + y * c) / (R * std::sin(d));
        *dd = d;
        return s + u * d - zeta;
    };
    double a = zeta - PI, b = zeta + PI, d;
    for (int it = 0; it < 200; ++it) {
        double m = 0.5 * (a + b);
        if (m == a || m == b) break;
        if (F(m, &d) < 0.0) a = m; else b = m;
    }
    double s = 0.5 * (a + b);
    F(s, &d);
    *li = s - d;
    *lo = s + d;
}

/* ---------- κ-line height, Eq. (11) P:l.134-136 ----------
 * flat (A27): the same κ-plane met by the plane at distance D: Eq. (11) / cos α at u = D tan α,
 * i.e. DP/(2πR) (ψ + (ψ/tanψ) u/D) — a straight line in (u, w) */
double w_kappa(const G &o, double alpha, double psi)
{
    double r = std::fabs(psi) < 1e-8 ? 1.0 - psi * psi / 3.0 : psi / std::tan(psi);  /* ψ/tanψ -> 1 */
    if (o.g.flat) return o.kappa_scale * (psi + r * alpha / o.g.D);
    return o.kappa_scale * (psi * std::cos(alpha) + r * std::sin(alpha));
}

/* ---------- ψ̂(α, w): "angle ψ of the smallest absolute value" with
 * w = w_κ(α, ψ)  (P:l.147-150).  Reading A8: the first root met moving out
 * from ψ = 0 (toward +ψ if w > w_κ(α,0), else toward -ψ) within
 * [-ψ_max, ψ_max]; none -> undefined.  Fine scan + bisection. */
bool psi_hat(const G &o, double alpha, double w, double *out)
{
    double f0 = w_kappa(o, alpha, 0.0) - w;
    if (f0 == 0.0) { *out = 0.0; return true; }
    const double dir = f0 < 0.0 ? 1.0 : -1.0;   /* w above w_κ(α,0): go to +ψ */
    const int NS = 20000;
    double prev_p = 0.0, prev_f = f0;
    for (int k = 1; k <= NS; ++k) {
        double p = dir * o.psi_max * k / NS;
        double f = w_kappa(o, alpha, p) - w;
        if ((f >= 0.0) != (prev_f >= 0.0) || f == 0.0) {
            double a = prev_p, b = p, fa = prev_f;
            for (int it = 0; it < 200; ++it) {
                double m = 0.5 * (a + b);
                if (m == a || m == b) break;
                double fm = w_kappa(o, alpha, m) - w;
                if ((fm >= 0.0) == (fa >= 0.0) && fm != 0.0) { a = m; fa = fm; } else b = m;
            }
            *out = 0.5 * (a + b);
            return true;
        }
        prev_p = p; prev_f = f;
    }
    return false;
}

/* ---------- BP end weights (A11, A12) ----------
 * t_i = λ_i/Δλ, t_o = λ_o/Δλ, view k owns the cell [k-½, k+½];
 * ω_k = |[k-½,k+½] ∩ [t_i,t_o]|, k_first = ⌊t_i+½⌋, k_last = ⌈t_o-½⌉. */
void bp_weights(const G &o, double li, double lo, int64_t *kf, int64_t *kl, double *wf, double *wl)
{
    double ti = li / o.dlam, to = lo / o.dlam;
    int64_t a = (int64_t)std::floor(snap(ti + 0.5));
    int64_t b = (int64_t)std::ceil(snap(to - 0.5));
    auto omega = [&](int64_t k) {
        double lo_ = std::max((double)k - 0.5, ti), hi_ = std::min((double)k + 0.5, to);
        return std::max(0.0, hi_ - lo_);
    };
    *kf = a; *kl = b; *wf = omega(a); *wl = omega(b);
}

/* Slab of pitch k (P:l.234-246): BP views [K_lo, K_hi] over
 * all in-FOV voxels of the pitch, plus one derivative halo view each side. */
void pitch_bp_range(const G &o, int pitch, int64_t *Klo, int64_t *Khi)
{
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    const int nx = o.g.nx, ny = o.g.ny, nz = o.g.nz;
    #pragma omp parallel for collapse(2) reduction(min:lo) reduction(max:hi) schedule(dynamic, 4)
    for (int j = 0; j < nz; ++j)
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix) {
                double x = x_i(o, ix), y = y_i(o, iy);
                if (!in_fov(o, x, y)) continue;
                double li, lo_;
                pi_line(o, x, y, z_j(o, j, pitch), &li, &lo_);
                int64_t kf, kl; double wf, wl;
                bp_weights(o, li, lo_, &kf, &kl, &wf, &wl);
                lo = std::min(lo, kf); hi = std::max(hi, kl);
            }
    *Klo = lo; *Khi = hi;
}

/* ---------- Rebinning maps, pre-calculated once (P:l.174, l.193) ----------
 * Forward: row position of w_κ(α_l, ψ_i) (Eq. 11) on the w grid.
 * Backward: ψ-grid position of ψ̂(α_l, w_m) (Eq. 14, reading A8).
 * Index/fraction in the canonical A12 form; idx = -1 marks "0 contribution". */
struct Rebin {
    std::vector<int32_t> fi, bi;
    std::vector<double> ff, bf;
};

Rebin rebin_maps(const G &o)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols, np = o.n_psi;
    Rebin rb;
    rb.fi.assign((size_t)np * nc, -1); rb.ff.assign((size_t)np * nc, 0.0);
    rb.bi.assign((size_t)nr * nc, -1); rb.bf.assign((size_t)nr * nc, 0.0);
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < np; ++i)
        for (int l = 0; l < nc; ++l) {
            double pos = w_kappa(o, alpha_l(o, l), psi_i(o, i)) / o.g.d_w + 0.5 * (nr - 1);
            int m; double f;
            if (lin_index(pos, nr, &m, &f)) { rb.fi[(size_t)i * nc + l] = m; rb.ff[(size_t)i * nc + l] = f; }
        }
    #pragma omp parallel for schedule(dynamic, 1)
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            double ph; int i; double f;
            if (psi_hat(o, alpha_l(o, l), w_m(o, m), &ph) && lin_index((ph + o.psi_max) / o.dpsi, np, &i, &f)) {
                rb.bi[(size_t)m * nc + l] = i; rb.bf[(size_t)m * nc + l] = f;
            }
        }
    return rb;
}

/* ---------- Filtering steps 1-6 for one view (P:l.117-154, Eqs. 8-15) ----------
 * g(v) at sino[v - s0]; writes optional stage outputs (double, [rows][cols] or
 * [n_psi][cols]).  Discretisation readings: A5 (centred differences, one-sided
 * at the α edges), A9 (linear rebins, 0 outside), A10 (band-limited Hilbert). */
/* NEXT-4, reading A26: the Hann-apodised Hilbert filter — step 4's kernel with its frequency response
 * -i sgn(σ) multiplied by the Hann window cos²(πσΔα) (σ in cycles per radian; 1 at DC, 0 at the
 * Nyquist frequency 1/(2Δα)), i.e. K applied to the κ-line smoothed by [1/4, 1/2, 1/4] along α
 * (zeros beyond the detector columns, as Eq. 12's sum).  The smoothing matrix is symmetric, so it is
 * its own transpose in the adjoint. */
void hann_smooth(const G &o, double *line)
{
    const int nc = o.g.n_cols;
    std::vector<double> t(line, line + nc);
    for (int l = 0; l < nc; ++l)
        line[l] = 0.5 * t[l] + 0.25 * ((l > 0 ? t[l - 1] : 0.0) + (l + 1 < nc ? t[l + 1] : 0.0));
}

/* Steps 2-6 of one view from its g1 = step 1's output [rows][cols] (double). */
void filter_from_g1(const G &o, const double *g1, const std::vector<double> &Kh, const Rebin &rb,
                    double *g2o, double *g3o, double *g4o, double *gFo)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols, np = o.n_psi;
    std::vector<double> g2((size_t)nr * nc), g3((size_t)np * nc), g4((size_t)np * nc);
    /* Step 2, Eq. (9): g2 = D/sqrt(D²+w²) g1 (flat, A27: D/sqrt(D²+u²+w²), the cosine of the ray to the
     * central ray) */
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            const double uu = o.g.flat ? alpha_l(o, l) * alpha_l(o, l) : 0.0;
            const double wgt = o.g.D / std::sqrt(o.g.D * o.g.D + uu + w_m(o, m) * w_m(o, m));
            g2[(size_t)m * nc + l] = wgt * g1[(size_t)m * nc + l];
        }
    /* Step 3, Eqs. (10)-(11): g3(α,ψ) = g2(α, w_κ(α,ψ)), linear in w, 0 outside */
    for (int i = 0; i < np; ++i)
        for (int l = 0; l < nc; ++l) {
            size_t t = (size_t)i * nc + l;
            int m = rb.fi[t]; double f = rb.ff[t];
            g3[t] = m < 0 ? 0.0 : (1.0 - f) * g2[(size_t)m * nc + l] + f * g2[(size_t)(m + 1) * nc + l];
        }
    /* Step 4, Eq. (12) with h_H(s) = 1/(πs) (Eq. e4): g4(α_l) = Σ_l' K[l-l'] g3(α_l')
     * (apodised variant, A26: on the Hann-smoothed κ-line; the g3 stage output stays unsmoothed) */
    std::vector<double> g3a;
    const double *g3h = g3.data();
    if (o.g.apod) {
        g3a = g3;
        for (int i = 0; i < np; ++i) hann_smooth(o, g3a.data() + (size_t)i * nc);
        g3h = g3a.data();
    }
    for (int i = 0; i < np; ++i)
        for (int l = 0; l < nc; ++l) {
            double acc = 0.0;
            for (int lp = 0; lp < nc; ++lp) acc += Kh[(size_t)(l - lp + nc - 1)] * g3h[(size_t)i * nc + lp];
            g4[(size_t)i * nc + l] = acc;
        }
    /* Steps 5-6, Eqs. (13)-(15): g5 = g4(α, ψ̂(α,w)), linear in ψ; gF = cosα g5 */
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            size_t t = (size_t)m * nc + l;
            int i = rb.bi[t]; double f = rb.bf[t];
            double val = i < 0 ? 0.0 : (1.0 - f) * g4[(size_t)i * nc + l] + f * g4[(size_t)(i + 1) * nc + l];
            if (gFo) gFo[t] = (o.g.flat ? 1.0 : std::cos(alpha_l(o, l))) * val;   /* flat: no post-cosine (A27) */
        }
    if (g2o) std::memcpy(g2o, g2.data(), sizeof(double) * g2.size());
    if (g3o) std::memcpy(g3o, g3.data(), sizeof(double) * g3.size());
    if (g4o) std::memcpy(g4o, g4.data(), sizeof(double) * g4.size());
}

/* ---------- Filtering steps 1-6 for one view (P:l.117-154, Eqs. 8-15) ----------
 * g(v) at sino[v - s0]; writes optional stage outputs (double, [rows][cols] or
 * [n_psi][cols]).  Discretisation readings: A5 (centred differences, one-sided
 * at the α edges), A9 (linear rebins, 0 outside), A10 (band-limited Hilbert). */
void filter_view(const G &o, const float *sino, int64_t s0, int64_t v,
                 const std::vector<double> &Kh, const Rebin &rb,
                 double *g2o, double *g3o, double *g4o, double *gFo)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols;
    auto g = [&](int64_t vv, int m, int l) { return (double)sino[((vv - s0) * nr + m) * (int64_t)nc + l]; };
    std::vector<double> g1((size_t)nr * nc);
    /* Step 1, Eq. (8): g1 = (∂_q + ∂_α) g |_{q=λ}; flat (A27): the derivative at constant ray direction
     * on the plane, (∂_q + (u²+D²)/D ∂_u + u w/D ∂_w) g, the w difference centred like α (one-sided at
     * the row edges) */
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            double dq = (g(v + 1, m, l) - g(v - 1, m, l)) / (2.0 * o.dlam);
            double da;
            if (l == 0) da = (g(v, m, 1) - g(v, m, 0)) / o.g.d_alpha;
            else if (l == nc - 1) da = (g(v, m, nc - 1) - g(v, m, nc - 2)) / o.g.d_alpha;
            else da = (g(v, m, l + 1) - g(v, m, l - 1)) / (2.0 * o.g.d_alpha);
            if (o.g.flat) {
                const double u = alpha_l(o, l), w = w_m(o, m), D = o.g.D;
                double dw;
                if (nr == 1) dw = 0.0;
                else if (m == 0) dw = (g(v, 1, l) - g(v, 0, l)) / o.g.d_w;
                else if (m == nr - 1) dw = (g(v, nr - 1, l) - g(v, nr - 2, l)) / o.g.d_w;
                else dw = (g(v, m + 1, l) - g(v, m - 1, l)) / (2.0 * o.g.d_w);
                g1[(size_t)m * nc + l] = dq + (u * u + D * D) / D * da + u * w / D * dw;
            } else {
                g1[(size_t)m * nc + l] = dq + da;
            }
        }
    filter_from_g1(o, g1.data(), Kh, rb, g2o, g3o, g4o, gFo);
}

/* NEXT-4: Noo's half-sample derivative, the 2x2x2-cube scheme of [Noo2003a] (the
 * reference PAPER.md l.115 cites for implementing Eq. (8); reading A25).  g1 lives at the
 * cube centre (λ_{k+½}, α_{l+½}, w_{m+½}) of raw views k, k+1, columns l, l+1 and rows m, m+1:
 *   ∂_q g ≈ 1/(4Δλ) Σ_{i,j ∈ {0,1}} [g(k+1, m+j, l+i) - g(k, m+j, l+i)]
 *   ∂_α g ≈ 1/(4Δα) Σ_{i,j ∈ {0,1}} [g(k+i, m+j, l+1) - g(k+i, m+j, l)]
 *   g1 = ∂_q g + ∂_α g                                             (Eq. 8's chain rule)
 * on (n_rows - 1) x (n_cols - 1) half-shifted samples; o is the PHYSICAL geometry. */
void deriv_half(const G &o, const float *sino, int64_t s0, int64_t k, double *g1)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols;
    auto g = [&](int64_t vv, int m, int l) { return (double)sino[((vv - s0) * nr + m) * (int64_t)nc + l]; };
    for (int m = 0; m + 1 < nr; ++m)
        for (int l = 0; l + 1 < nc; ++l) {
            double dq = 0.0, da = 0.0;
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) {
                    dq += g(k + 1, m + j, l + i) - g(k, m + j, l + i);
                    da += g(k + i, m + j, l + 1) - g(k + i, m + j, l);
                }
            g1[(size_t)m * (nc - 1) + l] = dq / (4.0 * o.dlam) + da / (4.0 * o.g.d_alpha);
        }
}

/* Band-limited kernel of h_H(sin(α-α')) dα' (A10):
 * K[d] = Δα (1 - cos πd) / (π sin(dΔα)), K[0] = 0; 1 - cos πd = 1 - (-1)^d.
 * flat (A27): h_H(u-u') du' on the uniform u grid, K[d] = Δu (1 - cos πd) / (π dΔu) = (1 - cos πd)/(πd). */
std::vector<double> hilbert_kernel(const G &o)
{
    const int nc = o.g.n_cols;
    std::vector<double> K((size_t)(2 * nc - 1), 0.0);
    for (int d = -(nc - 1); d <= nc - 1; ++d) {
        if (d == 0) continue;
        double one_minus_cos = (d % 2 == 0) ? 0.0 : 2.0;
        K[(size_t)(d + nc - 1)] = o.g.flat ? one_minus_cos / (PI * d)
                                           : o.g.d_alpha * one_minus_cos / (PI * std::sin(d * o.g.d_alpha));
    }
    return K;
}

/* Detector coordinates of voxel (x, y, z) at view angle λ (index k): v*, the column coordinate
 * (α* curved, u* flat) and w* (P:l.161-170; flat A27). */
inline void project_voxel(const G &o, double x, double y, double z, double lam, double *vstar, double *acoord,
                          double *wstar)
{
    double c = std::cos(lam + o.g.lambda0), s = std::sin(lam + o.g.lambda0);
    *vstar = o.g.R - x * c - y * s;
    const double ut = -x * s + y * c, dz = z - o.g.z0 - o.h * lam;
    if (o.g.flat) {
        *acoord = o.g.D * ut / *vstar;                       /* u* = D x·e_t / v* */
        *wstar = o.g.D * dz / *vstar;                        /* w* = D (z - z_src) / v* */
    } else {
        *acoord = std::atan(ut / *vstar);                    /* α* (P:l.166) */
        *wstar = o.g.D * std::cos(*acoord) / *vstar * dz;    /* w* (P:l.170) */
    }
}

/* Bilinear sample of gF(view) at (α*, w*); 0 outside the sample range (A9). */
inline double sample(const G &o, const double *gv, double alpha, double w)
{
    int l, m; double fa, fw;
    if (!lin_index(alpha / o.g.d_alpha + 0.5 * (o.g.n_cols - 1) - o.g.alpha_offset, o.g.n_cols, &l, &fa)) return 0.0;
    if (!lin_index(w / o.g.d_w + 0.5 * (o.g.n_rows - 1), o.g.n_rows, &m, &fw)) return 0.0;
    const int nc = o.g.n_cols;
    double a0 = (1.0 - fa) * gv[(size_t)m * nc + l] + fa * gv[(size_t)m * nc + l + 1];
    double a1 = (1.0 - fa) * gv[(size_t)(m + 1) * nc + l] + fa * gv[(size_t)(m + 1) * nc + l + 1];
    return (1.0 - fw) * a0 + fw * a1;
}

/* ---------- Step 7 backprojection for one voxel (P:l.155-171; O5) ----------
 * f(x) = (1/2π) ∫_{λi}^{λo} dλ gF(λ, α*, w*)/v*  with the rectangle rule and
 * fractional end weights (A11):  f = Δλ/2π Σ_k ω_k gF_k(α*_k, w*_k) / v*_k,
 * v* = R - x cos(λ+λ0) - y sin(λ+λ0)                       (P:l.161)
 * α* = arctan((-x sin(λ+λ0) + y cos(λ+λ0)) / v*)           (P:l.166)
 * w* = D cos α* / v* · (z - z0 - P λ / 2π)                 (P:l.170)
 * gF views are indexed absolutely: view k at gF + (k - gF0) * rows*cols. */
double bp_voxel(const G &o, double x, double y, double z, const double *gF, int64_t gF0, int64_t gFn, int *oob)
{
    if (!in_fov(o, x, y)) return 0.0;
    double li, lo;
    pi_line(o, x, y, z, &li, &lo);
    int64_t kf, kl; double wf, wl;
    bp_weights(o, li, lo, &kf, &kl, &wf, &wl);
    if (kf < gF0 || kl >= gF0 + gFn) { if (oob) *oob = 1; return 0.0; }
    const size_t vs = (size_t)o.g.n_rows * o.g.n_cols;
    double acc = 0.0;
    for (int64_t k = kf; k <= kl; ++k) {
        double om = (k == kf) ? wf : (k == kl) ? wl : 1.0;   /* kf == kl: wf = t_o - t_i */
        double vstar, astar, wstar;
        project_voxel(o, x, y, z, k * o.dlam, &vstar, &astar, &wstar);
        acc += om * sample(o, gF + (size_t)(k - gF0) * vs, astar, wstar) / vstar;
    }
    return acc * o.dlam / (2.0 * PI);      /* +1/2π (step 7, P:l.157; reading A3) */
}

/* ---------- Adjoint (NEXT-1): the transpose of the linear map
 * sinogram -> volume above, written step by step in reverse order.  Pinned by
 * the dot-product identity <A x, y> = <x, A^T y> against the forward
 * (tests/test_oracle_adjoint.py), per stage and for the whole layer. */

/* Transpose of sample(): scatter `val` onto the four bilinear taps. */
inline void sample_T(const G &o, double *gvT, double alpha, double w, double val)
{
    int l, m; double fa, fw;
    if (!lin_index(alpha / o.g.d_alpha + 0.5 * (o.g.n_cols - 1) - o.g.alpha_offset, o.g.n_cols, &l, &fa)) return;
    if (!lin_index(w / o.g.d_w + 0.5 * (o.g.n_rows - 1), o.g.n_rows, &m, &fw)) return;
    const int nc = o.g.n_cols;
    gvT[(size_t)m * nc + l] += (1.0 - fw) * (1.0 - fa) * val;
    gvT[(size_t)m * nc + l + 1] += (1.0 - fw) * fa * val;
    gvT[(size_t)(m + 1) * nc + l] += fw * (1.0 - fa) * val;
    gvT[(size_t)(m + 1) * nc + l + 1] += fw * fa * val;
}

/* Transpose of bp_voxel() for one voxel: adds y * d f / d gF into gFT. */
void bp_voxel_T(const G &o, double x, double y_, double z, double yv, double *gFT, int64_t gF0, int64_t gFn)
{
    if (!in_fov(o, x, y_)) return;
    double li, lo;
    pi_line(o, x, y_, z, &li, &lo);
    int64_t kf, kl; double wf, wl;
    bp_weights(o, li, lo, &kf, &kl, &wf, &wl);
    if (kf < gF0 || kl >= gF0 + gFn) return;
    const size_t vs = (size_t)o.g.n_rows * o.g.n_cols;
    for (int64_t k = kf; k <= kl; ++k) {
        double om = (k == kf) ? wf : (k == kl) ? wl : 1.0;
        double vstar, astar, wstar;
        project_voxel(o, x, y_, z, k * o.dlam, &vstar, &astar, &wstar);
        sample_T(o, gFT + (size_t)(k - gF0) * vs, astar, wstar, yv * om / vstar * o.dlam / (2.0 * PI));
    }
}

/* Transpose of filter_view() steps 2-6 for one view: gFT (rows x cols) ->
 * g1T (rows x cols) = (step 2..6)^T gFT; step 1's stencil is applied by the caller. */
void filter_view_T(const G &o, const std::vector<double> &Kh, const Rebin &rb, const double *gFT, double *g1T)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols, np = o.n_psi;
    std::vector<double> g4T((size_t)np * nc, 0.0), g3T((size_t)np * nc, 0.0), g2T((size_t)nr * nc, 0.0);
    /* steps 5-6^T: gF = cos(alpha) lerp_psi(g4) */
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            size_t t = (size_t)m * nc + l;
            int i = rb.bi[t]; double f = rb.bf[t];
            if (i < 0) continue;
            double v = (o.g.flat ? 1.0 : std::cos(alpha_l(o, l))) * gFT[t];
            g4T[(size_t)i * nc + l] += (1.0 - f) * v;
            g4T[(size_t)(i + 1) * nc + l] += f * v;
        }
    /* step 4^T: g4(l) = sum_l' K[l-l'] g3(l')  =>  g3T(l') = sum_l K[l-l'] g4T(l) */
    for (int i = 0; i < np; ++i)
        for (int lp = 0; lp < nc; ++lp) {
            double acc = 0.0;
            for (int l = 0; l < nc; ++l) acc += Kh[(size_t)(l - lp + nc - 1)] * g4T[(size_t)i * nc + l];
            g3T[(size_t)i * nc + lp] = acc;
        }
    if (o.g.apod)                                 /* the symmetric smoothing is its own transpose */
        for (int i = 0; i < np; ++i) hann_smooth(o, g3T.data() + (size_t)i * nc);
    /* step 3^T: g3 = lerp_w(g2) */
    for (int i = 0; i < np; ++i)
        for (int l = 0; l < nc; ++l) {
            size_t t = (size_t)i * nc + l;
            int m = rb.fi[t]; double f = rb.ff[t];
            if (m < 0) continue;
            g2T[(size_t)m * nc + l] += (1.0 - f) * g3T[t];
            g2T[(size_t)(m + 1) * nc + l] += f * g3T[t];
        }
    /* step 2^T: g2 = D/sqrt(D^2 (+u^2) +w^2) g1 */
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            const double uu = o.g.flat ? alpha_l(o, l) * alpha_l(o, l) : 0.0;
            const double wgt = o.g.D / std::sqrt(o.g.D * o.g.D + uu + w_m(o, m) * w_m(o, m));
            g1T[(size_t)m * nc + l] = wgt * g2T[(size_t)m * nc + l];
        }
}

/* Step 1^T: g1(v) = (g(v+1) - g(v-1))/(2 dlam) + D_alpha g(v)  =>  scatter g1T(v). */
void deriv_T(const G &o, const double *g1T, int64_t v, double *outT, int64_t s0)
{
    const int nr = o.g.n_rows, nc = o.g.n_cols;
    auto at = [&](int64_t vv, int m, int l) -> double & { return outT[((vv - s0) * nr + m) * (int64_t)nc + l]; };
    for (int m = 0; m < nr; ++m)
        for (int l = 0; l < nc; ++l) {
            double t = g1T[(size_t)m * nc + l];
            at(v + 1, m, l) += t / (2.0 * o.dlam);
            at(v - 1, m, l) -= t / (2.0 * o.dlam);
            double ta = t, tw = 0.0;                       /* flat (A27): the u and w stencils' weights */
            if (o.g.flat) {
                const double u = alpha_l(o, l), w = w_m(o, m), D = o.g.D;
                ta = t * (u * u + D * D) / D;
                tw = t * u * w / D;
            }
            if (l == 0) { at(v, m, 1) += ta / o.g.d_alpha; at(v, m, 0) -= ta / o.g.d_alpha; }
            else if (l == nc - 1) { at(v, m, nc - 1) += ta / o.g.d_alpha; at(v, m, nc - 2) -= ta / o.g.d_alpha; }
            else { at(v, m, l + 1) += ta / (2.0 * o.g.d_alpha); at(v, m, l - 1) -= ta / (2.0 * o.g.d_alpha); }
            if (o.g.flat && nr > 1) {
                if (m == 0) { at(v, 1, l) += tw / o.g.d_w; at(v, 0, l) -= tw / o.g.d_w; }
                else if (m == nr - 1) { at(v, nr - 1, l) += tw / o.g.d_w; at(v, nr - 2, l) -= tw / o.g.d_w; }
                else { at(v, m + 1, l) += tw / (2.0 * o.g.d_w); at(v, m - 1, l) -= tw / (2.0 * o.g.d_w); }
            }
        }
}

/* ---------- NEXT-3: data generation (P:l.353-404; SPEC "simulate") ----------
 * Scan ray of detector sample (v, m, l) (P:l.87-94 helix, curved detector
 * P:l.117, l.311-349): source a(λ) = (R cos(λ+λ0), R sin(λ+λ0), z0 + hλ),
 * direction ∝ D sinα e_t − D cosα e_r + w e_z, e_r = (cos, sin, 0),
 * e_t = (−sin, cos, 0) at angle λ+λ0 — the geometry bp_voxel inverts
 * (α* = atan(u/v*), w* = D cosα* (z − z_src)/v*). */
void scan_ray(const G &o, int64_t v, int m, int l, double src[3], double dir[3])
{
    const double lam = v * o.dlam;
    const double c = std::cos(lam + o.g.lambda0), sn = std::sin(lam + o.g.lambda0);
    src[0] = o.g.R * c; src[1] = o.g.R * sn; src[2] = o.g.z0 + o.h * lam;
    const double a = alpha_l(o, l), w = w_m(o, m);
    /* curved: D sinα e_t − D cosα e_r + w e_z; flat (A27): u e_t − D e_r + w e_z */
    const double sa = o.g.flat ? a : o.g.D * std::sin(a), ca = o.g.flat ? o.g.D : o.g.D * std::cos(a);
    double d[3] = {-sa * sn - ca * c, sa * c - ca * sn, w};
    const double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    dir[0] = d[0] / n; dir[1] = d[1] / n; dir[2] = d[2] / n;
}

/* Length of a unit-speed line inside an ellipsoid {c, semi-axes a,b,c (c <= 0:
 * infinite cylinder along z), rotation φ about z}: the roots of a quadratic. */
double ellipsoid_chord(const double *e, const double o[3], const double d[3])
{
    const double cp = std::cos(e[6]), sp = std::sin(e[6]);
    const double ox = o[0] - e[0], oy = o[1] - e[1], oz = o[2] - e[2];
    const double px = (cp * ox + sp * oy) / e[3], py = (-sp * ox + cp * oy) / e[4];
    const double qx = (cp * d[0] + sp * d[1]) / e[3], qy = (-sp * d[0] + cp * d[1]) / e[4];
    double A = qx * qx + qy * qy, B = 2.0 * (px * qx + py * qy), C = px * px + py * py - 1.0;
    if (e[5] > 0.0) {
        const double pz = oz / e[5], qz = d[2] / e[5];
        A += qz * qz; B += 2.0 * pz * qz; C += pz * pz;
    }
    if (A <= 0.0) return 0.0;
    const double disc = B * B - 4.0 * A * C;
    return disc > 0.0 ? std::sqrt(disc) / A : 0.0;
}

/* Philox4x32-10 (Salmon et al., SC'11): counter-based stream, identical on the GPU side. */
void philox(uint32_t ctr[4], const uint32_t key[2])
{
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0], p1 = (uint64_t)0xCD9E8D57u * ctr[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ ctr[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ ctr[3] ^ k1;
        ctr[1] = (uint32_t)p1; ctr[3] = (uint32_t)p0; ctr[0] = n0; ctr[2] = n2;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
}

/* Stream of one sample: counter (index lo, index hi, draw, 0), key = seed; two
 * uniforms in (0, 1) with 53 bits per Philox call. */
struct Stream {
    uint32_t key[2]; uint64_t idx; uint32_t draw = 0; double buf[2]; int left = 0;
    double uniform()
    {
        if (!left) {
            uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), draw++, 0u};
            philox(c, key);
            buf[0] = ((double)((((uint64_t)(c[0] >> 5)) << 26) | (c[1] >> 6)) + 0.5) * 0x1p-53;
            buf[1] = ((double)((((uint64_t)(c[2] >> 5)) << 26) | (c[3] >> 6)) + 0.5) * 0x1p-53;
            left = 2;
        }
        return buf[2 - left--];
    }
};

/* Poisson(lam) for lam >= 10: PTRS, transformed rejection with squeeze
 * (W. Hörmann, Insurance: Math. Econ. 12, 1993). */
int64_t poisson_ptrs(double lam, Stream &st)
{
    const double slam = std::sqrt(lam), loglam = std::log(lam);
    const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
    for (;;) {
        const double U = st.uniform() - 0.5, V = st.uniform();
        const double us = 0.5 - std::fabs(U);
        const double k = std::floor((2.0 * a / us + b) * U + lam + 0.43);
        if (us >= 0.07 && V <= vr) return (int64_t)k;
        if (k < 0.0 || (us < 0.013 && V > us)) continue;
        if (std::log(V) + std::log(invalpha) - std::log(a / (us * us) + b) <= -lam + k * loglam - std::lgamma(k + 1.0))
            return (int64_t)k;
    }
}

/* Standard normal by Box-Muller (one uniform pair per draw). */
double normal(Stream &st)
{
    const double u1 = st.uniform(), u2 = st.uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * PI * u2);
}

}  // namespace

extern "C" {

/* Derived scalars for tests: [dlam, h, r_fov, alpha_m, psi_max, dpsi, kappa_scale, n_psi] */
void ora_derived(const ora_geom *g, double *out)
{
    G o = make(g);
    out[0] = o.dlam; out[1] = o.h; out[2] = o.r_fov; out[3] = o.alpha_m;
    out[4] = o.psi_max; out[5] = o.dpsi; out[6] = o.kappa_scale; out[7] = o.n_psi;
}

void ora_pi_line(const ora_geom *g, double x, double y, double z, double *li, double *lo)
{
    G o = make(g);
    pi_line(o, x, y, z, li, lo);
}

void ora_pi_lines(const ora_geom *g, const double *pts, int64_t n, double *li, double *lo)
{
    G o = make(g);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) pi_line(o, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], li + i, lo + i);
}

double ora_w_kappa(const ora_geom *g, double alpha, double psi) { G o = make(g); return w_kappa(o, alpha, psi); }

int ora_psi_hat(const ora_geom *g, double alpha, double w, double *psi)
{
    G o = make(g);
    return psi_hat(o, alpha, w, psi) ? 1 : 0;
}

/* Hilbert kernel K[d], d = -(nc-1)..nc-1 (2nc-1 values). */
void ora_hilbert_kernel(const ora_geom *g, double *K)
{
    G o = make(g);
    std::vector<double> k = hilbert_kernel(o);
    std::memcpy(K, k.data(), sizeof(double) * k.size());
}

/* Integer/fraction tables in the canonical A12 form, for the bit-exact test.
 * fr_idx/fr_frac [n_psi][n_cols]: row index m of w_κ(α_l, ψ_i) (-1 = outside)
 * br_idx/br_frac [n_rows][n_cols]: ψ index of ψ̂(α_l, w_m) (-1 = none/outside) */
void ora_rebin_tables(const ora_geom *g, int32_t *fr_idx, double *fr_frac, int32_t *br_idx, double *br_frac)
{
    G o = make(g);
    Rebin rb = rebin_maps(o);
    std::memcpy(fr_idx, rb.fi.data(), sizeof(int32_t) * rb.fi.size());
    std::memcpy(fr_frac, rb.ff.data(), sizeof(double) * rb.ff.size());
    std::memcpy(br_idx, rb.bi.data(), sizeof(int32_t) * rb.bi.size());
    std::memcpy(br_frac, rb.bf.data(), sizeof(double) * rb.bf.size());
}

/* PI-window BP weights for every voxel of pitch `pitch` at absolute
 * coordinates (no periodicity used).  Out-of-FOV voxels get
 * kf = 0, kl = -1, weights 0.  Arrays [nz][ny][nx]. */
void ora_bp_weights(const ora_geom *g, int32_t pitch, int64_t *kf, int64_t *kl, double *wf, double *wl)
{
    G o = make(g);
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    #pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int j = 0; j < nz; ++j)
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix) {
                size_t id = ((size_t)j * ny + iy) * nx + ix;
                double x = x_i(o, ix), y = y_i(o, iy);
                if (!in_fov(o, x, y)) { kf[id] = 0; kl[id] = -1; wf[id] = 0; wl[id] = 0; continue; }
                double li, lo;
                pi_line(o, x, y, z_j(o, j, pitch), &li, &lo);
                bp_weights(o, li, lo, kf + id, kl + id, wf + id, wl + id);
            }
}

/* BP weights of selected voxels idx[n][3] = (ix, iy, j) of pitch `pitch`. */
void ora_bp_weights_voxels(const ora_geom *g, int32_t pitch, const int32_t *idx, int64_t n,
                           int64_t *kf, int64_t *kl, double *wf, double *wl)
{
    G o = make(g);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double x = x_i(o, idx[3 * i]), y = y_i(o, idx[3 * i + 1]);
        if (!in_fov(o, x, y)) { kf[i] = 0; kl[i] = -1; wf[i] = 0; wl[i] = 0; continue; }
        double li, lo;
        pi_line(o, x, y, z_j(o, idx[3 * i + 2], pitch), &li, &lo);
        bp_weights(o, li, lo, kf + i, kl + i, wf + i, wl + i);
    }
}

/* Views a pitch needs: slab [K_lo - 1, K_hi + 1]. */
void ora_pitch_slab(const ora_geom *g, int32_t pitch, int64_t *first_view, int64_t *n_views)
{
    G o = make(g);
    int64_t lo, hi;
    pitch_bp_range(o, pitch, &lo, &hi);
    *first_view = lo - 1;
    *n_views = hi - lo + 3;
}

/* Filter views [v_first, v_first + n_out) of a sinogram whose first view is
 * s0 (needs views v_first-1 .. v_first+n_out).  Optional outputs (double):
 * g2 [n_out][rows][cols], g3/g4 [n_out][n_psi][cols], gF [n_out][rows][cols]. */
/* The filter's per-geometry set-up (Hilbert kernel, rebin maps), built once so
 * bench.py's cpu_baseline can time steps 1-6 alone (test infrastructure: no
 * arithmetic differs from ora_filter, which is prepare + run + free). */
struct ora_filter_ctx { G o; std::vector<double> K; Rebin rb; };

ora_filter_ctx *ora_filter_prepare(const ora_geom *g)
{
    ora_filter_ctx *c = new ora_filter_ctx;
    c->o = make(g);
    c->K = hilbert_kernel(c->o);
    c->rb = rebin_maps(c->o);
    return c;
}

void ora_filter_free(ora_filter_ctx *c) { delete c; }

int ora_filter_run(const ora_filter_ctx *c, const float *sino, int64_t s0, int64_t sn,
                   int64_t v_first, int64_t n_out, double *g2, double *g3, double *g4, double *gF)
{
    const G &o = c->o;
    if (v_first - 1 < s0 || v_first + n_out + 1 > s0 + sn) return -1;
    const size_t rs = (size_t)o.g.n_rows * o.g.n_cols, ps = (size_t)o.n_psi * o.g.n_cols;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n_out; ++i)
        filter_view(o, sino, s0, v_first + i, c->K, c->rb,
                    g2 ? g2 + i * rs : nullptr, g3 ? g3 + i * ps : nullptr,
                    g4 ? g4 + i * ps : nullptr, gF ? gF + i * rs : nullptr);
    return 0;
}

/* Filter views [v_first, v_first + n_out) of a sinogram whose first view is
 * s0 (needs views v_first-1 .. v_first+n_out).  Optional outputs (double):
 * g2 [n_out][rows][cols], g3/g4 [n_out][n_psi][cols], gF [n_out][rows][cols]. */
int ora_filter(const ora_geom *g, const float *sino, int64_t s0, int64_t sn,
               int64_t v_first, int64_t n_out, double *g2, double *g3, double *g4, double *gF)
{
    if (v_first - 1 < s0 || v_first + n_out + 1 > s0 + sn) return -1;
    ora_filter_ctx *c = ora_filter_prepare(g);
    const int rc = ora_filter_run(c, sino, s0, sn, v_first, n_out, g2, g3, g4, gF);
    ora_filter_free(c);
    return rc;
}

/* NEXT-4: half-sample derivative of raw views (physical geometry g): g1 [n_out][rows-1][cols-1] for
 * the half-shifted views v_first + ½ .. (needs raw views v_first .. v_first + n_out). */
int ora_deriv_half(const ora_geom *g, const float *sino, int64_t s0, int64_t sn, int64_t v_first, int64_t n_out,
                   double *g1)
{
    G o = make(g);
    if (v_first < s0 || v_first + n_out + 1 > s0 + sn) return -1;
    const size_t vs = (size_t)(g->n_rows - 1) * (g->n_cols - 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_out; ++i) deriv_half(o, sino, s0, v_first + i, g1 + i * vs);
    return 0;
}

/* Steps 2-6 from step-1 output g1 [n][rows][cols] (double) in the geometry g (for the half-sample
 * derivative: the half-shifted grid's geometry, reading A25).  Outputs as ora_filter. */
void ora_filter_g1(const ora_geom *g, const double *g1, int64_t n, double *g2, double *g3, double *g4, double *gF)
{
    G o = make(g);
    std::vector<double> K = hilbert_kernel(o);
    Rebin rb = rebin_maps(o);
    const size_t rs = (size_t)g->n_rows * g->n_cols, ps = (size_t)o.n_psi * g->n_cols;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i)
        filter_from_g1(o, g1 + i * rs, K, rb, g2 ? g2 + i * rs : nullptr, g3 ? g3 + i * ps : nullptr,
                       g4 ? g4 + i * ps : nullptr, gF ? gF + i * rs : nullptr);
}

/* OpenMP threads for the following oracle calls (bench.py: single-thread vs all-core timing). */
void ora_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int ora_get_threads(void) { return omp_get_max_threads(); }

/* Backproject a full pitch volume [nz][ny][nx] from filtered views gF
 * (views gF0 .. gF0+gFn-1, absolute).  Returns 1 if some voxel's PI-window
 * fell outside the provided views (those voxels are 0). */
int ora_backproject(const ora_geom *g, int32_t pitch, const double *gF, int64_t gF0, int64_t gFn, double *vol)
{
    G o = make(g);
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    int oob_any = 0;
    #pragma omp parallel for collapse(2) schedule(dynamic, 1) reduction(|:oob_any)
    for (int j = 0; j < nz; ++j)
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix) {
                int oob = 0;
                vol[((size_t)j * ny + iy) * nx + ix] = bp_voxel(o, x_i(o, ix), y_i(o, iy), z_j(o, j, pitch), gF, gF0, gFn, &oob);
                oob_any |= oob;
            }
    return oob_any;
}

/* Backproject selected voxels: idx[n][3] = (ix, iy, j). */
int ora_backproject_voxels(const ora_geom *g, int32_t pitch, const double *gF, int64_t gF0, int64_t gFn,
                           const int32_t *idx, int64_t n, double *out)
{
    G o = make(g);
    int oob_any = 0;
    #pragma omp parallel for schedule(dynamic, 16) reduction(|:oob_any)
    for (int64_t i = 0; i < n; ++i) {
        int oob = 0;
        out[i] = bp_voxel(o, x_i(o, idx[3 * i]), y_i(o, idx[3 * i + 1]), z_j(o, idx[3 * i + 2], pitch), gF, gF0, gFn, &oob);
        oob_any |= oob;
    }
    return oob_any;
}

/* Whole reconstruction of pitches [k0, k0+np) from a sinogram (first view s0):
 * for each pitch, slice its slab (P:l.246-248), filter steps 1-6 on the slab,
 * backproject (P:l.249-262).  vol [np*nz][ny][nx] (double).
 * Returns -1 if a slab is not covered by the sinogram. */
int ora_reconstruct(const ora_geom *g, const float *sino, int64_t s0, int64_t sn,
                    int32_t k0, int32_t np, double *vol)
{
    const size_t vs = (size_t)g->nx * g->ny * g->nz;
    const size_t rs = (size_t)g->n_rows * g->n_cols;
    for (int32_t k = k0; k < k0 + np; ++k) {
        int64_t fv, nv;
        ora_pitch_slab(g, k, &fv, &nv);
        if (fv < s0 || fv + nv > s0 + sn) return -1;
        std::vector<double> gF((size_t)(nv - 2) * rs);
        ora_filter(g, sino, s0, sn, fv + 1, nv - 2, nullptr, nullptr, nullptr, gF.data());
        ora_backproject(g, k, gF.data(), fv + 1, nv - 2, vol + (size_t)(k - k0) * vs);
    }
    return 0;
}

/* Adjoint of ora_backproject for pitch `pitch`: gFT [gFn][rows][cols] (double)
 * += BP^T vol.  (Separately pinned by <BP gF, y> = <gF, BP^T y>.) */
void ora_backproject_T(const ora_geom *g, int32_t pitch, const double *vol, int64_t gF0, int64_t gFn, double *gFT)
{
    G o = make(g);
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    const size_t vs = (size_t)g->n_rows * g->n_cols;
    /* voxels scatter into overlapping views: one private copy per thread, summed at the end */
    #pragma omp parallel
    {
        std::vector<double> loc((size_t)gFn * vs, 0.0);
        #pragma omp for collapse(2) schedule(dynamic, 1)
        for (int j = 0; j < nz; ++j)
            for (int iy = 0; iy < ny; ++iy)
                for (int ix = 0; ix < nx; ++ix)
                    bp_voxel_T(o, x_i(o, ix), y_i(o, iy), z_j(o, j, pitch), vol[((size_t)j * ny + iy) * nx + ix],
                               loc.data(), gF0, gFn);
        #pragma omp critical
        for (size_t i = 0; i < loc.size(); ++i) gFT[i] += loc[i];
    }
}

/* Adjoint of ora_filter (gF output) for views [v_first, v_first + n_out):
 * sinoT (double, views s0 .. s0+sn-1) += F^T gFT.  Needs v_first-1 >= s0 and
 * v_first+n_out+1 <= s0+sn. */
int ora_filter_T(const ora_geom *g, const double *gFT, int64_t v_first, int64_t n_out, int64_t s0, int64_t sn, double *sinoT)
{
    G o = make(g);
    if (v_first - 1 < s0 || v_first + n_out + 1 > s0 + sn) return -1;
    std::vector<double> K = hilbert_kernel(o);
    Rebin rb = rebin_maps(o);
    const size_t rs = (size_t)g->n_rows * g->n_cols;
    std::vector<double> g1T((size_t)n_out * rs);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n_out; ++i) filter_view_T(o, K, rb, gFT + i * rs, g1T.data() + i * rs);
    for (int64_t i = 0; i < n_out; ++i) deriv_T(o, g1T.data() + i * rs, v_first + i, sinoT, s0);
    return 0;
}

/* Adjoint of ora_reconstruct: vol [np*nz][ny][nx] (double) -> sinoT (double,
 * views s0 .. s0+sn-1, overwritten).  For each pitch: BP^T into its slab's
 * filtered views, then the filter's transpose onto the raw views (P:l.246-262
 * reversed).  Returns -1 if a slab is not covered. */
int ora_adjoint(const ora_geom *g, const double *vol, int32_t k0, int32_t np, int64_t s0, int64_t sn, double *sinoT)
{
    const size_t vs = (size_t)g->nx * g->ny * g->nz;
    const size_t rs = (size_t)g->n_rows * g->n_cols;
    std::memset(sinoT, 0, sizeof(double) * rs * (size_t)sn);
    for (int32_t k = k0; k < k0 + np; ++k) {
        int64_t fv, nv;
        ora_pitch_slab(g, k, &fv, &nv);
        if (fv < s0 || fv + nv > s0 + sn) return -1;
        std::vector<double> gFT((size_t)(nv - 2) * rs, 0.0);
        ora_backproject_T(g, k, vol + (size_t)(k - k0) * vs, fv + 1, nv - 2, gFT.data());
        ora_filter_T(g, gFT.data(), fv + 1, nv - 2, s0, sn, sinoT);
    }
    return 0;
}

/* ---- NEXT-3: data generation ---- */

/* Exact line integrals of an ellipsoid phantom ell[n][8] = {cx,cy,cz,a,b,c,φ,ρ}
 * for views v0 .. v0+nv-1: out[nv][rows][cols] (double). */
void ora_project_ellipsoids(const ora_geom *g, const double *ell, int32_t n, int64_t v0, int32_t nv, double *out)
{
    G o = make(g);
    const int nr = g->n_rows, nc = g->n_cols;
    #pragma omp parallel for collapse(2) schedule(static)
    for (int32_t iv = 0; iv < nv; ++iv)
        for (int m = 0; m < nr; ++m)
            for (int l = 0; l < nc; ++l) {
                double src[3], dir[3];
                scan_ray(o, v0 + iv, m, l, src, dir);
                double acc = 0.0;
                for (int k = 0; k < n; ++k) acc += ell[8 * k + 7] * ellipsoid_chord(ell + 8 * k, src, dir);
                out[((size_t)iv * nr + m) * nc + l] = acc;
            }
}

/* Sampled line integrals of a voxel volume vol[nzv][ny][nx] (the plan's x/y
 * grid x_i = (i - nx/2) dx, slices z_j = zv0 + j dzv), trilinear interpolation
 * with zeros outside the grid, along the segment of the ray inside the box
 * where the interpolant can be nonzero (one voxel beyond the outer centres),
 * split into N = ceil(len / (0.5 min(dx, dy, dzv))) equal steps sampled at
 * their midpoints (SPEC project_numeric).  *n_trunc counts rays whose segment
 * inside the x/y box leaves the volume's z extent (that part counts 0). */
void ora_project_volume(const ora_geom *g, const float *vol, int32_t nzv, double zv0, double dzv,
                        int64_t v0, int32_t nv, double *out, int64_t *n_trunc)
{
    G o = make(g);
    const int nr = g->n_rows, nc = g->n_cols, nx = g->nx, ny = g->ny;
    const double lo[3] = {x_i(o, 0) - g->dx, y_i(o, 0) - g->dy, zv0 - dzv};
    const double hi[3] = {x_i(o, nx - 1) + g->dx, y_i(o, ny - 1) + g->dy, zv0 + (nzv - 1) * dzv + dzv};
    const double ds = 0.5 * std::min(std::min(g->dx, g->dy), dzv);
    int64_t trunc = 0;
    auto at = [&](int i, int j, int k) -> double {
        if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nzv) return 0.0;
        return vol[((size_t)k * ny + j) * nx + i];
    };
    #pragma omp parallel for collapse(2) schedule(static) reduction(+:trunc)
    for (int32_t iv = 0; iv < nv; ++iv)
        for (int m = 0; m < nr; ++m)
            for (int l = 0; l < nc; ++l) {
                double src[3], dir[3];
                scan_ray(o, v0 + iv, m, l, src, dir);
                double t0 = -1e300, t1 = 1e300, t0xy = -1e300, t1xy = 1e300;
                for (int a = 0; a < 3; ++a) {
                    if (dir[a] == 0.0) {
                        if (src[a] < lo[a] || src[a] > hi[a]) { t0 = 1.0; t1 = 0.0; }
                        continue;
                    }
                    double ta = (lo[a] - src[a]) / dir[a], tb = (hi[a] - src[a]) / dir[a];
                    if (ta > tb) std::swap(ta, tb);
                    t0 = std::max(t0, ta); t1 = std::min(t1, tb);
                    if (a < 2) { t0xy = std::max(t0xy, ta); t1xy = std::min(t1xy, tb); }
                }
                double acc = 0.0;
                if (t1xy > t0xy && (t0 > t0xy + 1e-9 || t1 < t1xy - 1e-9)) ++trunc;
                if (t1 > t0) {
                    const int64_t N = (int64_t)std::ceil((t1 - t0) / ds);
                    const double h = (t1 - t0) / N;
                    for (int64_t i = 0; i < N; ++i) {
                        const double t = t0 + (i + 0.5) * h;
                        const double fx = (src[0] + t * dir[0] - x_i(o, 0)) / g->dx;
                        const double fy = (src[1] + t * dir[1] - y_i(o, 0)) / g->dy;
                        const double fz = (src[2] + t * dir[2] - zv0) / dzv;
                        const int ix = (int)std::floor(fx), iy = (int)std::floor(fy), iz = (int)std::floor(fz);
                        const double ax = fx - ix, ay = fy - iy, az = fz - iz;
                        double v = 0.0;
                        for (int c = 0; c < 8; ++c) {
                            const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
                            const double w = (dx ? ax : 1.0 - ax) * (dy ? ay : 1.0 - ay) * (dz ? az : 1.0 - az);
                            v += w * at(ix + dx, iy + dy, iz + dz);
                        }
                        acc += v * h;
                    }
                }
                out[((size_t)iv * nr + m) * nc + l] = acc;
            }
    if (n_trunc) *n_trunc = trunc;
}

/* α down/upsampling (P:l.394-397: α_sp = α_cor[0:stride:end], "upsample by
 * interpolation"): keeps columns 0, stride, ...; linear interpolation between
 * kept columns, the last kept value held beyond it.  sino/out [nv][rows][cols]. */
void ora_resample_alpha(const ora_geom *g, const double *sino, int64_t nv, int32_t stride, double *out)
{
    const int nr = g->n_rows, nc = g->n_cols;
    const int last = stride * ((nc - 1) / stride);
    for (int64_t r = 0; r < nv * nr; ++r) {
        const double *s = sino + r * nc;
        double *d = out + r * nc;
        for (int l = 0; l < nc; ++l) {
            if (l >= last) { d[l] = s[last]; continue; }
            const int l0 = stride * (l / stride);
            const double f = (double)(l - l0) / stride;
            d[l] = (1.0 - f) * s[l0] + f * s[l0 + stride];
        }
    }
}

/* 'Gaussian+Poisson' noise of P:l.398-404 on an (upsampled) sinogram of views
 * v_first .. v_first+nv-1 (absolute indices: the random stream of a sample is
 * keyed by (seed, (v * rows + m) * cols + l), so chunking does not change it):
 *   t = I0 exp(-g/M), s = Poisson(t) + Normal(0, var) (reading: a Poisson draw of
 *   mean t, not t + Poisson(t)), s = max(s, 1), out = log(I0/s) M.
 * M = max of g over the call (> 0).  counts (optional) receives the Poisson draws.
 * mode 1 = noiseless check: Poisson replaced by its mean and var = 0. */
int ora_add_noise(const ora_geom *g, const double *sino, int64_t v_first, int64_t nv, double I0, double var,
                  uint64_t seed, int mode, double *out, int64_t *counts, double *M_out)
{
    const int nr = g->n_rows, nc = g->n_cols;
    const int64_t n = nv * nr * nc;
    double M = 0.0;
    for (int64_t i = 0; i < n; ++i) M = std::max(M, sino[i]);
    if (!(M > 0.0)) return -1;
    if (M_out) *M_out = M;
    const double sd = std::sqrt(var);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double t = I0 * std::exp(-sino[i] / M);
        double s;
        if (mode == 1) {
            s = t;
        } else {
            Stream st;
            st.key[0] = (uint32_t)seed; st.key[1] = (uint32_t)(seed >> 32);
            st.idx = (uint64_t)(v_first * nr * nc) + (uint64_t)i;
            const int64_t k = poisson_ptrs(t, st);
            if (counts) counts[i] = k;
            s = (double)k + sd * normal(st);
        }
        s = std::max(s, 1.0);
        out[i] = std::log(I0 / s) * M;
    }
    return 0;
}

/* Philox4x32-10 of one counter (for the known-answer pin). */
void ora_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    philox(c, key);
    std::memcpy(out, c, sizeof(c));
}

}  // extern "C"
