/*
 * synth.c — seeded synthetic INPUT generator shared by tests, bench and the
 * oracle's tests.  It holds none of the Katsevich method's arithmetic: it is
 * the forward model (exact line integrals of ellipsoid phantoms along the rays
 * of a helical curved-detector scan) that produces the sinograms both the
 * oracle and the CUDA path reconstruct.
 *
 * Scan model (Eq. 1; curved detector l.117, l.311-349):
 *   source        a(λ) = (R cos(λ+λ0), R sin(λ+λ0), z0 + P λ / 2π)
 *   detector pt   a(λ) + D sinα e_u + D cosα e_v + w e_z
 *                 e_u = (-sin(λ+λ0), cos(λ+λ0), 0),  e_v = (-cos(λ+λ0), -sin(λ+λ0), 0)
 *   (SPEC.md l.49-52 detector_ray).  View index v <-> λ = v·2π/views_per_turn.
 *   Flat detector (flat = 1, NEXT-4): detector pt a(λ) + u e_u + D e_v + w e_z, u_l in mm.
 *   α_l = (l-(n_cols-1)/2+alpha_offset)·d_alpha,  w_m = (m-(n_rows-1)/2)·d_w.
 *
 * Phantom: list of ellipsoids {cx,cy,cz, a,b,c, phi, rho}; c <= 0 means an
 * infinite elliptic cylinder along z.  Densities add.
 * Chord of a ray through an ellipsoid: closed-form quadratic.
 *
 * Built as libsynth.so; called through synth/synth.py (ctypes).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

typedef struct {
    double R, D, P, lambda0, z0;
    int32_t n_rows; double d_w;
    int32_t n_cols; double d_alpha, alpha_offset;
    int32_t views_per_turn;
    int32_t flat;            /* 1: flat detector, columns u_l [mm] on the plane at distance D */
} synth_scan;

/* unnormalised ray direction to detector column coordinate a (α or u) and row w */
static void det_dir(const synth_scan *s, const double eu[2], const double ev[2], double a, double w, double d[3])
{
    double su = s->flat ? a : s->D * sin(a), sv = s->flat ? s->D : s->D * cos(a);
    d[0] = su * eu[0] + sv * ev[0];
    d[1] = su * eu[1] + sv * ev[1];
    d[2] = w;
}

/* ellipsoid record: 8 doubles */
enum { E_CX, E_CY, E_CZ, E_A, E_B, E_C, E_PHI, E_RHO, E_N };

static double ray_ellipsoid_chord(const double *e, const double o[3], const double d[3])
{
    /* rotate into the ellipsoid frame (rotation phi about z), scale by axes */
    double cp = cos(e[E_PHI]), sp = sin(e[E_PHI]);
    double ox = o[0] - e[E_CX], oy = o[1] - e[E_CY], oz = o[2] - e[E_CZ];
    double px = ( cp * ox + sp * oy) / e[E_A];
    double py = (-sp * ox + cp * oy) / e[E_B];
    double qx = ( cp * d[0] + sp * d[1]) / e[E_A];
    double qy = (-sp * d[0] + cp * d[1]) / e[E_B];
    double A, B, C;
    if (e[E_C] > 0.0) {
        double pz = oz / e[E_C], qz = d[2] / e[E_C];
        A = qx * qx + qy * qy + qz * qz;
        B = 2.0 * (px * qx + py * qy + pz * qz);
        C = px * px + py * py + pz * pz - 1.0;
    } else { /* infinite cylinder along z */
        A = qx * qx + qy * qy;
        B = 2.0 * (px * qx + py * qy);
        C = px * px + py * py - 1.0;
    }
    if (A <= 0.0) return 0.0;
    double disc = B * B - 4.0 * A * C;
    if (disc <= 0.0) return 0.0;
    /* |d| = 1, so the parameter span sqrt(disc)/A is the chord length in mm */
    return sqrt(disc) / A;
}

/* out[v][m][l] for views v0 .. v0+n_views-1 (float32, C order). */
void synth_project(const synth_scan *s, const double *ell, int32_t n_ell,
                   int64_t v0, int32_t n_views, float *out)
{
    const double dlam = 2.0 * M_PI / (double)s->views_per_turn;
    const int nr = s->n_rows, nc = s->n_cols;
    #pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int32_t iv = 0; iv < n_views; ++iv) {
        for (int m = 0; m < nr; ++m) {
            double lam = (double)(v0 + iv) * dlam;
            double cl = cos(lam + s->lambda0), sl = sin(lam + s->lambda0);
            double o[3] = { s->R * cl, s->R * sl, s->z0 + s->P * lam / (2.0 * M_PI) };
            double eu[2] = { -sl, cl }, ev[2] = { -cl, -sl };
            double w = ((double)m - 0.5 * (nr - 1)) * s->d_w;
            float *row = out + ((size_t)iv * nr + m) * nc;
            for (int l = 0; l < nc; ++l) {
                double al = ((double)l - 0.5 * (nc - 1) + s->alpha_offset) * s->d_alpha;
                double d[3];
                det_dir(s, eu, ev, al, w, d);
                double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                d[0] /= nrm; d[1] /= nrm; d[2] /= nrm;
                double acc = 0.0;
                for (int k = 0; k < n_ell; ++k)
                    acc += ell[k * E_N + E_RHO] * ray_ellipsoid_chord(ell + k * E_N, o, d);
                row[l] = (float)acc;
            }
        }
    }
}

/* Numerical quadrature of the same line integral (midpoint rule, step h over
 * the ray parameter range [t0, t1]) — used only to pin synth_project. */
double synth_ray_quadrature(const synth_scan *s, const double *ell, int32_t n_ell,
                            double lam, double alpha, double w,
                            double t0, double t1, double h)
{
    double cl = cos(lam + s->lambda0), sl = sin(lam + s->lambda0);
    double o[3] = { s->R * cl, s->R * sl, s->z0 + s->P * lam / (2.0 * M_PI) };
    double eu[2] = { -sl, cl }, ev[2] = { -cl, -sl };
    double d[3];
    det_dir(s, eu, ev, alpha, w, d);
    double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] /= nrm; d[1] /= nrm; d[2] /= nrm;
    double acc = 0.0;
    long n = (long)ceil((t1 - t0) / h);
    double hh = (t1 - t0) / (double)n;
    for (long i = 0; i < n; ++i) {
        double t = t0 + (i + 0.5) * hh;
        double p[3] = { o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2] };
        for (int k = 0; k < n_ell; ++k) {
            const double *e = ell + k * E_N;
            double cp = cos(e[E_PHI]), sp = sin(e[E_PHI]);
            double x = p[0] - e[E_CX], y = p[1] - e[E_CY], z = p[2] - e[E_CZ];
            double u = (cp * x + sp * y) / e[E_A], v = (-sp * x + cp * y) / e[E_B];
            double r2 = u * u + v * v + (e[E_C] > 0.0 ? (z / e[E_C]) * (z / e[E_C]) : 0.0);
            if (r2 <= 1.0) acc += e[E_RHO] * hh;
        }
    }
    return acc;
}

/* Ground-truth density f_true at points pts[n][3]. */
void synth_phantom_eval(const double *ell, int32_t n_ell, const double *pts, int64_t n, double *out)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < n_ell; ++k) {
            const double *e = ell + k * E_N;
            double cp = cos(e[E_PHI]), sp = sin(e[E_PHI]);
            double x = pts[3 * i] - e[E_CX], y = pts[3 * i + 1] - e[E_CY], z = pts[3 * i + 2] - e[E_CZ];
            double u = (cp * x + sp * y) / e[E_A], v = (-sp * x + cp * y) / e[E_B];
            double r2 = u * u + v * v + (e[E_C] > 0.0 ? (z / e[E_C]) * (z / e[E_C]) : 0.0);
            if (r2 <= 1.0) acc += e[E_RHO];
        }
        out[i] = acc;
    }
}
