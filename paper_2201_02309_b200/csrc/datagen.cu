// datagen.cu — the data-generation path of PAPER.md l.353-404 (SURVEY §8(f)
// NEXT-3) on the GPU: helical curved-detector forward projection (exact chords
// of ellipsoid phantoms; trilinear ray marching through voxel volumes), the
// α down/upsampling of the sparse-view protocol and the 'Gaussian+Poisson'
// noise model.  Produces training-shaped inputs at scale instead of the CPU.
//
// Scan ray of detector sample (v, m, l) (helix P:l.87-94, curved detector
// P:l.117, l.311-349): source a(λ) = (R cos(λ+λ0), R sin(λ+λ0), z0 + hλ),
// direction ∝ D sinα e_t − D cosα e_r + w e_z — the geometry step 7 inverts.
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace kats {

namespace {

__device__ __forceinline__ void scan_ray(const DataGenParams &p, int64_t v, int m, int l, double src[3], double dir[3])
{
    const double lam = (double)v * p.dlam;
    double sn, c;
    sincos(lam + p.lambda0, &sn, &c);
    src[0] = p.R * c;
    src[1] = p.R * sn;
    src[2] = p.z0 + p.h * lam;
    const double a = ((double)l - 0.5 * (p.nc - 1) + p.alpha_offset) * p.d_alpha;
    const double w = ((double)m - 0.5 * (p.nr - 1)) * p.d_w;
    double sa, ca;
    if (p.flat) { sa = a; ca = p.D; }                   // flat (A27): u e_t - D e_r + w e_z
    else { sincos(a, &sa, &ca); sa *= p.D; ca *= p.D; }
    const double d0 = -sa * sn - ca * c, d1 = sa * c - ca * sn, d2 = w;
    const double inv = rsqrt(d0 * d0 + d1 * d1 + d2 * d2);
    dir[0] = d0 * inv;
    dir[1] = d1 * inv;
    dir[2] = d2 * inv;
}

}  // namespace

// ---------------------------------------------------------------------------
// Exact line integrals of an ellipsoid phantom {c, semi-axes (c <= 0: infinite
// cylinder along z), rotation φ about z, density ρ}; fp64 (B200 runs FP64 at
// half the FP32 rate), one thread per ray, the phantom in shared memory with
// cos φ, sin φ precomputed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_project_ellipsoids(DataGenParams p, const double *__restrict__ ell, int n,
                                                            int64_t v0, float *__restrict__ out)
{
    extern __shared__ double es[];                                 // [n][10]
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double *e = ell + 8 * i;
        double *d = es + 10 * i;
        for (int k = 0; k < 8; ++k) d[k] = e[k];
        sincos(e[6], &d[9], &d[8]);                                 // d[8] = cos φ, d[9] = sin φ
    }
    __syncthreads();
    const int l = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
    const int64_t iv = blockIdx.z;
    if (l >= p.nc) return;
    double o[3], d[3];
    scan_ray(p, v0 + iv, m, l, o, d);
    double acc = 0.0;
    for (int k = 0; k < n; ++k) {
        const double *e = es + 10 * k;
        const double cp = e[8], sp = e[9];
        const double ox = o[0] - e[0], oy = o[1] - e[1], oz = o[2] - e[2];
        const double px = (cp * ox + sp * oy) / e[3], py = (-sp * ox + cp * oy) / e[4];
        const double qx = (cp * d[0] + sp * d[1]) / e[3], qy = (-sp * d[0] + cp * d[1]) / e[4];
        double A = qx * qx + qy * qy, B = 2.0 * (px * qx + py * qy), C = px * px + py * py - 1.0;
        if (e[5] > 0.0) {
            const double pz = oz / e[5], qz = d[2] / e[5];
            A += qz * qz;
            B += 2.0 * pz * qz;
            C += pz * pz;
        }
        if (A <= 0.0) continue;
        const double disc = B * B - 4.0 * A * C;
        if (disc > 0.0) acc += e[7] * sqrt(disc) / A;
    }
    out[(iv * p.nr + m) * p.nc + l] = (float)acc;
}

// ---------------------------------------------------------------------------
// Sampled line integrals of a voxel volume [nzv][ny][nx] (the plan's x/y grid,
// slices z_j = zv0 + j dzv): trilinear interpolation with zeros outside the
// grid along the ray's segment inside the box where the interpolant can be
// nonzero, N = ceil(len / (0.5 min voxel)) equal steps sampled at midpoints.
// fp32 (positions relative to the source: |t dir| <~ 2000 mm, 1e-4 mm).  Rays
// whose x/y segment leaves the volume's z extent are counted (n_trunc).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_project_volume(DataGenParams p, const float *__restrict__ vol, int nzv,
                                                        float zv0, float dzv, int64_t v0, float *__restrict__ out,
                                                        unsigned long long *n_trunc)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
    const int64_t iv = blockIdx.z;
    if (l >= p.nc) return;
    double od[3], dd[3];
    scan_ray(p, v0 + iv, m, l, od, dd);
    const float x0 = (float)(-0.5 * p.nx * p.dx), y0 = (float)(-0.5 * p.ny * p.dy);
    const float dx = (float)p.dx, dy = (float)p.dy;
    const float o[3] = {(float)od[0], (float)od[1], (float)od[2]}, d[3] = {(float)dd[0], (float)dd[1], (float)dd[2]};
    const float lo[3] = {x0 - dx, y0 - dy, zv0 - dzv};
    const float hi[3] = {x0 + p.nx * dx, y0 + p.ny * dy, zv0 + nzv * dzv};
    float t0 = -3.0e38f, t1 = 3.0e38f, t0xy = -3.0e38f, t1xy = 3.0e38f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (d[a] == 0.f) {
            if (o[a] < lo[a] || o[a] > hi[a]) { t0 = 1.f; t1 = 0.f; }
            continue;
        }
        float ta = (lo[a] - o[a]) / d[a], tb = (hi[a] - o[a]) / d[a];
        if (ta > tb) { const float q = ta; ta = tb; tb = q; }
        t0 = fmaxf(t0, ta);
        t1 = fminf(t1, tb);
        if (a < 2) { t0xy = fmaxf(t0xy, ta); t1xy = fminf(t1xy, tb); }
    }
    float acc = 0.f;
    if (t1xy > t0xy && (t0 > t0xy + 1e-3f || t1 < t1xy - 1e-3f)) atomicAdd(n_trunc, 1ull);
    if (t1 > t0) {
        const float ds = 0.5f * fminf(fminf(dx, dy), dzv);
        const int N = (int)ceilf((t1 - t0) / ds);
        const float h = (t1 - t0) / N;
        const float ix0 = 1.f / dx, iy0 = 1.f / dy, iz0 = 1.f / dzv;
        const size_t plane = (size_t)p.nx * p.ny;
        for (int i = 0; i < N; ++i) {
            const float t = fmaf((float)i + 0.5f, h, t0);
            const float fx = (fmaf(t, d[0], o[0]) - x0) * ix0;
            const float fy = (fmaf(t, d[1], o[1]) - y0) * iy0;
            const float fz = (fmaf(t, d[2], o[2]) - zv0) * iz0;
            const int ix = (int)floorf(fx), iy = (int)floorf(fy), iz = (int)floorf(fz);
            const float ax = fx - ix, ay = fy - iy, az = fz - iz;
            float v = 0.f;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int cx = ix + (c & 1), cy = iy + ((c >> 1) & 1), cz = iz + (c >> 2);
                if (cx < 0 || cx >= p.nx || cy < 0 || cy >= p.ny || cz < 0 || cz >= nzv) continue;
                const float w = ((c & 1) ? ax : 1.f - ax) * (((c >> 1) & 1) ? ay : 1.f - ay) * ((c >> 2) ? az : 1.f - az);
                v = fmaf(w, __ldg(vol + (size_t)cz * plane + (size_t)cy * p.nx + cx), v);
            }
            acc = fmaf(v, h, acc);
        }
    }
    out[(iv * p.nr + m) * p.nc + l] = acc;
}

// ---------------------------------------------------------------------------
// α down/upsampling (P:l.394-397): keep columns 0, stride, ...; linear
// interpolation back, the last kept value held beyond it.  Also the max.
// ---------------------------------------------------------------------------
__global__ void k_resample_alpha(const float *__restrict__ in, int64_t rows, int nc, int stride,
                                 float *__restrict__ out, unsigned *maxbits)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float v = 0.f;
    if (i < rows * nc) {
        const int64_t r = i / nc;
        const int l = (int)(i - r * nc);
        const float *s = in + r * nc;
        const int last = stride * ((nc - 1) / stride);
        if (l >= last) {
            v = s[last];
        } else {
            // in fp64, uncontracted, rounded once: the fp32 value of the exact interpolant
            // (the noise step's integer draws depend on it bit for bit)
            const int l0 = stride * (l / stride);
            const double f = (double)(l - l0) / (double)stride;
            v = (float)__dadd_rn(__dmul_rn(1.0 - f, (double)s[l0]), __dmul_rn(f, (double)s[l0 + stride]));
        }
        out[i] = v;
    }
    // non-negative floats order as their bits (the noise model takes g >= 0)
    const unsigned b = __reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(v, 0.f)));
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, b);
}

namespace {

// Philox4x32-10 (Salmon et al., SC'11), same stream as the oracle
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c[0]), l0 = 0xD2511F53u * c[0];
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c[2]), l1 = 0xCD9E8D57u * c[2];
        const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = l1; c[2] = n2; c[3] = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

struct Stream {
    uint32_t k0, k1, draw;
    uint64_t idx;
    double buf[2];
    int left;
    __device__ double uniform()
    {
        if (!left) {
            uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), draw++, 0u};
            philox(c, k0, k1);
            buf[0] = ((double)((((uint64_t)(c[0] >> 5)) << 26) | (c[1] >> 6)) + 0.5) * 0x1p-53;
            buf[1] = ((double)((((uint64_t)(c[2] >> 5)) << 26) | (c[3] >> 6)) + 0.5) * 0x1p-53;
            left = 2;
        }
        return buf[2 - left--];
    }
};

// Poisson(lam), lam >= 10: PTRS (Hörmann 1993).  Uncontracted fp64 arithmetic
// (__dmul_rn / __dadd_rn) where it decides the integer, as the oracle computes it.
__device__ int64_t poisson_ptrs(double lam, Stream &st)
{
    const double slam = sqrt(lam), loglam = log(lam);
    const double b = __dadd_rn(0.931, __dmul_rn(2.53, slam));
    const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
    const double invalpha = __dadd_rn(1.1239, 1.1328 / __dadd_rn(b, -3.4));
    const double vr = __dadd_rn(0.9277, -(3.6224 / __dadd_rn(b, -2.0)));
    for (;;) {
        const double U = __dadd_rn(st.uniform(), -0.5), V = st.uniform();
        const double us = __dadd_rn(0.5, -fabs(U));
        const double k = floor(__dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(2.0 * a / us, b), U), lam), 0.43));
        if (us >= 0.07 && V <= vr) return (int64_t)k;
        if (k < 0.0 || (us < 0.013 && V > us)) continue;
        const double lhs = __dadd_rn(__dadd_rn(log(V), log(invalpha)), -log(__dadd_rn(a / __dmul_rn(us, us), b)));
        const double rhs = __dadd_rn(__dadd_rn(-lam, __dmul_rn(k, loglam)), -lgamma(__dadd_rn(k, 1.0)));
        if (lhs <= rhs) return (int64_t)k;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// 'Gaussian+Poisson' noise (P:l.398-404): t = I0 exp(-g/M), s = Poisson(t) +
// Normal(0, var) (reading: a Poisson draw of mean t), s >= 1,
// out = log(I0/s) M.  The stream of a sample is keyed by (seed, absolute sample
// index), so results do not depend on chunking.  mode 1: noiseless check.
// ---------------------------------------------------------------------------
__global__ void k_add_noise(const float *__restrict__ g, int64_t n, int64_t idx0, double I0, double sd,
                            uint64_t seed, int mode, const unsigned *maxbits, float *__restrict__ out,
                            long long *counts, float *M_out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double M = (double)__uint_as_float(*maxbits);
    if (i == 0 && M_out) *M_out = (float)M;
    if (i >= n) return;
    const double t = I0 * exp(-(double)g[i] / M);
    double s;
    if (mode == 1) {
        s = t;
    } else {
        Stream st{(uint32_t)seed, (uint32_t)(seed >> 32), 0u, (uint64_t)(idx0 + i), {0.0, 0.0}, 0};
        const int64_t k = poisson_ptrs(t, st);
        if (counts) counts[i] = (long long)k;
        const double u1 = st.uniform(), u2 = st.uniform();
        s = __dadd_rn((double)k, __dmul_rn(sd, __dmul_rn(sqrt(-2.0 * log(u1)), cospi(2.0 * u2))));
    }
    s = fmax(s, 1.0);
    out[i] = (float)(log(I0 / s) * M);
}

void launch_project_ellipsoids(const DataGenParams &p, const double *ell, int n, int64_t v0, int64_t nv, float *out,
                               cudaStream_t s)
{
    const size_t smem = sizeof(double) * 10 * (size_t)n;            // <= 160 KB (the ABI caps n at 2048)
    smem_opt_in((const void *)k_project_ellipsoids, smem);
    for (int64_t c = 0; c < nv; c += 65535)                           // grid.z <= 65535 views per launch
        k_project_ellipsoids<<<dim3((p.nc + 127) / 128, p.nr, (unsigned)std::min<int64_t>(65535, nv - c)), 128, smem,
                               s>>>(p, ell, n, v0 + c, out + (size_t)c * p.nr * p.nc);
}

void launch_project_volume(const DataGenParams &p, const float *vol, int nzv, float zv0, float dzv, int64_t v0,
                           int64_t nv, float *out, unsigned long long *n_trunc, cudaStream_t s)
{
    for (int64_t c = 0; c < nv; c += 65535)                           // grid.z <= 65535 views per launch
        k_project_volume<<<dim3((p.nc + 127) / 128, p.nr, (unsigned)std::min<int64_t>(65535, nv - c)), 128, 0, s>>>(
            p, vol, nzv, zv0, dzv, v0 + c, out + (size_t)c * p.nr * p.nc, n_trunc);
}

void launch_degrade(const DataGenParams &p, const float *in, int64_t v0, int64_t nv, int stride, double I0, double var,
                    uint64_t seed, int mode, float *up, unsigned *maxbits, float *out, long long *counts, float *M_out,
                    cudaStream_t s)
{
    const int64_t rows = nv * p.nr, n = rows * p.nc;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    cudaMemsetAsync(maxbits, 0, sizeof(unsigned), s);
    k_resample_alpha<<<blocks, 256, 0, s>>>(in, rows, p.nc, stride, up, maxbits);
    k_add_noise<<<blocks, 256, 0, s>>>(up, n, v0 * p.nr * p.nc, I0, sqrt(var), seed, mode, maxbits, out, counts,
                                       M_out);
}

}  // namespace kats
