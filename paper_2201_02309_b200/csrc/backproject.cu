// backproject.cu — step 7 of PAPER.md §II (l.155-171; reconstruction step 2,
// l.251-262): PI-interval-limited, voxel-driven weighted backprojection
//   f(x) = Δλ/2π Σ_{k=k_first}^{k_last} ω_k gF_k(α*_k, w*_k) / v*_k
// with v* = R - x cos(λ+λ0) - y sin(λ+λ0), α* = atan(u/v*),
// u = -x sin(λ+λ0) + y cos(λ+λ0), w* = D cos α*/v* (z - z0 - hλ)  (P:l.161-170).
//
// Pitch-relative coordinates: view k is pitch-relative, z_j = j dz,
// so the periodic tables (T_pi, T_view) serve every pitch bit-identically.
// v*, α* (one atan2) and the column position are z-independent; w* is affine
// in z, so each thread owns an (x, y) column chunk of JZ slices and walks the
// union of their PI-windows; bilinear interpolation in fp32 (A9).
// D cos α*/v* = D / sqrt(u² + v*²) (no cos needed).  Interior views carry
// weight 1; the fractional end weights are applied as a correction
// (ω - 1)·term after the main loop, keeping the hot loop branch-light.
#include <climits>

#include "kernels.cuh"

namespace kats {

namespace {

constexpr int TX = 16, TY = 16, JZ = 8;

struct ViewSetup {
    bool ok;
    const float *col;   // &gF[k][0][l]
    float fa, inv_v, base, step;
};

__device__ __forceinline__ ViewSetup view_setup(const BPParams &p, const float *gitem, int k, float x, float y, float zbase)
{
    ViewSetup s;
    const ViewGeom vg = p.view[k - p.view_lo];
    const float vstar = p.R - x * vg.c - y * vg.s;
    const float u = -x * vg.s + y * vg.c;
    const float colpos = atan2f(u, vstar) * p.inv_dalpha + p.col_c;
    s.ok = colpos >= 0.f && colpos <= (float)(p.nc - 1);
    int l = min((int)colpos, p.nc - 2);
    l = max(l, 0);
    s.fa = colpos - (float)l;
    s.inv_v = 1.0f / vstar;
    const float sc = p.D * rsqrtf(fmaf(u, u, vstar * vstar)) * p.inv_dw;   // (D cos α*/v*)/Δw
    s.base = fmaf(sc, zbase - vg.zc, p.row_c);
    s.step = sc * p.dz;
    s.col = gitem + (int64_t)k * p.nr * p.nc + l;
    return s;
}

__device__ __forceinline__ float sample(const BPParams &p, const ViewSetup &s, float pos)
{
    if (!(pos >= 0.f && pos <= (float)(p.nr - 1))) return 0.f;
    int m = min((int)pos, p.nr - 2);
    const float fw = pos - (float)m;
    const float *q = s.col + m * p.nc;
    const float a0 = __ldg(q), a1 = __ldg(q + 1), b0 = __ldg(q + p.nc), b1 = __ldg(q + p.nc + 1);
    const float r0 = fmaf(s.fa, a1 - a0, a0), r1 = fmaf(s.fa, b1 - b0, b0);
    return fmaf(fw, r1 - r0, r0) * s.inv_v;
}

}  // namespace

__global__ void __launch_bounds__(TX *TY) k_backproject(BPParams p)
{
    const int ix = blockIdx.x * TX + threadIdx.x;
    const int iy = blockIdx.y * TY + threadIdx.y;
    const int nchunk = (p.nz + JZ - 1) / JZ;
    const int chunk = blockIdx.z % nchunk;
    const int item = blockIdx.z / nchunk;
    if (ix >= p.nx || iy >= p.ny) return;
    const int j0 = chunk * JZ;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col0 = (size_t)iy * p.nx + ix;

    int kf[JZ], kl[JZ];
    int kbeg = INT_MAX, kend = INT_MIN;
#pragma unroll
    for (int t = 0; t < JZ; ++t) {
        kf[t] = INT_MAX; kl[t] = INT_MIN;
        if (j0 + t < p.nz) {
            const int2 e = p.pi_k[(size_t)(j0 + t) * plane + col0];
            if (e.x <= e.y) {
                kf[t] = e.x; kl[t] = e.y;
                kbeg = min(kbeg, e.x); kend = max(kend, e.y);
            }
        }
    }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const float zbase = j0 * p.dz;
    const float *gitem = p.gF + (p.off0 + (int64_t)item * p.item_views) * p.nr * p.nc;

    float acc[JZ];
#pragma unroll
    for (int t = 0; t < JZ; ++t) acc[t] = 0.f;

    for (int k = kbeg; k <= kend; ++k) {
        const ViewSetup s = view_setup(p, gitem, k, x, y, zbase);
        if (!s.ok) continue;
#pragma unroll
        for (int t = 0; t < JZ; ++t) {
            if (k >= kf[t] && k <= kl[t]) acc[t] += sample(p, s, fmaf((float)t, s.step, s.base));
        }
    }
    // fractional end weights: main loop used ω = 1 for every view in [k_first, k_last]
#pragma unroll
    for (int t = 0; t < JZ; ++t) {
        if (kf[t] <= kl[t]) {
            const float2 w = p.pi_w[(size_t)(j0 + t) * plane + col0];
            const ViewSetup sf = view_setup(p, gitem, kf[t], x, y, zbase);
            if (sf.ok) acc[t] += (w.x - 1.f) * sample(p, sf, fmaf((float)t, sf.step, sf.base));
            if (kl[t] != kf[t]) {
                const ViewSetup sl = view_setup(p, gitem, kl[t], x, y, zbase);
                if (sl.ok) acc[t] += (w.y - 1.f) * sample(p, sl, fmaf((float)t, sl.step, sl.base));
            }
        }
    }
    float *out = p.vol + (size_t)item * p.nz * plane + col0;
#pragma unroll
    for (int t = 0; t < JZ; ++t)
        if (j0 + t < p.nz) out[(size_t)(j0 + t) * plane] = acc[t] * p.scale;
}

void launch_backproject(const BPParams &p, cudaStream_t s)
{
    const int nchunk = (p.nz + JZ - 1) / JZ;
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, nchunk * p.n_items);
    k_backproject<<<grid, dim3(TX, TY), 0, s>>>(p);
}

}  // namespace kats
