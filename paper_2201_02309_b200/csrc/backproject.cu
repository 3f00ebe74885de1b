// backproject.cu — step 7 of PAPER.md §II (l.155-171; reconstruction step 2,
// l.251-262): PI-interval-limited, voxel-driven weighted backprojection
//   f(x) = Δλ/2π Σ_{k=k_first}^{k_last} ω_k gF_k(α*_k, w*_k) / v*_k
// with v* = R - x cos(λ+λ0) - y sin(λ+λ0), α* = atan(u/v*),
// u = -x sin(λ+λ0) + y cos(λ+λ0), w* = D cos α*/v* (z - z0 - hλ)  (P:l.161-170).
//
// Design:
//  * pitch-relative coordinates: one table serves every pitch;
//  * a thread owns an (x, y) column chunk of JZ slices: v*, α*, 1/v* and the
//    detector column are computed once per (x, y, view) and reused by every
//    slice of the chunk that sees the view; w* is affine in z;
//  * D cos α*/v* = D / sqrt(u² + v*²) (rsqrt, no cos);  α* from a minimax
//    polynomial of u/v* when the fan is narrow enough (|α| < 36.8°, error
//    < 1e-8 rad), atan2f otherwise;
//  * filtered views arrive as column-major 2x2 sum/difference tap quads
//    (filter.cu K4): one 128-bit load per bilinear sample; pairs of slices run
//    on the packed-fp32 pipe (FFMA2/FADD2/FMUL2, sm_100a): row position,
//    round-to-nearest magic-number floor and fraction for two slices per
//    instruction, then two FFMA2 per sample into a (sum, difference)
//    accumulator pair; addresses by LEA on the integer pipe;
//  * interior views (k_first < k < k_last) lie strictly inside the PI window,
//    hence inside the Tam–Danielsson window and the detector when the plan's
//    margin check passed (two zero pad rows absorb fp32 rounding); the two end
//    views per voxel carry the fractional weights and the full
//    out-of-detector test (A9, A11);
//  * which slices of the chunk see view k is a bitmask recomputed only at the
//    2·JZ events where a slice's interior window opens or closes.
#include <climits>

#include "kernels.cuh"

namespace kats {

namespace {

constexpr int TX = 16, TY = 16, JZ = 8;
constexpr float kMagic = 12582912.0f;          // 1.5 * 2^23: x + kMagic rounds x to an integer
constexpr unsigned kMagicBits = 0x4B400000u;

typedef unsigned long long u64;

__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// packed fp32x2 helpers (sm_100a FFMA2 / FADD2 / FMUL2)
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(u64 v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

__device__ __forceinline__ float4 ldq(u64 addr) { return __ldg(reinterpret_cast<const float4 *>(addr)); }

struct ViewSetup {
    u64 colbase;         // &Q[k][l][0] - kMagicBits*16  (quad row r at colbase + (kMagicBits + r) * 16)
    u64 W;               // ((1 - frac_α)/v*, frac_α/v*)
    float base, step;    // quad-row position (= row position + 1.5) of slice 0 of the chunk, increment
    float colpos;        // column position (checked path)
};

template <bool POLY>
__device__ __forceinline__ ViewSetup view_setup(const BPParams &p, u64 viewbase, const float4 &vg,
                                                float x, float y, float zb)
{
    ViewSetup s;
    const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
    const float u = fmaf(y, vg.x, -x * vg.y);
    const float inv_v = rcp_approx(vstar);
    float colpos;
    if (POLY) {
        const float t = u * inv_v, q = t * t;
        float a = p.at[6];
        a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
        a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
        colpos = fmaf(t, a, p.col_c);                       // α*/Δα + (nc-1)/2 - offset
    } else {
        colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
    }
    s.colpos = colpos;
    const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
    const int l = __float2int_rz(cp);                        // per view: conversion pipe is idle
    const float fa = cp - __int2float_rn(l);
    const float w1 = fa * inv_v;
    s.W = pk(inv_v - w1, w1);
    const float sc = p.D_over_dw * rsqrt_approx(fmaf(u, u, vstar * vstar));
    s.base = fmaf(sc, zb - vg.z, p.row_c15);
    s.step = sc * p.dz;
    s.colbase = viewbase + (u64)l * p.colbytes - (u64)kMagicBits * 16ull;
    return s;
}

// accumulate two slices (quad-row positions pm0, pm1 as a pair) into acc pairs
__device__ __forceinline__ void tap2(const ViewSetup &s, u64 PM, u64 &acc0, u64 &acc1)
{
    const u64 Q = add2(PM, pk(kMagic, kMagic));
    const u64 FW = sub2(PM, sub2(Q, pk(kMagic, kMagic)));    // fraction - ½ for both slices
    float q0, q1, f0, f1;
    upk(Q, q0, q1);
    upk(FW, f0, f1);
    const float4 g0 = ldq(s.colbase + ((u64)__float_as_uint(q0) << 4));
    const float4 g1 = ldq(s.colbase + ((u64)__float_as_uint(q1) << 4));
    acc0 = fma2(pk(g0.x, g0.y), s.W, acc0);
    acc0 = fma2(pk(g0.z, g0.w), mul2(s.W, pk(f0, f0)), acc0);
    acc1 = fma2(pk(g1.x, g1.y), s.W, acc1);
    acc1 = fma2(pk(g1.z, g1.w), mul2(s.W, pk(f1, f1)), acc1);
}

__device__ __forceinline__ void tap1(const ViewSetup &s, float pm, u64 &acc)
{
    const float q = pm + kMagic;
    const float f = pm - (q - kMagic);
    const float4 g = ldq(s.colbase + ((u64)__float_as_uint(q) << 4));
    acc = fma2(pk(g.x, g.y), s.W, acc);
    acc = fma2(pk(g.z, g.w), mul2(s.W, pk(f, f)), acc);
}

// checked end-view sample with weight ω (reading A9: zero outside the closed node range)
template <bool POLY>
__device__ __forceinline__ void tap_checked(const BPParams &p, u64 qbase, int k, float x, float y,
                                            float zb, int t, float weight, u64 &acc)
{
    const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
    ViewSetup s = view_setup<POLY>(p, qbase + (u64)((int64_t)k * p.viewbytes), vg, x, y, zb);
    if (!(s.colpos >= 0.f && s.colpos <= p.colmax)) return;
    const float pm = fmaf((float)t, s.step, s.base);
    if (!(pm >= 1.5f && pm <= p.rowmax + 1.5f)) return;
    s.W = mul2(s.W, pk(weight, weight));
    tap1(s, pm, acc);
}

}  // namespace

template <bool POLY, bool CHECK>
__global__ void __launch_bounds__(TX *TY, 3) k_backproject(BPParams p)
{
    // 16x16 tile of (x, y) columns; each warp covers an 8x4 sub-tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ix = blockIdx.x * TX + (warp & 1) * 8 + (lane & 7);
    const int iy = blockIdx.y * TY + (warp >> 1) * 4 + (lane >> 3);
    const int nchunk = (p.nz + JZ - 1) / JZ;
    const int chunk = blockIdx.z % nchunk;
    const int item = blockIdx.z / nchunk;
    if (ix >= p.nx || iy >= p.ny) return;
    const int j0 = chunk * JZ;
    const int nzc = min(JZ, p.nz - j0);
    const size_t plane = (size_t)p.nx * p.ny;
    const int2 *pik = p.pi_k + (size_t)j0 * plane + (size_t)iy * p.nx + ix;

    // interior view range of the chunk [K0, K1]
    int K0 = INT_MAX, K1 = INT_MIN;
    for (int t = 0; t < nzc; ++t) {
        const int2 e = pik[t * plane];
        if (e.x + 1 <= e.y - 1) { K0 = min(K0, e.x + 1); K1 = max(K1, e.y - 1); }
    }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const float zb = j0 * p.dz;
    const u64 qbase = reinterpret_cast<u64>(p.gq) + (u64)((p.off0 + (int64_t)item * p.item_views) * p.viewbytes);

    u64 acc[JZ];
#pragma unroll
    for (int t = 0; t < JZ; ++t) acc[t] = 0ull;

    unsigned mask = 0;
    int next_ev = K0;
    u64 viewbase = qbase + (u64)((int64_t)K0 * p.viewbytes);
    const float4 *vgp = reinterpret_cast<const float4 *>(p.view) + (K0 - p.view_lo);
    for (int k = K0; k <= K1; ++k, viewbase += p.viewbytes, ++vgp) {
        if (k >= next_ev) {      // a slice's interior window opens or closes: rebuild the mask
            mask = 0;
            next_ev = INT_MAX;
            for (int t = 0; t < nzc; ++t) {
                const int2 e = pik[t * plane];
                const int a = e.x + 1, b = e.y - 1;
                if (a <= b) {
                    if (a <= k && k <= b) mask |= 1u << t;
                    if (a > k) next_ev = min(next_ev, a);
                    if (b >= k) next_ev = min(next_ev, b + 1);
                }
            }
            if (mask == 0) { k = next_ev - 1; viewbase = qbase + (u64)((int64_t)k * p.viewbytes); vgp = reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo); continue; }
        }
        const float4 vg = __ldg(vgp);
        const ViewSetup s = view_setup<POLY>(p, viewbase, vg, x, y, zb);
        if (CHECK) {
            if (!(s.colpos >= 0.f && s.colpos <= p.colmax)) continue;
#pragma unroll
            for (int t = 0; t < JZ; ++t) {
                const float pm = fmaf((float)t, s.step, s.base);
                if ((mask & (1u << t)) && pm >= 1.5f && pm <= p.rowmax + 1.5f) tap1(s, pm, acc[t]);
            }
        } else if (mask == (1u << JZ) - 1) {
            const u64 B = pk(s.base, s.base), S = pk(s.step, s.step);
#pragma unroll
            for (int t = 0; t < JZ; t += 2)
                tap2(s, fma2(pk((float)t, (float)(t + 1)), S, B), acc[t], acc[t + 1]);
        } else {
#pragma unroll
            for (int t = 0; t < JZ; ++t)
                if (mask & (1u << t)) tap1(s, fmaf((float)t, s.step, s.base), acc[t]);
        }
    }
    // end views: fractional weights ω_first, ω_last and the full range test
    const float2 *piw = p.pi_w + (size_t)j0 * plane + (size_t)iy * p.nx + ix;
#pragma unroll
    for (int t = 0; t < JZ; ++t) {
        if (t < nzc) {
            const int2 e = pik[t * plane];
            if (e.x <= e.y) {
                const float2 w = piw[t * plane];
                tap_checked<POLY>(p, qbase, e.x, x, y, zb, t, w.x, acc[t]);
                if (e.y != e.x) tap_checked<POLY>(p, qbase, e.y, x, y, zb, t, w.y, acc[t]);
            }
        }
    }
    float *out = p.vol + (size_t)item * p.nz * plane + (size_t)j0 * plane + (size_t)iy * p.nx + ix;
#pragma unroll
    for (int t = 0; t < JZ; ++t) {
        if (t < nzc) {
            float a, b;
            upk(acc[t], a, b);
            out[t * plane] = (a + b) * p.scale;
        }
    }
}

// plain gF [n][nr][nc] -> column-major sum/difference tap quads [n][nc][nr+2] (debug entry point)
__global__ void k_make_quads(const float *gF, float4 *q, int64_t n, int nr, int nc)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nq = nr + 2;
    if (i >= n * nq * nc) return;
    const int r = (int)(i % nq);
    const int l = (int)((i / nq) % nc);
    const int64_t v = i / ((int64_t)nc * nq);
    const float *g = gF + v * nr * nc;
    auto at = [&](int mm, int ll) { return (mm >= 0 && mm < nr && ll < nc) ? g[(int64_t)mm * nc + ll] : 0.f; };
    const int m = r - 2;
    const float a0 = at(m, l), c0 = at(m + 1, l), a1 = at(m, l + 1), c1 = at(m + 1, l + 1);
    q[i] = make_float4(0.5f * (a0 + c0), 0.5f * (a1 + c1), c0 - a0, c1 - a1);
}

void launch_make_quads(const float *gF, float4 *q, int64_t n, int nr, int nc, cudaStream_t s)
{
    const int64_t total = n * (nr + 2) * nc;
    k_make_quads<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gF, q, n, nr, nc);
}

void launch_backproject(const BPParams &p, cudaStream_t s)
{
    const int nchunk = (p.nz + JZ - 1) / JZ;
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, nchunk * p.n_items);
    const int block = TX * TY;
    if (p.poly) {
        if (p.checked) k_backproject<true, true><<<grid, block, 0, s>>>(p);
        else k_backproject<true, false><<<grid, block, 0, s>>>(p);
    } else {
        if (p.checked) k_backproject<false, true><<<grid, block, 0, s>>>(p);
        else k_backproject<false, false><<<grid, block, 0, s>>>(p);
    }
}

}  // namespace kats
