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
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include <cuda.h>

#include "kernels.cuh"

namespace kats {

namespace {

constexpr int TX = kTileX, TY = kTileY, JZ = kChunkZ;   // staged kernel: 16 slices per thread
constexpr int JZL = 8;                                    // L1-path fallback kernel: 8 slices per thread
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
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ void fma2_acc(u64 &acc, u64 a, u64 b) { asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b)); }

__device__ __forceinline__ float4 ldq(u64 addr) { return __ldg(reinterpret_cast<const float4 *>(addr)); }
__device__ __forceinline__ float4 lds128(unsigned saddr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
    return v;
}

struct ViewSetup {
    u64 colbase;         // &Q[k][l][0] - kMagicBits*16  (quad row r at colbase + (kMagicBits + r) * 16)
    u64 W;               // ((1 - frac_α)/v*, frac_α/v*)
    float base, step;    // centred quad-row position (row + 1.5 - c) of slice 0 of the chunk, increment
    float qmagic;        // kMagic + c: (position + qmagic) has the quad row's index in its low bits
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
    const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
    s.base = fmaf(sc, zb - vg.z, p.row_cc);
    s.qmagic = p.qmagic;
    s.step = sc * p.dz;
    s.colbase = viewbase + (u64)l * p.colbytes - (u64)kMagicBits * 16ull;
    return s;
}

// accumulate two slices (quad-row positions pm0, pm1 as a pair) into acc pairs
__device__ __forceinline__ void tap2(const ViewSetup &s, u64 PM, u64 &acc0, u64 &acc1)
{
    const u64 Q = add2(PM, pk(s.qmagic, s.qmagic));
    float q0, q1, p0, p1;
    upk(Q, q0, q1);
    upk(PM, p0, p1);
    const float4 g0 = ldq(s.colbase + ((u64)__float_as_uint(q0) << 4));
    const float4 g1 = ldq(s.colbase + ((u64)__float_as_uint(q1) << 4));
    fma2_acc(acc0, s.W, fma2(pk(g0.z, g0.w), pk(p0, p0), pk(g0.x, g0.y)));
    fma2_acc(acc1, s.W, fma2(pk(g1.z, g1.w), pk(p1, p1), pk(g1.x, g1.y)));
}

__device__ __forceinline__ void tap1(const ViewSetup &s, float pm, u64 &acc)
{
    const float q = pm + s.qmagic;
    const float4 g = ldq(s.colbase + ((u64)__float_as_uint(q) << 4));
    fma2_acc(acc, s.W, fma2(pk(g.z, g.w), pk(pm, pm), pk(g.x, g.y)));
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
    if (!(pm >= p.pm_lo && pm <= p.pm_hi)) return;
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
    const int nchunk = (p.nz + JZL - 1) / JZL;
    const int chunk = blockIdx.z % nchunk;
    const int item = blockIdx.z / nchunk;
    if (ix >= p.nx || iy >= p.ny) return;
    const int j0 = chunk * JZL;
    const int nzc = min(JZL, p.nz - j0);
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

    u64 acc[JZL];
#pragma unroll
    for (int t = 0; t < JZL; ++t) acc[t] = 0ull;

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
            for (int t = 0; t < JZL; ++t) {
                const float pm = fmaf((float)t, s.step, s.base);
                if ((mask & (1u << t)) && pm >= p.pm_lo && pm <= p.pm_hi) tap1(s, pm, acc[t]);
            }
        } else if (mask == (1u << JZL) - 1) {
            const u64 B = pk(s.base, s.base), S = pk(s.step, s.step);
#pragma unroll
            for (int t = 0; t < JZL; t += 2)
                tap2(s, fma2(pk((float)t, (float)(t + 1)), S, B), acc[t], acc[t + 1]);
        } else {
#pragma unroll
            for (int t = 0; t < JZL; ++t)
                if (mask & (1u << t)) tap1(s, fmaf((float)t, s.step, s.base), acc[t]);
        }
    }
    // end views: fractional weights ω_first, ω_last and the full range test
    const float2 *piw = p.pi_w + (size_t)j0 * plane + (size_t)iy * p.nx + ix;
#pragma unroll
    for (int t = 0; t < JZL; ++t) {
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
    for (int t = 0; t < JZL; ++t) {
        if (t < nzc) {
            float a, b;
            upk(acc[t], a, b);
            out[t * plane] = (a + b) * p.scale;
        }
    }
}

// ---------------------------------------------------------------------------
// Shared-memory staged, warp-specialized variant (interior views, detector
// margin check passed) — the default.  Per CTA, a producer warp plans the quad
// box (fp_cols x fp_rows) each view of the CTA's view range needs (from the
// tile's corner rays; 32 views per planning step, one per lane) and streams
// it with bulk async copies (cp.async.bulk, TMA engine) into a ring of slots
// guarded by full/empty mbarriers; 8 consumer warps read the taps with
// LDS.128 (4 wavefronts per warp instead of ~8 for scattered 128-bit global
// loads through L1) and release each slot with one mbarrier arrive.  No CTA
// barrier inside the view loop, so warps drift freely within the ring depth.
// ---------------------------------------------------------------------------
constexpr int kBoxesBytes = 128;  // (unused head); keeps the stage 128-B aligned for TMA
static_assert(kBoxesBytes % 16 == 0, "stage buffer must stay 16-byte aligned");

__device__ __forceinline__ void mbar_init(unsigned addr, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned addr, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
// producer-side wait: suspend in hardware until the phase completes (time hint 1 ms) so the
// waiting warp does not spin on issue slots
__device__ __forceinline__ void mbar_wait_sleep(unsigned addr, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, 1000000;\n\t"
        "@!done bra WAITS_%=;\n}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n}" ::"r"(addr), "r"(parity) : "memory");
}
// bulk async copy global -> shared (TMA engine), completion counted on an mbarrier
// 3-D tensor TMA: box {4*fp_rows floats, fp_cols columns, 1 view} at (4*r0, c0, view)
__device__ __forceinline__ void tma_box(unsigned dst, const CUtensorMap *map, int c_row, int c_col, int c_view, unsigned mbar)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c_row), "r"(c_col), "r"(c_view), "r"(mbar) : "memory");
}
// L2 prefetch of a box (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map, int c_row, int c_col, int c_view)
{
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c_row), "r"(c_col), "r"(c_view) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

template <bool POLY>
__device__ __forceinline__ float col_of(const BPParams &p, float x, float y, float c, float s)
{
    const float vstar = fmaf(-x, c, fmaf(-y, s, p.R));
    const float u = fmaf(y, c, -x * s);
    if (POLY) {
        const float t = u * rcp_approx(vstar), q = t * t;
        float a = p.at[6];
        a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
        a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
        return fmaf(t, a, p.col_c);
    }
    return fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
}

// quad box origin (first column, first quad row) for view k of a CTA tile
template <bool POLY>
__device__ __forceinline__ int2 plan_box(const BPParams &p, int k, float xa, float ya, float zb)
{
    const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
    const float xb = xa + (TX - 1) * p.dx, yb = ya + (TY - 1) * p.dy;
    float cmin = 1e30f, pmin = 1e30f;
    const float cx[4] = {xa, xb, xa, xb}, cy[4] = {ya, ya, yb, yb};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        cmin = fminf(cmin, col_of<POLY>(p, cx[q], cy[q], vg.x, vg.y));
        const float vstar = fmaf(-cx[q], vg.x, fmaf(-cy[q], vg.y, p.R));
        const float u = fmaf(cy[q], vg.x, -cx[q] * vg.y);
        const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
        const float p0 = fmaf(sc, zb - vg.z, p.row_c15);
        pmin = fminf(pmin, fminf(p0, fmaf(sc, (JZ - 1) * p.dz, p0)));
    }
    int c0 = (int)floorf(cmin) - 1, r0 = (int)floorf(pmin) - 1;
    c0 = max(0, min(c0, p.nc - p.fp_cols));
    r0 = max(0, min(r0, p.nr + 2 - p.fp_rows));
    return make_int2(c0, r0);
}

__device__ __forceinline__ void mbar_arrive(unsigned addr)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

// Warp-specialized: warps 0..7 consume (16x16 columns, 8x4 per warp), warp 8 produces.
constexpr int kConsumerWarps = (TX * TY) / 32;
constexpr int kWsThreads = TX * TY + 32;
constexpr int kMaxSlots = 16;
constexpr int kGroup = 8;          // window entries per conditional block (ILP vs. predicated-off waste)

// column of the tile's quad box for view k (rows: the whole detector)
template <bool POLY>
__device__ __forceinline__ int plan_col(const BPParams &p, int k, float xa, float ya)
{
    const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
    const float xb = xa + (TX - 1) * p.dx, yb = ya + (TY - 1) * p.dy;
    float cmin = fminf(fminf(col_of<POLY>(p, xa, ya, vg.x, vg.y), col_of<POLY>(p, xb, ya, vg.x, vg.y)),
                       fminf(col_of<POLY>(p, xa, yb, vg.x, vg.y), col_of<POLY>(p, xb, yb, vg.x, vg.y)));
    int c0 = (int)floorf(cmin) - 1;
    return max(0, min(c0, p.nc - p.fp_cols_column));
}

// End views of the staged kernels' slices, ahead of them: vol = the two fractional end-view taps
// (reading A9, full range tests) of every voxel, unscaled; the staged kernels finish a slice with
// vol = (interior sum + vol) * scale, so their warp-uniform flush has no dependent gathers.
template <bool POLY>
__global__ void __launch_bounds__(128) k_bp_ends(BPParams p)
{
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    const int t = blockIdx.z % p.nz, item = blockIdx.z / p.nz;
    if (ix >= p.nx) return;
    const size_t plane = (size_t)p.nx * p.ny, col = (size_t)iy * p.nx + ix;
    const int2 e = p.pi_k[(size_t)t * plane + col];
    float v = 0.f;
    if (e.x <= e.y) {
        const float2 w = p.pi_w[(size_t)t * plane + col];
        const u64 qbase = reinterpret_cast<u64>(p.gq) + (u64)((p.off0 + (int64_t)item * p.item_views) * p.viewbytes);
        const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
        u64 ends = 0ull;
        tap_checked<POLY>(p, qbase, e.x, x, y, 0.f, t, w.x, ends);
        tap_checked<POLY>(p, qbase, e.y, x, y, 0.f, t, w.y, ends);
        float ea, eb;
        upk(ends, ea, eb);
        v = ea + eb;
    }
    p.vol[(size_t)item * p.nz * plane + (size_t)t * plane + col] = v;
}

// column tile of a window-kernel CTA: the plan's heaviest-first order over a 1-D grid (the last wave
// holds the lightest, FOV-edge tiles: C2 1.383 -> 1.356 ms, C5 2.355 -> 2.329 ms), else the 2-D grid
__device__ __forceinline__ int2 bp_tile(const BPParams &p)
{
    if (!p.tile_order) return make_int2(blockIdx.x, blockIdx.y);
    const int t = __ldg(p.tile_order + blockIdx.x), ntx = (p.nx + TX - 1) / TX;
    return make_int2(t % ntx, t / ntx);
}

// Tensor maps of the staged kernels: box widths p.box_w[0] (= the largest box) >= [1] >= [2] columns.
struct QMaps { CUtensorMap m[3]; };
bool make_quad_map(const BPParams &p, int64_t n_views, CUtensorMap *map, int width, int height = 0);
// the three box widths of a plan: the full column box, 4/5 and 16/25 of it (C5: 56, 45, 36 columns;
// the tile widths of its views average 35.5)
inline void set_box_widths(BPParams &p)
{
    const int w = p.fp_cols_column;
    p.box_w[0] = w;
    p.box_w[1] = std::min(w, (4 * w + 4) / 5);
    p.box_w[2] = std::min(p.box_w[1], (16 * w + 24) / 25);
}
bool make_quad_maps(BPParams &p, QMaps *m)
{
    set_box_widths(p);
    for (int i = 0; i < 3; ++i)
        if (!make_quad_map(p, p.gq_views, &m->m[i], p.box_w[i])) return false;
    return true;
}

// Window kernel: box widths x heights (4 height classes: the staged column and three shorter ones),
// map index wcls * 4 + hcls
struct QMapsW { CUtensorMap m[12]; };
constexpr int kCropMaxZ = 64;      // row crop: per-slice tile windows in shared memory (nz <= 64)

// staged box of view k for a CTA tile: first column c0 (clamped like plan_col) and the narrowest
// width class covering the tile's corner-ray columns + 1 column of fp32 slack: c0 | class << 16
template <bool POLY>
__device__ __forceinline__ int plan_col_cls(const BPParams &p, int k, float xa, float ya)
{
    const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
    const float xb = xa + (TX - 1) * p.dx, yb = ya + (TY - 1) * p.dy;
    const float ca = col_of<POLY>(p, xa, ya, vg.x, vg.y), cb = col_of<POLY>(p, xb, ya, vg.x, vg.y);
    const float cc = col_of<POLY>(p, xa, yb, vg.x, vg.y), cd = col_of<POLY>(p, xb, yb, vg.x, vg.y);
    const float cmin = fminf(fminf(ca, cb), fminf(cc, cd)), cmax = fmaxf(fmaxf(ca, cb), fmaxf(cc, cd));
    const int c0 = max(0, min((int)floorf(cmin) - 1, p.nc - p.fp_cols_column));
    const int need = (int)floorf(cmax) + 2 - c0;
    const int cls = need <= p.box_w[2] ? 2 : need <= p.box_w[1] ? 1 : 0;
    return c0 | (cls << 16);
}

// the same, plus the quad rows of the view: the rows the tile's open slices [jlo, jhi] at view k
// reach (corner rays bound 1/sqrt(u^2 + v*^2) over the tile; one row of slack either side), inside
// the staged rows [q_lo, q_lo + nq_s); the shortest height class holding them and its first row r0:
// c0 | wcls << 16 | hcls << 20 | r0 << 24.  kf/kl: per-slice tile windows (min first / max last
// interior view over the tile's columns; nondecreasing in the slice)
template <bool POLY>
__device__ __forceinline__ int plan_box_crop(const BPParams &p, int k, float xa, float ya, const int *kf, const int *kl)
{
    const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
    const float xb = xa + (TX - 1) * p.dx, yb = ya + (TY - 1) * p.dy;
    const float ca = col_of<POLY>(p, xa, ya, vg.x, vg.y), cb = col_of<POLY>(p, xb, ya, vg.x, vg.y);
    const float cc = col_of<POLY>(p, xa, yb, vg.x, vg.y), cd = col_of<POLY>(p, xb, yb, vg.x, vg.y);
    const float cmin = fminf(fminf(ca, cb), fminf(cc, cd)), cmax = fmaxf(fmaxf(ca, cb), fmaxf(cc, cd));
    const int c0 = max(0, min((int)floorf(cmin) - 1, p.nc - p.fp_cols_column));
    const int need = (int)floorf(cmax) + 2 - c0;
    const int wcls = need <= p.box_w[2] ? 2 : need <= p.box_w[1] ? 1 : 0;
    int jlo = -1, jhi = -1;
    for (int j = 0; j < p.nz; ++j)
        if (kf[j] <= k && k <= kl[j]) { if (jlo < 0) jlo = j; jhi = j; }
    const int qa = p.q_lo, qb = p.q_lo + p.nq_s - 1;
    int hcls = 3, r0 = qa;
    if (jlo >= 0) {
        float smin = 3.4e38f, smax = 0.f;
        const float cx[4] = {xa, xb, xa, xb}, cy[4] = {ya, ya, yb, yb};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float vs = fmaf(-cx[q], vg.x, fmaf(-cy[q], vg.y, p.R)), us = fmaf(cy[q], vg.x, -cx[q] * vg.y);
            const float sc = p.D_over_dw * rsqrtf(fmaf(us * p.uu, us, vs * vs));
            smin = fminf(smin, sc); smax = fmaxf(smax, sc);
        }
        const float dlo = fmaf((float)jlo, p.dz, -vg.z), dhi = fmaf((float)jhi, p.dz, -vg.z);
        const float plo = p.row_c15 + (dlo >= 0.f ? smin * dlo : smax * dlo);
        const float phi = p.row_c15 + (dhi >= 0.f ? smax * dhi : smin * dhi);
        const int rlo = max(qa, (int)floorf(plo + 0.5f) - 1), rhi = min(qb, (int)floorf(phi + 0.5f) + 1);
        const int nr = rhi - rlo + 1;
        hcls = 0;
#pragma unroll
        for (int h = 1; h < 4; ++h)
            if (nr <= p.box_h[h]) hcls = h;
        r0 = min(rlo, qb + 1 - p.box_h[hcls]);
    }
    return c0 | (wcls << 16) | (hcls << 20) | (r0 << 24);
}

// ---------------------------------------------------------------------------
// Sliding-window kernel.  A thread owns a whole (x, y) column of the pitch and
// keeps W scalar accumulators for exactly the slices whose interior PI windows
// contain the current view (a contiguous, monotonically advancing slice range
// [t_lo, t_hi]; requires the host's monotone-window check).  Slices enter the
// window when their window opens and are flushed from its bottom (end views
// with their fractional weights added, volume written, registers shifted)
// when it closes, so no view does partial work and the per-(x, y, view) setup
// is shared by every active slice (~40 at C3/C4).
// ---------------------------------------------------------------------------
// Variants V (compile time, so the plain kernel's code is untouched by the others):
//   V = 0  plain;
//   V = 1  + warp-uniform sample tail: entries past every lane's last open slice are not sampled;
//   V = 2  + two batch items per CTA (C5: one-pitch slabs share the geometry, so each view's
//          per-lane setup serves both boxes) + 4 x 2 column blocks per quarter-warp (fewer
//          detector columns, hence bank groups, per LDS.128 wavefront).
// RING (row-cropped boxes, p.crop): the views' boxes are variable-size regions of one byte ring
// (p.ring_bytes) with 16 views of metadata (region offset, view geometry) in flight, instead of
// fixed slots sized for the largest box; one producer lane allocates regions in view order and
// waits for releases only when the ring is full.
template <bool POLY, int W, int V, bool RING = false>
// (the tensor map is the first parameter: it must sit 64-byte aligned in the parameter space)
__global__ void __launch_bounds__(kWsThreads, (W * (V == 3 ? 4 : V == 2 ? 2 : 1) <= 16 ? 3 : 2)) k_bp_window(const __grid_constant__ QMapsW qm, BPParams p)
{
    constexpr int NI = V == 3 ? 4 : V == 2 ? 2 : 1;                // V = 3: four items per CTA (byte ring only)
    constexpr bool TAIL = V >= 1, QMAP42 = V >= 2;
    extern __shared__ __align__(128) unsigned char smem[];
    const int BW = p.fp_cols_column, NQ = p.nq_s, S = RING ? kMaxSlots : p.nbatch;   // NQ: staged column pitch (quads)
    const int vq = (BW * NQ + 7) & ~7;                                   // quads per staged box (128-B aligned)
    const int vs = NI * vq;                                              // quads per slot (NI items' boxes)
    float4 *stage = reinterpret_cast<float4 *>(smem + kBoxesBytes);
    int *boxc = reinterpret_cast<int *>(smem + kBoxesBytes + (RING ? (size_t)p.ring_bytes : (size_t)S * vs * 16));   // first column per view
    __shared__ __align__(8) unsigned long long s_full[kMaxSlots], s_empty[kMaxSlots];
    __shared__ int s_k0, s_k1;
    __shared__ int s_kf[kCropMaxZ], s_kl[kCropMaxZ];             // row crop: per-slice tile windows
    __shared__ unsigned s_off[RING ? kMaxSlots : 1], s_end[RING ? kMaxSlots : 1];   // ring: region offset / end
    __shared__ float4 s_vgm[RING ? kMaxSlots : 1];                                  // ring: view geometry

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = warp == kConsumerWarps;
    // a warp owns 8 x 4 columns; each quarter-warp (the lanes one LDS.128 wavefront serves) a 4 x 2
    // block of them, so its samples spread over fewer detector columns (bank groups)
    const int2 bt = bp_tile(p);
    const int ix = bt.x * TX + (warp & 1) * 8 + (QMAP42 ? (lane & 3) + 4 * ((lane >> 3) & 1) : lane & 7);
    const int iy = bt.y * TY + (warp >> 1) * 4 + (QMAP42 ? ((lane >> 2) & 1) + 2 * (lane >> 4) : lane >> 3);
    const int item0 = blockIdx.z * NI;
    const bool inside = !producer && ix < p.nx && iy < p.ny;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)min(iy, p.ny - 1) * p.nx + min(ix, p.nx - 1);
    const int2 *pik = p.pi_k + col;
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&s_full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&s_empty[0]);

    if (tid == 0) {
        s_k0 = INT_MAX; s_k1 = INT_MIN;
        for (int i = 0; i < S; ++i) { mbar_init(full0 + 8u * i, 1); mbar_init(empty0 + 8u * i, TX * TY); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (p.crop)
        for (int t = tid; t < p.nz; t += kWsThreads) { s_kf[t] = INT_MAX; s_kl[t] = INT_MIN; }
    __syncthreads();
    int K0 = INT_MAX, K1 = INT_MIN;
    if (inside) {
        const int2 e0 = pik[0];
        if (e0.x <= e0.y) { K0 = e0.x + 1; K1 = pik[(size_t)(p.nz - 1) * plane].y - 1; }
    }
    int wk0 = K0, wk1 = K1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wk0 = min(wk0, __shfl_xor_sync(0xffffffffu, wk0, o));
        wk1 = max(wk1, __shfl_xor_sync(0xffffffffu, wk1, o));
    }
    if (lane == 0 && !producer) { atomicMin(&s_k0, wk0); atomicMax(&s_k1, wk1); }
    if (p.crop && !producer) {                                          // per-slice tile windows
        for (int t = 0; t < p.nz; ++t) {
            int a = INT_MAX, b = INT_MIN;
            if (inside && K0 <= K1) {
                const int2 e = pik[(size_t)t * plane];
                if (e.x + 1 <= e.y - 1) { a = e.x + 1; b = e.y - 1; }
            }
            a = __reduce_min_sync(0xffffffffu, a);
            b = __reduce_max_sync(0xffffffffu, b);
            if (lane == 0) { atomicMin(&s_kf[t], a); atomicMax(&s_kl[t], b); }
        }
    }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const u64 qbase = reinterpret_cast<u64>(p.gq) + (u64)((p.off0 + (int64_t)item0 * p.item_views) * p.viewbytes);
    const u64 qitem = (u64)(p.item_views * p.viewbytes);                // bytes between items' views
    __syncthreads();
    const int KC0 = s_k0, KC1 = s_k1;
    const int NV = KC1 - KC0 + 1;
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(stage);
    {
        const float xa = p.x0 + bt.x * TX * p.dx, ya = p.y0 + bt.y * TY * p.dy;
        if (p.crop)
            for (int n = tid; n < NV; n += kWsThreads) boxc[n] = plan_box_crop<POLY>(p, KC0 + n, xa, ya, s_kf, s_kl);
        else
            for (int n = tid; n < NV; n += kWsThreads)
                boxc[n] = plan_col_cls<POLY>(p, KC0 + n, xa, ya) | (((unsigned)p.q_lo) << 24);   // hcls 0 = nq_s
    }
    __syncthreads();

    if (RING && producer) {
        if (NV <= 0 || lane != 0) return;
        // ---- producer lane: view n's region [head, head + bytes) of the byte ring (absolute offsets;
        // a region never wraps: the ring's tail is skipped), free once every older view is released ----
        const int vbase = (int)(p.off0 + (int64_t)item0 * p.item_views) + KC0;
        const unsigned RB = (unsigned)p.ring_bytes;
        unsigned head = 0, hp = 0, rel_end = 0;
        int o = 0;
        for (int n = 0; n < NV; ++n) {
            const int ms = n & (kMaxSlots - 1);
            const int bc = boxc[n], wcls = (bc >> 16) & 15, hcls = (bc >> 20) & 15;
            const unsigned bytes = (unsigned)(p.box_w[wcls] * p.box_h[hcls]) * 16u, bb = (bytes + 127u) & ~127u;
            const unsigned last_end = head;                         // end of every region issued so far
            if (hp + NI * bb > RB) { head += RB - hp; hp = 0; }
            // the region's ring bytes last held absolute offsets [head + size - RB - size, head + size - RB):
            // free once every view ending there (never past the last issued one: the skipped tail) is released
            const unsigned need = head + NI * bb > RB ? min(head + NI * bb - RB, last_end) : 0u;
            while (o <= n - kMaxSlots || rel_end < need) {
                mbar_wait_sleep(empty0 + 8u * (o & (kMaxSlots - 1)), (unsigned)(o >> 4) & 1u);
                rel_end = s_end[o & (kMaxSlots - 1)];
                ++o;
            }
            s_end[ms] = head + NI * bb;
            s_off[ms] = hp;
            s_vgm[ms] = __ldg(reinterpret_cast<const float4 *>(p.view) + (KC0 + n - p.view_lo));
            const unsigned full = full0 + 8u * ms;
            mbar_expect_tx(full, NI * bytes);
#pragma unroll
            for (int i = 0; i < NI; ++i)
                tma_box(stage_sa + hp + (unsigned)i * bb, &qm.m[wcls * 4 + hcls], 2 * (int)((unsigned)bc >> 24),
                        bc & 0xFFFF, vbase + (int)(i * p.item_views) + n, full);
            if (p.ring_prefetch > 0 && n + p.ring_prefetch < NV) {     // the boxes of a view further ahead into L2
                const int m = n + p.ring_prefetch, bm = boxc[m];
                const CUtensorMap *map = &qm.m[((bm >> 16) & 15) * 4 + ((bm >> 20) & 15)];
#pragma unroll
                for (int i = 0; i < NI; ++i)
                    tma_prefetch(map, 2 * (int)((unsigned)bm >> 24), bm & 0xFFFF, vbase + (int)(i * p.item_views) + m);
            }
            head += NI * bb;
            hp += NI * bb;
        }
        return;
    }
    if (producer) {
        if (NV <= 0) return;
        // ---- producer warp: lanes 0..3 stream one view's column boxes (NI items) each per round ----
        const int vbase = (int)(p.off0 + (int64_t)item0 * p.item_views) + KC0;
        const int G = min(4, S);                              // lanes in flight; divides S (powers of 2)
        if (lane < G) {
            int sl = lane;
            unsigned phase = 0;
            for (int n = lane; n < NV; n += G) {
                if (n >= S) mbar_wait_sleep(empty0 + 8u * sl, phase ^ 1u);
                const unsigned full = full0 + 8u * sl;
                const int bc = boxc[n], wcls = (bc >> 16) & 15, hcls = (bc >> 20) & 15;
                mbar_expect_tx(full, NI * (unsigned)(p.box_w[wcls] * p.box_h[hcls]) * 16u);
#pragma unroll
                for (int i = 0; i < NI; ++i)
                    tma_box(stage_sa + (unsigned)(sl * vs + i * vq) * 16u, &qm.m[wcls * 4 + hcls], 2 * (int)((unsigned)bc >> 24),
                            bc & 0xFFFF, vbase + (int)(i * p.item_views) + n, full);
                sl += G;
                if (sl >= S) { sl -= S; phase ^= 1u; }
            }
        }
        return;
    }

    // ---- consumer warps ----
    float acc[NI][W];
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
        for (int i = 0; i < W; ++i) acc[b][i] = 0.f;
    const float2 *piw = p.pi_w + col;
    float *out = p.vol + (size_t)item0 * p.nz * plane + col;
    const bool active_col = inside && K0 <= K1;
    int t_lo = 0, t_hi = -1;
    int next_open = active_col ? K0 : INT_MAX, next_close = INT_MAX;

    // slice t_lo's window is closed: add its two end views, write it, shift the register window
    auto flush = [&]() {                                          // (end views: k_bp_ends wrote them to out)
#pragma unroll
        for (int b = 0; b < NI; ++b) {
            float *o = out + (size_t)b * p.nz * plane + (size_t)t_lo * plane;
            *o = (acc[b][0] + *o) * p.scale;
#pragma unroll
            for (int i = 0; i < W - 1; ++i) acc[b][i] = acc[b][i + 1];
            acc[b][W - 1] = 0.f;
        }
        ++t_lo;
        next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;   // b + 1 = k_last
    };

    const int lgS = __ffs(S) - 1;                                   // ring size is a power of two
    for (int n = 0; n < NV; ++n) {
        const int k = KC0 + n;
        const int sl = n & (S - 1);                                 // slot and parity from n: no live state
        mbar_wait(full0 + 8u * sl, (unsigned)(n >> lgS) & 1u);
        if (active_col) {
            while (k >= next_open) {                              // slice t_hi+1's interior window opens
                ++t_hi;
                if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
                next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
            }
            while (k >= next_close) flush();                      // slice t_lo's window closed
            const int n_act = t_hi - t_lo + 1;
            if (n_act > 0 && k <= K1) {
                const float4 vg = RING ? s_vgm[sl] : __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
                const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
                const float u = fmaf(y, vg.x, -x * vg.y);
                const float inv_v = rcp_approx(vstar);
                float colpos;
                if (POLY) {
                    const float tt = u * inv_v, q = tt * tt;
                    float a = p.at[6];
                    a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
                    a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
                    colpos = fmaf(tt, a, p.col_c);
                } else {
                    colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
                }
                const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
                const int l = __float2int_rz(cp);
                const float fa = cp - __int2float_rn(l);
                const float w1 = fa * inv_v, w0 = inv_v - w1;
                const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
                const float step = sc * p.dz;
                const float base = fmaf((float)t_lo, step, fmaf(sc, -vg.z, p.row_cc));    // entry 0 = slice t_lo
                const int bcn = boxc[n];
                const int ci = min(max(l - (bcn & 0xFFFF), 0), BW - 1);
                const unsigned H = (unsigned)p.box_h[(bcn >> 20) & 15], r0 = (unsigned)bcn >> 24;   // staged rows
                // ring: the view's region and the item stride (its box rounded to 128 B)
                const unsigned rbase = RING ? stage_sa + s_off[sl] : stage_sa + (unsigned)(sl * vs) * 16u;
                const unsigned ibytes = RING ? ((unsigned)p.box_w[(bcn >> 16) & 15] * H * 16u + 127u) & ~127u
                                             : (unsigned)vq * 16u;
                const u64 S2 = pk(2.f * step, 2.f * step);
                // (V >= 1) entries past every working lane's last open slice are not sampled at all
                int n_w = W;
                if constexpr (TAIL) n_w = __reduce_max_sync(__activemask(), n_act);
#pragma unroll
                for (int b = 0; b < NI; ++b) {
                    // XOR with a runtime zero keeps ptxas from re-splitting the magic offset: one LEA per sample
                    const unsigned colbase =
                        (rbase + (unsigned)b * ibytes + (unsigned)ci * H * 16u - (kMagicBits + r0) * 16u) ^ p.zero;
                    u64 PM = pk(base, base + step);
#pragma unroll
                    for (int g = 0; g < W; g += kGroup) {
                        if (g < n_act) {
#pragma unroll
                            for (int j = 0; j < kGroup; j += 2) {
                                const int i = g + j;
                                // entries >= n_act (not yet open) read at most a few quad rows past the
                                // column (a tail pad keeps them inside the allocation); their sums are dropped
                                const u64 Q = add2(PM, pk(p.qmagic, p.qmagic));
                                float q0, q1, p0, p1;
                                upk(Q, q0, q1);
                                upk(PM, p0, p1);
                                if constexpr (TAIL) {
                                    if (i >= n_w) break;
                                }
                                const float4 g0 = lds128(colbase + __float_as_uint(q0) * 16u);
                                const float4 g1 = lds128(colbase + __float_as_uint(q1) * 16u);
                                // the two columns' row samples s' + p d, then their α weights
                                float a0, b0, a1, b1;
                                upk(fma2(pk(g0.z, g0.w), pk(p0, p0), pk(g0.x, g0.y)), a0, b0);
                                upk(fma2(pk(g1.z, g1.w), pk(p1, p1), pk(g1.x, g1.y)), a1, b1);
                                if (i < n_act) acc[b][i] = fmaf(a0, w0, fmaf(b0, w1, acc[b][i]));
                                if (i + 1 < n_act) acc[b][i + 1] = fmaf(a1, w0, fmaf(b1, w1, acc[b][i + 1]));
                                PM = add2(PM, S2);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < kGroup; j += 2) PM = add2(PM, S2);
                        }
                    }
                }
            }
        }
        mbar_arrive(empty0 + 8u * sl);
    }
    if (!inside) return;
    if (!active_col) {                                            // outside U: the column is 0
        for (int b = 0; b < NI; ++b)
            for (int t = 0; t < p.nz; ++t) out[(size_t)b * p.nz * plane + (size_t)t * plane] = 0.f;
        return;
    }
    while (t_hi + 1 < p.nz) ++t_hi;                               // (all windows opened by K1)
    while (t_lo <= t_hi) flush();
}

// ---------------------------------------------------------------------------
// TMEM-window kernel (default; KATS_BP_KERNEL=window selects the register window): the sliding window of
// per-slice accumulators lives in tensor memory instead of registers.  Each
// lane owns one TMEM lane (row); slice t of the column accumulates in TMEM
// column t mod Wc of the warp's column range, so the window is a true circular
// buffer (no register shifts, no static unrolling over the window).  A warp
// walks the union of its lanes' open slices in groups of 8 columns
// (tcgen05.ld.32x32b.x8 -> FFMA work -> tcgen05.st.x8); a slice is flushed
// (end views, write, column zeroed) warp-uniformly once every lane has closed
// it.  Without the ~48 accumulator registers three CTAs share an SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tm_ld8_nowait(unsigned ta, float (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(ta));
}
// wait for the loads in flight; the registers are tied in so no use is scheduled before the wait
__device__ __forceinline__ void tm_wait_ld8(float (&v)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7])
                 :: "memory");
}
__device__ __forceinline__ void tm_st8(unsigned ta, const float (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(ta), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ float tm_ld1(unsigned ta)
{
    float v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return v;
}
__device__ __forceinline__ void tm_st1(unsigned ta, float v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "f"(v) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__host__ __device__ inline size_t tmem_head_bytes(const BPParams &p)
{
    return (16 * (size_t)p.pad_quads + 127) & ~(size_t)127;
}

size_t tmem_smem_bytes(const BPParams &p)
{
    const int vq = (p.fp_cols_column * p.nq_s + 7) & ~7;
    return tmem_head_bytes(p) + (size_t)p.nbatch * std::max(1, p.bp_items) * vq * sizeof(float4) +
           sizeof(int) * (size_t)p.max_cta_views + 16 * (size_t)p.pad_quads;
}

// PP = 2 (pitch pairs): the CTA backprojects two items (pitches) of the same tile: their windows,
// per-view geometry, group setup and flush points are identical (pitch-relative tables), so all of
// that is shared and only the samples double; each view's slot holds both items' boxes, each item
// has its own Wc TMEM columns per warp; the flush writes raw interior sums (end views and the
// Δλ/2π scale follow in k_bp_ends_add_t).  2 CTAs per SM.
// Q44: lanes of the warp's 8 x 4 columns in 4 x 2 quarter-warps / 4 x 4 half-warps instead of rows of 8:
// LDS.128 serves a half-warp in one wavefront when its adjacent lane pairs share quads and all its quads
// lie in one 128-byte segment, which compact half-warps meet more often (C3: K5 7.48 -> 7.20 ms; C4 no
// change, so the pitch-pair kernel keeps rows; scripts/ab/gpu_qmap44.sh, scripts/micro/lds128_merge.cu)
template <bool POLY, int VP, bool ENDS_PRE, int PP = 1, bool Q44 = false>
// (the tensor map is the first parameter: it must sit 64-byte aligned in the parameter space)
__global__ void __launch_bounds__(kWsThreads, PP == 1 ? 3 : 2) k_bp_tmem(const __grid_constant__ QMaps qm, BPParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int BW = p.fp_cols_column, NQ = p.nq_s, S = p.nbatch, Wc = p.tmem_cols;   // NQ: staged column pitch
    const int vq = (BW * NQ + 7) & ~7;
    const size_t head = tmem_head_bytes(p);                   // pad for reads below the first column
    float4 *stage = reinterpret_cast<float4 *>(smem + head);
    int *boxc = reinterpret_cast<int *>(smem + head + (size_t)S * PP * vq * 16);
    const unsigned box_bytes = 16u * (unsigned)vq;          // one item's box inside a slot
    __shared__ __align__(8) unsigned long long s_full[kMaxSlots], s_empty[kMaxSlots];
    __shared__ int s_k0, s_k1;
    __shared__ unsigned s_tmem;
    __shared__ float4 s_vg[kMaxSlots];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = warp == kConsumerWarps;
    const int ix = blockIdx.x * TX + (warp & 1) * 8 + (Q44 ? (lane & 3) + 4 * (lane >> 4) : lane & 7);
    const int iy = blockIdx.y * TY + (warp >> 1) * 4 + (Q44 ? (lane >> 2) & 3 : lane >> 3);
    const int item = blockIdx.z * PP;
    const bool inside = !producer && ix < p.nx && iy < p.ny;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)min(iy, p.ny - 1) * p.nx + min(ix, p.nx - 1);
    const int2 *pik = p.pi_k + col;
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&s_full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&s_empty[0]);

    if (warp == 0) {    // TMEM for the CTA: 2 x Wc columns (warps w and w+4 share a lane quarter)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"((unsigned)p.tmem_alloc));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        s_k0 = INT_MAX; s_k1 = INT_MIN;
        for (int i = 0; i < S; ++i) { mbar_init(full0 + 8u * i, 1); mbar_init(empty0 + 8u * i, TX * TY); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int K0 = INT_MAX, K1 = INT_MIN;
    if (inside) {
        const int2 e0 = pik[0];
        if (e0.x <= e0.y) { K0 = e0.x + 1; K1 = pik[(size_t)(p.nz - 1) * plane].y - 1; }
    }
    int wk0 = K0, wk1 = K1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wk0 = min(wk0, __shfl_xor_sync(0xffffffffu, wk0, o));
        wk1 = max(wk1, __shfl_xor_sync(0xffffffffu, wk1, o));
    }
    if (lane == 0 && !producer) { atomicMin(&s_k0, wk0); atomicMax(&s_k1, wk1); }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const u64 qbase = reinterpret_cast<u64>(p.gq) + (u64)((p.off0 + (int64_t)item * p.item_views) * p.viewbytes);
    __syncthreads();
    const int KC0 = s_k0, KC1 = s_k1;
    const int NV = KC1 - KC0 + 1;
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(stage);
    {
        const float xa = p.x0 + blockIdx.x * TX * p.dx, ya = p.y0 + blockIdx.y * TY * p.dy;
        for (int n = tid; n < NV; n += kWsThreads) boxc[n] = plan_col_cls<POLY>(p, KC0 + n, xa, ya);
    }
    __syncthreads();

    if (producer) {
        if (NV <= 0) return;
        const int vbase = (int)(p.off0 + (int64_t)item * p.item_views) + KC0;
        if (lane == 0) {
            int sl = 0;
            unsigned phase = 0;
            for (int n = 0; n < NV; ++n) {
                if (n >= S) mbar_wait_sleep(empty0 + 8u * sl, phase ^ 1u);
                const unsigned full = full0 + 8u * sl;
                // the view's geometry record rides with its slot (released by the arrive below)
                s_vg[sl] = __ldg(reinterpret_cast<const float4 *>(p.view) + (KC0 + n - p.view_lo));
                const int bc = boxc[n], cls = bc >> 16;
                mbar_expect_tx(full, (unsigned)(PP * p.box_w[cls] * NQ) * 16u);
#pragma unroll
                for (int b = 0; b < PP; ++b)
                    tma_box(stage_sa + (unsigned)(sl * PP * vq) * 16u + (unsigned)b * box_bytes, &qm.m[cls], 2 * p.q_lo,
                            bc & 0xFFFF, vbase + (int)(b * p.item_views) + n, full);
                if (++sl == S) { sl = 0; phase ^= 1u; }
            }
        }
        return;
    }

    // ---- consumer warps ----
    // quad row r of slot s, column c: slot0 + s*slot_bytes + c*col_bytes + (kMagicBits + r)*16 (the box's
    // first staged quad row is q_lo)
    const unsigned slot0 = stage_sa - (kMagicBits + (unsigned)p.q_lo) * 16u;
    // slice t -> TMEM column t mod Wc of the warp's range (lane = TMEM lane)
    const unsigned tw = s_tmem + (((unsigned)(warp & 3) * 32u) << 16) + (unsigned)((warp >> 2) * PP * Wc);
    {
        float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int c = 0; c < PP * Wc; c += 8) tm_st8(tw + c, z);
        tm_wait_st();
    }
    const float2 *piw = p.pi_w + col;
    float *out = p.vol + (size_t)item * p.nz * plane + col;
    const bool active_col = inside && K0 <= K1;
    int t_lo = 0, t_hi = -1, t_f = 0;                 // lane window [t_lo, t_hi]; warp flush point t_f
    int next_open = active_col ? K0 : INT_MAX, next_close = INT_MAX;

    // warp-uniform: slice t is closed in every lane -> finish and write it, zero its column
    // end views: either written ahead by k_bp_ends (ENDS_PRE; the next slice's value is loaded one
    // flush ahead) or sampled here (the kernel is LSU-bound and other warps hide the gathers: C4)
    float end_next = active_col && ENDS_PRE ? out[0] : 0.f;
    auto flush_pp = [&](int t) {                                  // pitch pairs: raw interior sums
#pragma unroll
        for (int b = 0; b < PP; ++b) {
            const unsigned tc = tw + (unsigned)(b * Wc) + ((unsigned)t & (unsigned)(Wc - 1));
            const float a = tm_ld1(tc);
            if (active_col && t < p.nz) out[(size_t)b * p.nz * plane + (size_t)t * plane] = a;
            tm_st1(tc, 0.f);
        }
    };
    auto flush_slice = [&](int t) {
        if constexpr (PP > 1) { flush_pp(t); return; }
        const unsigned tc = tw + ((unsigned)t & (unsigned)(Wc - 1));
        const float a = tm_ld1(tc);
        if (active_col && t < p.nz) {
            float ev;
            if constexpr (ENDS_PRE) {
                ev = end_next;
                if (t + 1 < p.nz) end_next = out[(size_t)(t + 1) * plane];
            } else {
                const int2 e = pik[(size_t)t * plane];
                const float2 w = piw[(size_t)t * plane];
                u64 ends = 0ull;
                tap_checked<POLY>(p, qbase, e.x, x, y, 0.f, t, w.x, ends);
                tap_checked<POLY>(p, qbase, e.y, x, y, 0.f, t, w.y, ends);
                float ea, eb;
                upk(ends, ea, eb);
                ev = ea + eb;
            }
            out[(size_t)t * plane] = (a + ev) * p.scale;
        }
        tm_st1(tc, 0.f);
    };

    // advance the lane's window [t_lo, t_hi] to view k (opens at k_first + 1, closes at k_last)
    auto advance = [&](int k) {
        if (!active_col) return;
        while (k >= next_open) {
            ++t_hi;
            if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
            next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
        }
        while (k >= next_close) {
            ++t_lo;
            next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;
        }
    };
    // the lane's sample geometry for a view: column weights (1/v* folded in), centred row position
    // of slice 0 and its per-slice step, box column
    auto geom = [&](const float4 vg, int n, float &w0, float &w1, float &base, float &step, int &ci) {
        const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
        const float u = fmaf(y, vg.x, -x * vg.y);
        const float inv_v = rcp_approx(vstar);
        float colpos;
        if (POLY) {
            const float tt = u * inv_v, q = tt * tt;
            float a = p.at[6];
            a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
            a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
            colpos = fmaf(tt, a, p.col_c);
        } else {
            colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
        }
        const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
        const int l = __float2int_rz(cp);
        const float fa = cp - __int2float_rn(l);
        w1 = fa * inv_v;
        w0 = inv_v - w1;
        const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
        step = sc * p.dz;
        base = fmaf(sc, -vg.z, p.row_cc);                       // slice 0 (centred quad-row position)
        ci = min(max(l - (boxc[n] & 0xFFFF), 0), BW - 1);
    };
    const unsigned wmask = (unsigned)Wc - 1u;                    // Wc is a power of two
    // 8 samples of one view for the group's slices (PM: packed positions of slices j, j+1)
    auto sample8 = [&](unsigned colbase, u64 PM, u64 S2, float (&v)[8][2]) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            const u64 Q = add2(PM, pk(p.qmagic, p.qmagic));
            float q0, q1, p0, p1;
            upk(Q, q0, q1);
            upk(PM, p0, p1);
            const float4 g0 = lds128(colbase + __float_as_uint(q0) * 16u);
            const float4 g1 = lds128(colbase + __float_as_uint(q1) * 16u);
            upk(fma2(pk(g0.z, g0.w), pk(p0, p0), pk(g0.x, g0.y)), v[j][0], v[j][1]);
            upk(fma2(pk(g1.z, g1.w), pk(p1, p1), pk(g1.x, g1.y)), v[j + 1][0], v[j + 1][1]);
            PM = add2(PM, S2);
        }
    };
    // a8 += w0 v0 + w1 v1 for the slices of the group inside the lane's window (fast: every slice)
    auto accum8 = [&](float (&a8)[8], const float (&v)[8][2], float w0, float w1, bool fast, int tb, int lo, int hi,
                      bool work) {
        if (fast) {
            // all 8 slices open in every working lane; idle lanes add exactly 0 (w = 0, finite reads)
#pragma unroll
            for (int j = 0; j < 8; ++j) a8[j] = fmaf(v[j][0], w0, fmaf(v[j][1], w1, a8[j]));
        } else {
            const int jl = min(max(lo - tb, 0), 8), jh = min(max(hi - tb + 1, 0), 8);
            const unsigned mask = work ? ((0xffu << jl) & ((1u << jh) - 1u)) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (mask & (1u << j)) a8[j] = fmaf(v[j][0], w0, fmaf(v[j][1], w1, a8[j]));
        }
    };

    if constexpr (VP == 1) {
    for (int n = 0; n < NV; ++n) {
        const int k = KC0 + n;
        const int sl = n & (S - 1);                   // ring size is a power of two
        mbar_wait(full0 + 8u * sl, (unsigned)(n >> p.lg_nbatch) & 1u);
        advance(k);
        const int lo_all = __reduce_min_sync(0xffffffffu, active_col ? t_lo : INT_MAX);
        while (t_f < lo_all && t_f < p.nz) flush_slice(t_f++);
        const bool work = active_col && t_hi >= t_lo && k <= K1;
        const int lo_w = __reduce_min_sync(0xffffffffu, work ? t_lo : INT_MAX);
        const int hi_w = __reduce_max_sync(0xffffffffu, work ? t_hi : -1);
        if (hi_w >= lo_w) {
            float w0 = 0.f, w1 = 0.f, base = 0.f, step = 0.f;
            int ci = 0;                                              // idle lanes read column 0 of the slot
            if (work) geom(s_vg[sl], n, w0, w1, base, step, ci);
            // XOR with a runtime zero keeps ptxas from re-splitting the magic offset: one LEA per sample
            const unsigned colbase = (slot0 + (unsigned)sl * p.slot_bytes + (unsigned)ci * p.col_bytes) ^ p.zero;
            // slices open in every working lane: groups inside [lo_full, hi_full] need no mask
            const int lo_full = __reduce_max_sync(0xffffffffu, work ? t_lo : INT_MIN);
            const int hi_full = __reduce_min_sync(0xffffffffu, work ? t_hi : INT_MAX);
            const u64 S2 = pk(2.f * step, 2.f * step), S8 = pk(8.f * step, 8.f * step);
            const int m0 = lo_w & ~7;
            unsigned cc = (unsigned)m0 & wmask;                      // column of the group's first slice
            // every read stays within (warp span + 7) slices of an open slice: the pads cover that
            u64 PM = pk(fmaf((float)m0, step, base), fmaf((float)(m0 + 1), step, base));
            for (int tb = m0; tb <= hi_w; tb += 8) {                 // warp-uniform groups of 8 slices
#pragma unroll
                for (int b = 0; b < PP; ++b) {
                    float a8[8];
                    tm_ld8_nowait(tw + (unsigned)(b * Wc) + cc, a8);
                    float v[8][2];
                    sample8(colbase + (unsigned)b * box_bytes, PM, S2, v);
                    if (b == PP - 1) PM = add2(PM, S8);
                    tm_wait_ld8(a8);
                    accum8(a8, v, w0, w1, tb >= lo_full && tb + 7 <= hi_full, tb, t_lo, t_hi, work);
                    tm_st8(tw + (unsigned)(b * Wc) + cc, a8);
                }
                cc = (cc + 8u) & wmask;
            }
            tm_wait_st();
        }
        mbar_arrive(empty0 + 8u * sl);
    }
    } else {
    // two consecutive views (A = k, B = k + 1) per pass: one window walk, flush, group setup and
    // TMEM load/store per group for both (the host sized Wc and the pads with the pair span)
    for (int n = 0; n < NV; n += 2) {
        const int k = KC0 + n;
        const bool hasB = n + 1 < NV;                                // warp-uniform
        const int slA = n & (S - 1), slB = (n + 1) & (S - 1);
        mbar_wait(full0 + 8u * slA, (unsigned)(n >> p.lg_nbatch) & 1u);
        if (hasB) mbar_wait(full0 + 8u * slB, (unsigned)((n + 1) >> p.lg_nbatch) & 1u);
        advance(k);
        const int loA = t_lo, hiA = t_hi;
        const bool workA = active_col && t_hi >= t_lo && k <= K1;
        const int lo_all = __reduce_min_sync(0xffffffffu, active_col ? t_lo : INT_MAX);
        while (t_f < lo_all && t_f < p.nz) flush_slice(t_f++);
        bool workB = false;
        if (hasB) {
            advance(k + 1);
            workB = active_col && t_hi >= t_lo && k + 1 <= K1;
        }
        const int loB = t_lo, hiB = t_hi;
        const int lo_w = __reduce_min_sync(0xffffffffu, min(workA ? loA : INT_MAX, workB ? loB : INT_MAX));
        const int hi_w = __reduce_max_sync(0xffffffffu, max(workA ? hiA : -1, workB ? hiB : -1));
        if (hi_w >= lo_w) {
            float w0A = 0.f, w1A = 0.f, baseA = 0.f, stepA = 0.f, w0B = 0.f, w1B = 0.f, baseB = 0.f, stepB = 0.f;
            int ciA = 0, ciB = 0;
            if (workA) geom(s_vg[slA], n, w0A, w1A, baseA, stepA, ciA);
            if (workB) geom(s_vg[slB], n + 1, w0B, w1B, baseB, stepB, ciB);
            const unsigned colA = (slot0 + (unsigned)slA * p.slot_bytes + (unsigned)ciA * p.col_bytes) ^ p.zero;
            // without a view B its (zero-weight) reads go to slot A, which holds finite data
            const unsigned colB = (slot0 + (unsigned)(hasB ? slB : slA) * p.slot_bytes + (unsigned)ciB * p.col_bytes) ^ p.zero;
            const int lo_fA = __reduce_max_sync(0xffffffffu, workA ? loA : INT_MIN);
            const int hi_fA = __reduce_min_sync(0xffffffffu, workA ? hiA : INT_MAX);
            const int lo_fB = __reduce_max_sync(0xffffffffu, workB ? loB : INT_MIN);
            const int hi_fB = __reduce_min_sync(0xffffffffu, workB ? hiB : INT_MAX);
            const int m0 = lo_w & ~7;
            unsigned cc = (unsigned)m0 & wmask;
            u64 PMA = pk(fmaf((float)m0, stepA, baseA), fmaf((float)(m0 + 1), stepA, baseA));
            u64 PMB = pk(fmaf((float)m0, stepB, baseB), fmaf((float)(m0 + 1), stepB, baseB));
            const u64 S2A = pk(2.f * stepA, 2.f * stepA), S2B = pk(2.f * stepB, 2.f * stepB);
            const u64 S8A = pk(8.f * stepA, 8.f * stepA), S8B = pk(8.f * stepB, 8.f * stepB);
            for (int tb = m0; tb <= hi_w; tb += 8) {
#pragma unroll
                for (int b = 0; b < PP; ++b) {
                    float a8[8];
                    tm_ld8_nowait(tw + (unsigned)(b * Wc) + cc, a8);
                    float v[8][2];
                    sample8(colA + (unsigned)b * box_bytes, PMA, S2A, v);
                    tm_wait_ld8(a8);
                    accum8(a8, v, w0A, w1A, tb >= lo_fA && tb + 7 <= hi_fA, tb, loA, hiA, workA);
                    sample8(colB + (unsigned)b * box_bytes, PMB, S2B, v);
                    accum8(a8, v, w0B, w1B, tb >= lo_fB && tb + 7 <= hi_fB, tb, loB, hiB, workB);
                    tm_st8(tw + (unsigned)(b * Wc) + cc, a8);
                }
                PMA = add2(PMA, S8A);
                PMB = add2(PMB, S8B);
                cc = (cc + 8u) & wmask;
            }
            tm_wait_st();
        }
        mbar_arrive(empty0 + 8u * slA);
        if (hasB) mbar_arrive(empty0 + 8u * slB);
    }
    }
    // every window has closed by K1 + 1: flush the rest
    const int hi_all = __reduce_max_sync(0xffffffffu, active_col ? p.nz - 1 : -1);
    while (t_f <= hi_all) flush_slice(t_f++);
    tm_wait_st();
    if (inside && !active_col)
        for (int b = 0; b < PP; ++b)
            for (int t = 0; t < p.nz; ++t) out[(size_t)b * p.nz * plane + (size_t)t * plane] = 0.f;
    // release TMEM once every consumer warp is done with it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(TX * TY));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"((unsigned)p.tmem_alloc));
}

// ---------------------------------------------------------------------------
// Items kernel (batches of one-pitch slabs whose windows hold <= 8 slices: the paper's training
// layer, C5).  All NI slabs of a CTA share the tile's geometry, so the per-(x, y, view) setup — v*,
// α*, the column, the row positions of the lane's open slices — is computed once per view and
// reused for the NI slabs, whose boxes stream through the ring one slab after the other (slot
// sequence (view 0, slab 0), (view 0, slab 1), ...).  A lane's accumulators live in tensor memory,
// 8 columns per slab in window-relative order (register j = slice t_lo + j of the lane): when a
// lane's window closes a slice it writes that slice's interior sum and shifts its 8 columns down
// (a per-lane flush; TMEM ld/st are warp-wide but each lane owns its row), so sampling touches only
// the lane's own open slices — a warp loop over the warp's widest window with a per-lane predicate,
// no samples of slices outside a lane's window.  The fractional end views and the Δλ/2π scale
// follow in k_bp_ends_add.
// ---------------------------------------------------------------------------
constexpr int kMaxItemSlots = 16;

template <bool POLY>
__global__ void __launch_bounds__(kWsThreads, 2) k_bp_items(const __grid_constant__ QMaps qm, BPParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int BW = p.fp_cols_column, NQ = p.nq_s, S = p.nbatch, NI = p.bp_items;
    const int vq = (BW * NQ + 7) & ~7;                                   // quads per slot (one slab's box)
    float4 *stage = reinterpret_cast<float4 *>(smem + kBoxesBytes);
    int *boxc = reinterpret_cast<int *>(smem + kBoxesBytes + (size_t)S * vq * 16);
    __shared__ __align__(8) unsigned long long s_full[kMaxItemSlots], s_empty[kMaxItemSlots];
    __shared__ int s_k0, s_k1;
    __shared__ unsigned s_tmem;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = warp == kConsumerWarps;
    const int2 bt = bp_tile(p);
    const int ix = bt.x * TX + (warp & 1) * 8 + (lane & 7);
    const int iy = bt.y * TY + (warp >> 1) * 4 + (lane >> 3);
    const int item0 = blockIdx.z * NI;
    const bool inside = !producer && ix < p.nx && iy < p.ny;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)min(iy, p.ny - 1) * p.nx + min(ix, p.nx - 1);
    const int2 *pik = p.pi_k + col;
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&s_full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&s_empty[0]);

    if (warp == 0) {    // TMEM: NI x 8 columns per warp, warps w and w + 4 share a lane quarter
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"((unsigned)p.tmem_alloc));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        s_k0 = INT_MAX; s_k1 = INT_MIN;
        for (int i = 0; i < S; ++i) { mbar_init(full0 + 8u * i, 1); mbar_init(empty0 + 8u * i, TX * TY); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int K0 = INT_MAX, K1 = INT_MIN;
    if (inside) {
        const int2 e0 = pik[0];
        if (e0.x <= e0.y) { K0 = e0.x + 1; K1 = pik[(size_t)(p.nz - 1) * plane].y - 1; }
    }
    int wk0 = K0, wk1 = K1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wk0 = min(wk0, __shfl_xor_sync(0xffffffffu, wk0, o));
        wk1 = max(wk1, __shfl_xor_sync(0xffffffffu, wk1, o));
    }
    if (lane == 0 && !producer) { atomicMin(&s_k0, wk0); atomicMax(&s_k1, wk1); }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    __syncthreads();
    const int KC0 = s_k0, KC1 = s_k1;
    const int NV = KC1 - KC0 + 1;
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(stage);
    {
        const float xa = p.x0 + bt.x * TX * p.dx, ya = p.y0 + bt.y * TY * p.dy;
        for (int n = tid; n < NV; n += kWsThreads) boxc[n] = plan_col_cls<POLY>(p, KC0 + n, xa, ya);
    }
    __syncthreads();

    if (producer) {
        if (NV > 0 && lane == 0) {
            const int vbase = (int)(p.off0 + (int64_t)item0 * p.item_views) + KC0;
            int sl = 0;
            unsigned phase = 0;
            int seq = 0;
            for (int n = 0; n < NV; ++n) {
                const int bc = boxc[n], cls = bc >> 16;
                const unsigned bytes = (unsigned)(p.box_w[cls] * NQ) * 16u;
                for (int b = 0; b < NI; ++b, ++seq) {
                    if (seq >= S) mbar_wait_sleep(empty0 + 8u * sl, phase ^ 1u);
                    const unsigned full = full0 + 8u * sl;
                    mbar_expect_tx(full, bytes);
                    tma_box(stage_sa + (unsigned)(sl * vq) * 16u, &qm.m[cls], 2 * p.q_lo, bc & 0xFFFF,
                            vbase + (int)(b * p.item_views) + n, full);
                    if (++sl == S) { sl = 0; phase ^= 1u; }
                }
            }
        }
    } else {
        // ---- consumer warps ----
        const unsigned tw = s_tmem + (((unsigned)(warp & 3) * 32u) << 16) + (unsigned)((warp >> 2) * NI * 8);
        {
            float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int b = 0; b < NI; ++b) tm_st8(tw + 8u * b, z);
            tm_wait_st();
        }
        const unsigned slot0 = stage_sa - (kMagicBits + (unsigned)p.q_lo) * 16u;
        float *out = p.vol + (size_t)item0 * p.nz * plane + col;
        const size_t item_stride = (size_t)p.nz * plane;
        const bool active_col = inside && K0 <= K1;
        int t_lo = 0, t_hi = -1;
        int next_open = active_col ? K0 : INT_MAX, next_close = INT_MAX;
        int sl = 0;
        unsigned phase = 0;
        for (int n = 0; n < NV; ++n) {
            const int k = KC0 + n;
            int d = 0;                                               // slices this lane closes at view k
            if (active_col) {
                while (k >= next_open) {
                    ++t_hi;
                    if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
                    next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
                }
                while (k >= next_close) {
                    ++t_lo; ++d;
                    next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;
                }
            }
            const int dmax = __reduce_max_sync(0xffffffffu, d);
            if (dmax > 0) {
                // per-lane flush: the closed slices' interior sums go out, the window shifts down
                for (int b = 0; b < NI; ++b) {
                    float a8[8];
                    tm_ld8_nowait(tw + 8u * b, a8);
                    tm_wait_ld8(a8);
                    for (int st = 0; st < dmax; ++st) {
                        const bool f = st < d;
                        if (f) out[(size_t)b * item_stride + (size_t)(t_lo - d + st) * plane] = a8[0];
#pragma unroll
                        for (int j = 0; j < 7; ++j) a8[j] = f ? a8[j + 1] : a8[j];
                        a8[7] = f ? 0.f : a8[7];
                    }
                    tm_st8(tw + 8u * b, a8);
                }
                tm_wait_st();
            }
            const bool work = active_col && t_hi >= t_lo && k <= K1;
            const int n_act = work ? t_hi - t_lo + 1 : 0;
            const int nw = __reduce_max_sync(0xffffffffu, n_act);
            if (nw > 0) {
                // the lane's geometry for view k, shared by the NI slabs
                const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
                float w0 = 0.f, w1 = 0.f, base = 0.f, step = 0.f;
                int ci = 0;
                if (work) {
                    const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
                    const float u = fmaf(y, vg.x, -x * vg.y);
                    const float inv_v = rcp_approx(vstar);
                    float colpos;
                    if (POLY) {
                        const float tt = u * inv_v, q = tt * tt;
                        float a = p.at[6];
                        a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
                        a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
                        colpos = fmaf(tt, a, p.col_c);
                    } else {
                        colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
                    }
                    const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
                    const int l = __float2int_rz(cp);
                    const float fa = cp - __int2float_rn(l);
                    w1 = fa * inv_v;
                    w0 = inv_v - w1;
                    const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
                    step = sc * p.dz;
                    base = fmaf((float)t_lo, step, fmaf(sc, -vg.z, p.row_cc));   // slice t_lo
                    ci = min(max(l - (boxc[n] & 0xFFFF), 0), BW - 1);
                }
                // row positions and quad offsets of the lane's window entries j = 0..7
                float pj[8];
                unsigned oj[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    pj[j] = fmaf((float)j, step, base);
                    oj[j] = __float_as_uint(pj[j] + p.qmagic) * 16u;
                }
                const unsigned cbase = (unsigned)ci * p.col_bytes;
                const unsigned amask = (1u << n_act) - 1u;               // the lane's open window entries
                // one slab: its box in slot sl; J window entries sampled (J = 4 covers most views)
                auto slab = [&](auto Jc, int b) {
                    constexpr int J = decltype(Jc)::value;
                    mbar_wait(full0 + 8u * sl, phase);
                    const unsigned colbase = (slot0 + (unsigned)sl * p.slot_bytes + cbase) ^ p.zero;
                    float a8[8];
                    tm_ld8_nowait(tw + 8u * b, a8);
                    float4 g[J];
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        g[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (amask & (1u << j)) g[j] = lds128(colbase + oj[j]);   // only the lane's own slices
                    }
                    mbar_arrive(empty0 + 8u * sl);
                    if (++sl == S) { sl = 0; phase ^= 1u; }
                    tm_wait_ld8(a8);
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        float v0, v1;
                        upk(fma2(pk(g[j].z, g[j].w), pk(pj[j], pj[j]), pk(g[j].x, g[j].y)), v0, v1);
                        a8[j] = fmaf(v0, w0, fmaf(v1, w1, a8[j]));
                    }
                    tm_st8(tw + 8u * b, a8);
                };
                if (nw <= 4) {
                    for (int b = 0; b < NI; ++b) slab(std::integral_constant<int, 4>{}, b);
                } else {
                    for (int b = 0; b < NI; ++b) slab(std::integral_constant<int, 8>{}, b);
                }
                tm_wait_st();
            } else {
                for (int b = 0; b < NI; ++b) {                       // nothing to sample: release the slots
                    mbar_wait(full0 + 8u * sl, phase);
                    mbar_arrive(empty0 + 8u * sl);
                    if (++sl == S) { sl = 0; phase ^= 1u; }
                }
            }
        }
        // every window has closed by K1 + 1: the lane's remaining open slices t_lo .. nz-1 (the TMEM loads
        // are warp-wide, the stores per lane)
        for (int b = 0; b < NI; ++b) {
            float a8[8];
            tm_ld8_nowait(tw + 8u * b, a8);
            tm_wait_ld8(a8);
            if (active_col) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (t_lo + j < p.nz) out[(size_t)b * item_stride + (size_t)(t_lo + j) * plane] = a8[j];
            } else if (inside) {
                for (int t = 0; t < p.nz; ++t) out[(size_t)b * item_stride + (size_t)t * plane] = 0.f;
            }
        }
    }
    // release TMEM once every consumer warp is done with it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"((unsigned)p.tmem_alloc));
}

// Register form of the items kernel (NI = 4 slabs per CTA): the lane's window-relative accumulators
// acc[b][j] (slab b, slice t_lo + j) stay in registers (32 of them), shifted down with selects when
// the lane closes a slice, so a slab's pass over a view is its box wait, the lane's own gathers and
// their accumulates — no TMEM round trip; the geometry is computed once per view for the 4 slabs.
constexpr int kItemsR = 4;

template <bool POLY>
__global__ void __launch_bounds__(kWsThreads, 3) k_bp_items_reg(const __grid_constant__ QMaps qm, BPParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int BW = p.fp_cols_column, NQ = p.nq_s, S = p.nbatch;
    const int vq = (BW * NQ + 7) & ~7;
    float4 *stage = reinterpret_cast<float4 *>(smem + kBoxesBytes);
    int *boxc = reinterpret_cast<int *>(smem + kBoxesBytes + (size_t)S * vq * 16);
    __shared__ __align__(8) unsigned long long s_full[kMaxItemSlots], s_empty[kMaxItemSlots];
    __shared__ int s_k0, s_k1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = warp == kConsumerWarps;
    const int2 bt = bp_tile(p);
    const int ix = bt.x * TX + (warp & 1) * 8 + (lane & 7);
    const int iy = bt.y * TY + (warp >> 1) * 4 + (lane >> 3);
    const int item0 = blockIdx.z * kItemsR;
    const bool inside = !producer && ix < p.nx && iy < p.ny;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)min(iy, p.ny - 1) * p.nx + min(ix, p.nx - 1);
    const int2 *pik = p.pi_k + col;
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&s_full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&s_empty[0]);
    if (tid == 0) {
        s_k0 = INT_MAX; s_k1 = INT_MIN;
        // one arrive per consumer warp releases a slot (lane 0, after the warp's gathers)
        for (int i = 0; i < S; ++i) { mbar_init(full0 + 8u * i, 1); mbar_init(empty0 + 8u * i, kConsumerWarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int K0 = INT_MAX, K1 = INT_MIN;
    if (inside) {
        const int2 e0 = pik[0];
        if (e0.x <= e0.y) { K0 = e0.x + 1; K1 = pik[(size_t)(p.nz - 1) * plane].y - 1; }
    }
    int wk0 = K0, wk1 = K1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wk0 = min(wk0, __shfl_xor_sync(0xffffffffu, wk0, o));
        wk1 = max(wk1, __shfl_xor_sync(0xffffffffu, wk1, o));
    }
    if (lane == 0 && !producer) { atomicMin(&s_k0, wk0); atomicMax(&s_k1, wk1); }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    __syncthreads();
    const int KC0 = s_k0, KC1 = s_k1;
    const int NV = KC1 - KC0 + 1;
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(stage);
    {
        const float xa = p.x0 + bt.x * TX * p.dx, ya = p.y0 + bt.y * TY * p.dy;
        for (int n = tid; n < NV; n += kWsThreads) boxc[n] = plan_col_cls<POLY>(p, KC0 + n, xa, ya);
    }
    __syncthreads();

    if (producer) {
        if (NV <= 0 || lane != 0) return;
        const int vbase = (int)(p.off0 + (int64_t)item0 * p.item_views) + KC0;
        int sl = 0, seq = 0;
        unsigned phase = 0;
        for (int n = 0; n < NV; ++n) {
            const int bc = boxc[n], cls = bc >> 16;
            const unsigned bytes = (unsigned)(p.box_w[cls] * NQ) * 16u;
            for (int b = 0; b < kItemsR; ++b, ++seq) {
                if (seq >= S) mbar_wait_sleep(empty0 + 8u * sl, phase ^ 1u);
                const unsigned full = full0 + 8u * sl;
                mbar_expect_tx(full, bytes);
                tma_box(stage_sa + (unsigned)(sl * vq) * 16u, &qm.m[cls], 2 * p.q_lo, bc & 0xFFFF,
                        vbase + (int)(b * p.item_views) + n, full);
                if (++sl == S) { sl = 0; phase ^= 1u; }
            }
        }
        return;
    }

    // ---- consumer warps ----
    const unsigned slot0 = stage_sa - (kMagicBits + (unsigned)p.q_lo) * 16u;
    float *out = p.vol + (size_t)item0 * p.nz * plane + col;
    const size_t item_stride = (size_t)p.nz * plane;
    const bool active_col = inside && K0 <= K1;
    float acc[kItemsR][8];
#pragma unroll
    for (int b = 0; b < kItemsR; ++b)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;
    int t_lo = 0, t_hi = -1;
    int next_open = active_col ? K0 : INT_MAX, next_close = INT_MAX;
    int sl = 0;
    unsigned phase = 0;
    for (int n = 0; n < NV; ++n) {
        const int k = KC0 + n;
        if (active_col) {
            while (k >= next_open) {
                ++t_hi;
                if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
                next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
            }
            while (k >= next_close) {                            // slice t_lo closed: write it, shift down
#pragma unroll
                for (int b = 0; b < kItemsR; ++b) {
                    out[(size_t)b * item_stride + (size_t)t_lo * plane] = acc[b][0];
#pragma unroll
                    for (int j = 0; j < 7; ++j) acc[b][j] = acc[b][j + 1];
                    acc[b][7] = 0.f;
                }
                ++t_lo;
                next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;
            }
        }
        const bool work = active_col && t_hi >= t_lo && k <= K1;
        const int n_act = work ? t_hi - t_lo + 1 : 0;
        const int nw = __reduce_max_sync(0xffffffffu, n_act);
        float w0 = 0.f, w1 = 0.f, base = 0.f, step = 0.f;
        int ci = 0;
        if (work) {
            const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
            const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
            const float u = fmaf(y, vg.x, -x * vg.y);
            const float inv_v = rcp_approx(vstar);
            float colpos;
            if (POLY) {
                const float tt = u * inv_v, q = tt * tt;
                float a = p.at[6];
                a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
                a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
                colpos = fmaf(tt, a, p.col_c);
            } else {
                colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
            }
            const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
            const int l = __float2int_rz(cp);
            const float fa = cp - __int2float_rn(l);
            w1 = fa * inv_v;
            w0 = inv_v - w1;
            const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
            step = sc * p.dz;
            base = fmaf((float)t_lo, step, fmaf(sc, -vg.z, p.row_cc));
            ci = min(max(l - (boxc[n] & 0xFFFF), 0), BW - 1);
        }
        const unsigned amask = (1u << n_act) - 1u;
        const unsigned cbase = (unsigned)ci * p.col_bytes;
        auto slab = [&](auto Jc, int b) {
            constexpr int J = decltype(Jc)::value;
            mbar_wait(full0 + 8u * sl, phase);
            const unsigned colbase = (slot0 + (unsigned)sl * p.slot_bytes + cbase) ^ p.zero;
            float4 g[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                g[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                const float pj = fmaf((float)j, step, base);
                if (amask & (1u << j)) g[j] = lds128(colbase + __float_as_uint(pj + p.qmagic) * 16u);
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const float pj = fmaf((float)j, step, base);
                float v0, v1;
                upk(fma2(pk(g[j].z, g[j].w), pk(pj, pj), pk(g[j].x, g[j].y)), v0, v1);
                acc[b][j] = fmaf(v0, w0, fmaf(v1, w1, acc[b][j]));
            }
            __syncwarp();                                        // the warp's gathers from this slot are done
            if (lane == 0) mbar_arrive(empty0 + 8u * sl);
            if (++sl == S) { sl = 0; phase ^= 1u; }
        };
        if (nw <= 4) {
#pragma unroll
            for (int b = 0; b < kItemsR; ++b) slab(std::integral_constant<int, 4>{}, b);
        } else {
#pragma unroll
            for (int b = 0; b < kItemsR; ++b) slab(std::integral_constant<int, 8>{}, b);
        }
    }
    if (!inside) return;
    if (!active_col) {
        for (int b = 0; b < kItemsR; ++b)
            for (int t = 0; t < p.nz; ++t) out[(size_t)b * item_stride + (size_t)t * plane] = 0.f;
        return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (t_lo + j < p.nz)
#pragma unroll
            for (int b = 0; b < kItemsR; ++b) out[(size_t)b * item_stride + (size_t)(t_lo + j) * plane] = acc[b][j];
}

// vol = (interior sum + the two fractional end views) * Δλ/2π for every voxel (after k_bp_items)
template <bool POLY>
__global__ void __launch_bounds__(128) k_bp_ends_add_t(BPParams p)
{
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    const int t = blockIdx.z % p.nz, item = blockIdx.z / p.nz;
    if (ix >= p.nx) return;
    const size_t plane = (size_t)p.nx * p.ny, col = (size_t)iy * p.nx + ix;
    float *o = p.vol + (size_t)item * p.nz * plane + (size_t)t * plane + col;
    const int2 e = p.pi_k[(size_t)t * plane + col];
    float v = *o;
    if (e.x <= e.y) {
        const float2 w = p.pi_w[(size_t)t * plane + col];
        const u64 qbase = reinterpret_cast<u64>(p.gq) + (u64)((p.off0 + (int64_t)item * p.item_views) * p.viewbytes);
        const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
        u64 ends = 0ull;
        tap_checked<POLY>(p, qbase, e.x, x, y, 0.f, t, w.x, ends);
        tap_checked<POLY>(p, qbase, e.y, x, y, 0.f, t, w.y, ends);
        float ea, eb;
        upk(ends, ea, eb);
        v += ea + eb;
    }
    *o = v * p.scale;
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
    const float rc = (float)(r - (nr + 2) / 2);          // centred quad row (as K4)
    q[i] = make_float4(fmaf(-rc, c0 - a0, 0.5f * (a0 + c0)), fmaf(-rc, c1 - a1, 0.5f * (a1 + c1)), c0 - a0, c1 - a1);
}

// ---------------------------------------------------------------------------
// Adjoint of step 7 (NEXT-1).  The forward reads, per interior
// update, one quad Q = (s'0, s'1, d0, d1) of column l at quad row r and adds
//   w0 (s'0 + P d0) + w1 (s'1 + P d1)         (times scale at the end),
// so its transpose adds  y scale (w0, w1, w0 P, w1 P)  to that quad of the
// quad-adjoint buffer gqT [views][nc][nr+2] (float4, same layout as gq).
// Same tiles, PI windows, geometry, box planning and quad selection as the
// forward kernels; per view, a CTA accumulates its box (the footprint the
// forward TMA-loads) in shared memory with atomics and reduce-adds it into
// gqT (red.global.add.v4.f32).  End views (fractional weights, checked
// samples) are scattered per voxel by k_bp_adjoint_ends.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_add4(float4 *dst, float a, float b, float c, float d)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Interior views, plans whose footprints stay on the detector.  Same lanes,
// windows and geometry as the forward kernels; per view the CTA accumulates its
// footprint box (the box the forward TMA-loads) in shared memory, then
// reduce-adds it into gqT (red.global.add.v4.f32).
//  * sm_100a has no native shared-memory float add (atomicAdd is a CAS loop, a
//    chain of shared-memory round trips); 32-bit integer ATOMS.ADD is native
//    and fire-and-forget.  So the box holds fixed-point int32 sums with one
//    scale per CTA and view for the (w0, w1) components and one for the
//    (w0 P, w1 P) components: S = 2^21 / B, B = the view's largest single
//    contribution bound over the CTA (column max |y| x 1/v*, x max |P| of the
//    window ends).  Float -> int is one FFMA against 1.5 * 2^23 (exact
//    round-to-nearest for |v| < 2^22); sums of up to 2^10 contributions fit.
//    Rounding error per contribution <= 2^-22 B.
//  * Lanes of a warp that share a detector column would hit the same quad at
//    the same step; a lane therefore walks its window in a rotated order
//    (starting 3 x lane slices in), so ATOMS rarely serialize.
//  * y (scaled) is staged once in shared memory, column-major with an odd
//    stride, so the rotated slice reads are conflict-free.
//  * CS > 0: the four component planes sit CS ints apart (compile time), so one
//    address per update serves all four atomics (immediate offsets); CS = 0:
//    planes BW x NQP ints apart, one address per component.
__device__ __forceinline__ void red_s32(unsigned saddr, int v)
{
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
template <int OFF>
__device__ __forceinline__ void red_s32_off(unsigned saddr, int v)
{
    asm volatile("red.shared.add.s32 [%0+%1], %2;" ::"r"(saddr), "n"(OFF), "r"(v) : "memory");
}
template <bool POLY, int CS>
__global__ void __launch_bounds__(TX *TY, 2) k_bp_adjoint(BPParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];   // one symbol per TU: keep the TMA kernels' alignment
    const int BW = p.fp_cols_column, NQ = p.nr + 2, nzp = p.nz | 1;
    const int NQP = p.adj_nqp, nbox = CS > 0 ? CS : BW * NQP;        // box column stride (launcher: 0 mod 32 or odd)
    const int cpy = 4 * nbox + 16;                                     // second copy: 16 banks further
    int *pl = reinterpret_cast<int *>(smem);                           // [2 copies][4][BW][NQP] fixed-point components
    float *ys = reinterpret_cast<float *>(pl + 2 * cpy);               // [TX*TY][nzp] scale * y
    int *boxc = reinterpret_cast<int *>(ys + TX * TY * nzp);
    __shared__ int s_k0, s_k1;
    __shared__ unsigned s_ymax;                                        // CTA max |scale * y| (float bits, >= 0)
    __shared__ int s_rect[2][4];                                       // box columns / quad rows touched (view parity)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ix = blockIdx.x * TX + (warp & 1) * 8 + (lane & 7);
    const int iy = blockIdx.y * TY + (warp >> 1) * 4 + (lane >> 3);
    const int item = blockIdx.z;
    const bool inside = ix < p.nx && iy < p.ny;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)min(iy, p.ny - 1) * p.nx + min(ix, p.nx - 1);
    const int2 *pik = p.pi_k + col;
    if (tid == 0) {
        s_k0 = INT_MAX; s_k1 = INT_MIN; s_ymax = 0u;
        for (int i = 0; i < 2; ++i) { s_rect[i][0] = INT_MAX; s_rect[i][1] = -1; s_rect[i][2] = INT_MAX; s_rect[i][3] = -1; }
    }
    for (int i = tid; i < 2 * cpy; i += TX * TY) pl[i] = 0;
    float ycmax = 0.f;                                                 // this column's max |scale * y|
    {
        const float *yv = p.vol + (size_t)item * p.nz * plane + col;
        float *yc = ys + tid * nzp;
        for (int t = 0; t < p.nz; ++t) {
            const float v = inside ? yv[(size_t)t * plane] * p.scale : 0.f;
            yc[t] = v;
            ycmax = fmaxf(ycmax, fabsf(v));
        }
    }
    __syncthreads();
    int K0 = INT_MAX, K1 = INT_MIN;
    if (inside) {
        const int2 e0 = pik[0];
        if (e0.x <= e0.y) { K0 = e0.x + 1; K1 = pik[(size_t)(p.nz - 1) * plane].y - 1; }
    }
    int wk0 = K0, wk1 = K1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wk0 = min(wk0, __shfl_xor_sync(0xffffffffu, wk0, o));
        wk1 = max(wk1, __shfl_xor_sync(0xffffffffu, wk1, o));
    }
    const unsigned wy = __reduce_max_sync(0xffffffffu, __float_as_uint(ycmax));
    if (lane == 0) { atomicMin(&s_k0, wk0); atomicMax(&s_k1, wk1); atomicMax(&s_ymax, wy); }
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    __syncthreads();
    // fixed-point scales for every view of the CTA: a contribution is at most max|scale*y| / v*
    // (w0 + w1 = 1/v*, v* >= R - the tile's farthest corner radius) for (w0, w1), times
    // |P| <= (n_rows - 1)/2 + 1 (interior samples lie in the detector rows) for (w0 P, w1 P)
    float B01, B23;
    {
        const float xa = p.x0 + blockIdx.x * TX * p.dx, ya = p.y0 + blockIdx.y * TY * p.dy;
        const float xb = xa + (TX - 1) * p.dx, yb = ya + (TY - 1) * p.dy;
        const float rx = fmaxf(fabsf(xa), fabsf(xb)), ry = fmaxf(fabsf(ya), fabsf(yb));
        const float vmin = p.R - sqrtf(rx * rx + ry * ry);
        B01 = __uint_as_float(s_ymax) / fmaxf(vmin, 1e-3f * p.R) * 1.001f;
        B23 = B01 * (0.5f * (float)p.nr + 1.5f);
    }
    const float S01 = B01 > 0.f ? 2097152.f / B01 : 0.f, S23 = B23 > 0.f ? 2097152.f / B23 : 0.f;
    const float i01 = B01 * (1.f / 2097152.f), i23 = B23 * (1.f / 2097152.f);
    const int KC0 = s_k0, NV = s_k1 - s_k0 + 1;
    {
        const float xa = p.x0 + blockIdx.x * TX * p.dx, ya = p.y0 + blockIdx.y * TY * p.dy;
        for (int n = tid; n < NV; n += TX * TY) boxc[n] = plan_col<POLY>(p, KC0 + n, xa, ya);
    }
    __syncthreads();
    float4 *qT = p.gqT + (p.off0 + (int64_t)item * p.item_views) * (p.viewbytes / 16);
    const bool active_col = inside && K0 <= K1;
    int t_lo = 0, t_hi = -1;
    int next_open = active_col ? K0 : INT_MAX, next_close = INT_MAX;
    const float *yc = ys + tid * nzp;
    for (int n = 0; n < NV; ++n) {
        const int k = KC0 + n;
        if (active_col) {
            while (k >= next_open) {
                ++t_hi;
                if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
                next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
            }
            while (k >= next_close) {
                ++t_lo;
                next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;
            }
        }
        const bool work = active_col && t_hi >= t_lo && k <= K1;
        float w0 = 0.f, w1 = 0.f, base = 0.f, step = 0.f;
        int ci = 0, rlo = 0, rhi = -1;
        if (work) {
            const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
            const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
            const float u = fmaf(y, vg.x, -x * vg.y);
            const float inv_v = rcp_approx(vstar);
            float colpos;
            if (POLY) {
                const float tt = u * inv_v, q = tt * tt;
                float a = p.at[6];
                a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
                a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
                colpos = fmaf(tt, a, p.col_c);
            } else {
                colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
            }
            const float cp = fminf(fmaxf(colpos, 0.f), p.colmax);
            const int l = __float2int_rz(cp);
            const float fa = cp - __int2float_rn(l);
            w1 = fa * inv_v;
            w0 = inv_v - w1;
            const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
            step = sc * p.dz;
            base = fmaf(sc, -vg.z, p.row_cc);
            ci = min(max(l - boxc[n], 0), BW - 1);
            const float plo = fmaf((float)t_lo, step, base), phi = fmaf((float)t_hi, step, base);
            rlo = (int)(__float_as_uint(plo + p.qmagic) - kMagicBits);    // rows grow with t
            rhi = (int)(__float_as_uint(phi + p.qmagic) - kMagicBits);
        }
        const int c_lo = __reduce_min_sync(0xffffffffu, work ? ci : INT_MAX);
        const int c_hi = __reduce_max_sync(0xffffffffu, work ? ci : -1);
        const int q_lo = __reduce_min_sync(0xffffffffu, work ? rlo : INT_MAX);
        const int q_hi = __reduce_max_sync(0xffffffffu, work ? rhi : -1);
        int *rect = s_rect[n & 1];
        if (lane == 0) {
            atomicMin(&rect[0], c_lo); atomicMax(&rect[1], c_hi);
            atomicMin(&rect[2], q_lo); atomicMax(&rect[3], q_hi);
        }
        if (work) {
            // component 0's byte address of quad row 0 minus the magic bits (the row's magic-rounded
            // float bits, times 4, complete it: one LEA per update); odd lanes: the shifted copy
            const unsigned a0 = (unsigned)__cvta_generic_to_shared(pl + (lane & 1) * cpy + ci * NQP) - kMagicBits * 4u;
            const float e0 = w0 * S01, e1 = w1 * S01, f0 = w0 * S23, f1 = w1 * S23;
            const int nt = t_hi - t_lo + 1;
            // rotated start: lane L begins ~L rows below lane 0 (consecutive banks for a shared column);
            // every lane walks its nt slices in lockstep, wrapping from t_hi to t_lo (y by byte address)
            const int t0 = t_lo + (int)((float)lane * __frcp_rn(step)) % nt;
            const unsigned ylo = (unsigned)__cvta_generic_to_shared(yc + t_lo), yhi = ylo + 4u * (unsigned)(nt - 1);
            unsigned ya = ylo + 4u * (unsigned)(t0 - t_lo);
            const float Plo = fmaf((float)t_lo, step, base);
            float P = fmaf((float)t0, step, base);
            for (int i = 0; i < nt; ++i) {
                const unsigned ad = a0 + __float_as_uint(P + p.qmagic) * 4u;
                float yy;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(yy) : "r"(ya));
                const float yP = yy * P;
                const int v0 = (int)(__float_as_uint(fmaf(e0, yy, kMagic)) - kMagicBits);
                const int v1 = (int)(__float_as_uint(fmaf(e1, yy, kMagic)) - kMagicBits);
                const int v2 = (int)(__float_as_uint(fmaf(f0, yP, kMagic)) - kMagicBits);
                const int v3 = (int)(__float_as_uint(fmaf(f1, yP, kMagic)) - kMagicBits);
                if constexpr (CS > 0) {
                    red_s32_off<0>(ad, v0);
                    red_s32_off<4 * CS>(ad, v1);
                    red_s32_off<8 * CS>(ad, v2);
                    red_s32_off<12 * CS>(ad, v3);
                } else {
                    const unsigned nb4 = 4u * (unsigned)nbox;
                    red_s32(ad, v0);
                    red_s32(ad + nb4, v1);
                    red_s32(ad + 2u * nb4, v2);
                    red_s32(ad + 3u * nb4, v3);
                }
                const bool wrap = ya == yhi;
                ya = wrap ? ylo : ya + 4u;
                P = wrap ? Plo : P + step;
            }
        }
        __syncthreads();                                               // the view's scatter and bounds are done
        const int rc0 = rect[0], rc1 = rect[1], rq0 = max(rect[2], 0), rq1 = min(rect[3], NQ - 1);
        if (tid == 0) {                                                // the next view's bounds (its readers,
            int *nr = s_rect[(n + 1) & 1];                             // view n - 1, passed the last barrier)
            nr[0] = INT_MAX; nr[1] = -1; nr[2] = INT_MAX; nr[3] = -1;
        }
        float4 *dst = qT + (int64_t)k * (p.viewbytes / 16) + (int64_t)boxc[n] * NQ;
        // only the rectangle of box columns x quad rows the view touched
        const int nqr = rq1 - rq0 + 1, ntouch = rc1 >= rc0 && nqr > 0 ? (rc1 - rc0 + 1) * nqr : 0;
        for (int i = tid; i < ntouch; i += TX * TY) {
            const int cc = rc0 + i / nqr, rr = rq0 + (i - (i / nqr) * nqr);
            const int j = cc * NQP + rr;
            int *q0 = pl + j, *q1 = pl + cpy + j;
            const int a = q0[0] + q1[0], b = q0[nbox] + q1[nbox], c = q0[2 * nbox] + q1[2 * nbox],
                      d = q0[3 * nbox] + q1[3 * nbox];
            if (a | b | c | d) {
                red_add4(dst + cc * NQ + rr, (float)a * i01, (float)b * i01, (float)c * i23, (float)d * i23);
                q0[0] = 0; q0[nbox] = 0; q0[2 * nbox] = 0; q0[3 * nbox] = 0;
                q1[0] = 0; q1[nbox] = 0; q1[2 * nbox] = 0; q1[3 * nbox] = 0;
            }
        }
        __syncthreads();
    }
}

// Interior views, plans whose footprints may leave the detector: per-sample range
// tests (reading A9) and a direct global scatter (the chunked L1 forward's transpose).
template <bool POLY>
__global__ void __launch_bounds__(TX *TY) k_bp_adjoint_checked(BPParams p)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ix = blockIdx.x * TX + (warp & 1) * 8 + (lane & 7);
    const int iy = blockIdx.y * TY + (warp >> 1) * 4 + (lane >> 3);
    const int item = blockIdx.z;
    if (ix >= p.nx || iy >= p.ny) return;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)iy * p.nx + ix;
    const int2 *pik = p.pi_k + col;
    const int2 e0 = pik[0];
    if (!(e0.x <= e0.y)) return;
    const int K0 = e0.x + 1, K1 = pik[(size_t)(p.nz - 1) * plane].y - 1;
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const float *yv = p.vol + (size_t)item * p.nz * plane + col;
    float4 *qT = p.gqT + (p.off0 + (int64_t)item * p.item_views) * (p.viewbytes / 16);
    const int NQ = p.nr + 2;
    int t_lo = 0, t_hi = -1, next_open = K0, next_close = INT_MAX;
    for (int k = K0; k <= K1; ++k) {
        while (k >= next_open) {
            ++t_hi;
            if (t_hi == t_lo) next_close = pik[(size_t)t_lo * plane].y;
            next_open = t_hi + 1 < p.nz ? pik[(size_t)(t_hi + 1) * plane].x + 1 : INT_MAX;
        }
        while (k >= next_close) {
            ++t_lo;
            next_close = t_lo <= t_hi ? pik[(size_t)t_lo * plane].y : INT_MAX;
        }
        if (t_hi < t_lo) continue;
        const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
        const float vstar = fmaf(-x, vg.x, fmaf(-y, vg.y, p.R));
        const float u = fmaf(y, vg.x, -x * vg.y);
        const float inv_v = rcp_approx(vstar);
        float colpos;
        if (POLY) {
            const float tt = u * inv_v, q = tt * tt;
            float a = p.at[6];
            a = fmaf(a, q, p.at[5]); a = fmaf(a, q, p.at[4]); a = fmaf(a, q, p.at[3]);
            a = fmaf(a, q, p.at[2]); a = fmaf(a, q, p.at[1]); a = fmaf(a, q, p.at[0]);
            colpos = fmaf(tt, a, p.col_c);
        } else {
            colpos = fmaf(atan2f(u, vstar), p.inv_dalpha, p.col_c);
        }
        if (!(colpos >= 0.f && colpos <= p.colmax)) continue;
        const int l = __float2int_rz(colpos);
        const float fa = colpos - __int2float_rn(l);
        const float w1 = fa * inv_v, w0 = inv_v - w1;
        const float sc = p.D_over_dw * rsqrt_approx(fmaf(u * p.uu, u, vstar * vstar));
        const float step = sc * p.dz, base = fmaf(sc, -vg.z, p.row_cc);
        float4 *qc = qT + (int64_t)k * (p.viewbytes / 16) + (int64_t)l * NQ;
        for (int t = t_lo; t <= t_hi; ++t) {
            const float P = fmaf((float)t, step, base);
            if (!(P >= p.pm_lo && P <= p.pm_hi)) continue;
            const int r = (int)(__float_as_uint(P + p.qmagic) - kMagicBits);
            const float yy = yv[(size_t)t * plane] * p.scale;
            red_add4(qc + r, w0 * yy, w1 * yy, w0 * yy * P, w1 * yy * P);
        }
    }
}

// end views of every voxel: checked samples with the fractional weights (reading A9)
template <bool POLY>
__global__ void k_bp_adjoint_ends(BPParams p)
{
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y, t = blockIdx.z % p.nz;
    const int item = blockIdx.z / p.nz;
    if (ix >= p.nx) return;
    const size_t plane = (size_t)p.nx * p.ny;
    const size_t col = (size_t)iy * p.nx + ix;
    const int2 e0 = p.pi_k[col];
    if (!(e0.x <= e0.y)) return;                                   // outside U: the forward writes 0
    const int2 e = p.pi_k[(size_t)t * plane + col];
    const float2 w = p.pi_w[(size_t)t * plane + col];
    const float yy = p.vol[((size_t)item * p.nz + t) * plane + col] * p.scale;
    const float x = p.x0 + ix * p.dx, y = p.y0 + iy * p.dy;
    const u64 qbase = reinterpret_cast<u64>(p.gqT) + (u64)((p.off0 + (int64_t)item * p.item_views) * p.viewbytes);
#pragma unroll
    for (int end = 0; end < 2; ++end) {
        const int k = end ? e.y : e.x;
        const float weight = end ? w.y : w.x;
        const float4 vg = __ldg(reinterpret_cast<const float4 *>(p.view) + (k - p.view_lo));
        const ViewSetup s = view_setup<POLY>(p, qbase + (u64)((int64_t)k * p.viewbytes), vg, x, y, 0.f);
        if (!(s.colpos >= 0.f && s.colpos <= p.colmax)) continue;
        const float pm = fmaf((float)t, s.step, s.base);
        if (!(pm >= p.pm_lo && pm <= p.pm_hi)) continue;
        float w0, w1;
        upk(s.W, w0, w1);
        const float g = yy * weight;
        const float q = pm + s.qmagic;
        float4 *dst = reinterpret_cast<float4 *>(s.colbase + ((u64)__float_as_uint(q) << 4));
        red_add4(dst, w0 * g, w1 * g, w0 * g * pm, w1 * g * pm);
    }
}

// grid.z carries (slices or z chunks) x items and is limited to 65535: split the items into groups
template <typename F>
static int for_item_groups(const BPParams &p, int zper, int even, F &&launch)
{
    int maxi = std::max(1, 65535 / std::max(1, zper));
    if (even && maxi > 1) maxi &= ~1;
    if (p.n_items <= maxi) return launch(p);
    int rc = 0;
    const size_t vol_item = (size_t)p.nz * p.nx * p.ny;
    for (int b0 = 0; b0 < p.n_items; b0 += maxi) {
        BPParams q = p;
        q.n_items = std::min(maxi, p.n_items - b0);
        q.off0 = p.off0 + (int64_t)b0 * p.item_views;
        q.vol = p.vol + (size_t)b0 * vol_item;
        rc = launch(q);
        if (rc < 0) return rc;
    }
    return rc;
}

static int launch_backproject_adjoint_items(const BPParams &p, cudaStream_t s);

int launch_backproject_adjoint(const BPParams &p, cudaStream_t s)
{
    if (!p.windows_monotone) return -1;
    return for_item_groups(p, p.nz, 0, [&](const BPParams &q) { return launch_backproject_adjoint_items(q, s); });
}

static int launch_backproject_adjoint_items(const BPParams &p, cudaStream_t s)
{
    // box column stride: 0 mod 32 banks when a warp's lanes share detector columns (rows, spread by
    // the rotated start, pick the bank: C3, C4); odd when they spread over many columns (C5: ~1.7
    // columns per voxel, 56-column boxes; 0 mod 32 made every lane of a row hit one bank)
    BPParams q = p;
    q.adj_nqp = p.fp_cols_column >= 48 ? ((p.nr + 2) | 1) : ((p.nr + 2 + 31) & ~31);
    if (const char *e = std::getenv("KATS_ADJ_PITCH"))
        q.adj_nqp = std::string(e) == "odd" ? ((p.nr + 2) | 1) : ((p.nr + 2 + 31) & ~31);
    // component planes at a compile-time stride (1024 or 2048 ints) when the box fits one, so the four
    // atomics of an update share one address (KATS_ADJ_CS=0: the runtime stride, A/B)
    const size_t nbox = (size_t)p.fp_cols_column * q.adj_nqp;
    // (only where the padding costs little shared memory: C5's 1064-int box at 2048 halved its CTAs per SM)
    int cs = nbox <= 1024 ? 1024 : nbox <= 2048 ? 2048 : 0;
    if (cs && 4 * (size_t)cs > 5 * nbox) cs = 0;
    if (const char *e = std::getenv("KATS_ADJ_CS")) cs = std::atoi(e) == 0 ? 0 : cs;
    const size_t sm = sizeof(int) * 2 * (4 * (cs ? (size_t)cs : nbox) + 16) +
                      sizeof(float) * (size_t)TX * TY * (p.nz | 1) + sizeof(int) * (size_t)p.max_cta_views;
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, p.n_items);
    // KATS_BP_KERNEL=l1: the checked kernel (A/B); also the fallback when the fixed-point box could overflow
    if (!p.checked && p.staged && p.adj_fixed_ok && sm <= 200 * 1024) {
        auto go = [&](auto kern) {
            smem_opt_in((const void *)kern, 200 * 1024);
            kern<<<grid, TX * TY, sm, s>>>(q);
        };
        if (cs == 1024) { if (p.poly) go(k_bp_adjoint<true, 1024>); else go(k_bp_adjoint<false, 1024>); }
        else if (cs == 2048) { if (p.poly) go(k_bp_adjoint<true, 2048>); else go(k_bp_adjoint<false, 2048>); }
        else { if (p.poly) go(k_bp_adjoint<true, 0>); else go(k_bp_adjoint<false, 0>); }
    } else {
        if (p.poly) k_bp_adjoint_checked<true><<<grid, TX * TY, 0, s>>>(p);
        else k_bp_adjoint_checked<false><<<grid, TX * TY, 0, s>>>(p);
    }
    dim3 ge((p.nx + 127) / 128, p.ny, p.nz * p.n_items);
    if (p.poly) k_bp_adjoint_ends<true><<<ge, 128, 0, s>>>(p);
    else k_bp_adjoint_ends<false><<<ge, 128, 0, s>>>(p);
    return 0;
}

void launch_make_quads(const float *gF, float4 *q, int64_t n, int nr, int nc, cudaStream_t s)
{
    const int64_t total = n * (nr + 2) * nc;
    k_make_quads<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gF, q, n, nr, nc);
}

size_t backproject_smem_bytes(const BPParams &p)
{
    const size_t vq = ((size_t)p.fp_cols_column * p.nq_s + 7) & ~(size_t)7;
    return kBoxesBytes + (size_t)p.nbatch * p.bp_items * vq * sizeof(float4) + sizeof(int) * (size_t)p.max_cta_views +
           16 * (size_t)p.tail_quads;
}

void launch_bp_ends(const BPParams &p, cudaStream_t s)
{
    dim3 g((p.nx + 127) / 128, p.ny, p.nz * p.n_items);
    if (p.poly) k_bp_ends<true><<<g, 128, 0, s>>>(p);
    else k_bp_ends<false><<<g, 128, 0, s>>>(p);
}

template <bool POLY, int VP, bool ENDS_PRE, int PP = 1>
void launch_tmem_kernel(const BPParams &q, dim3 grid, size_t sm, const QMaps &qmap, cudaStream_t s)
{
    if constexpr (PP == 1 && VP == 1) {
        if (q.qmap44) {
            smem_opt_in((const void *)k_bp_tmem<POLY, VP, ENDS_PRE, PP, true>, 200 * 1024);
            k_bp_tmem<POLY, VP, ENDS_PRE, PP, true><<<grid, kWsThreads, sm, s>>>(qmap, q);
            return;
        }
    }
    smem_opt_in((const void *)k_bp_tmem<POLY, VP, ENDS_PRE, PP>, 200 * 1024);
    k_bp_tmem<POLY, VP, ENDS_PRE, PP><<<grid, kWsThreads, sm, s>>>(qmap, q);
}

template <bool POLY>
void launch_tmem(const BPParams &q, int vp, dim3 grid, size_t sm, const QMaps &qmap, cudaStream_t s)
{
    if (q.bp_items == 2) {                                        // pitch pairs (ends added after)
        if (vp == 2) launch_tmem_kernel<POLY, 2, false, 2>(q, grid, sm, qmap, s);
        else launch_tmem_kernel<POLY, 1, false, 2>(q, grid, sm, qmap, s);
        return;
    }
    if (vp == 2) {
        if (q.ends_pre) launch_tmem_kernel<POLY, 2, true>(q, grid, sm, qmap, s);
        else launch_tmem_kernel<POLY, 2, false>(q, grid, sm, qmap, s);
    } else {
        if (q.ends_pre) launch_tmem_kernel<POLY, 1, true>(q, grid, sm, qmap, s);
        else launch_tmem_kernel<POLY, 1, false>(q, grid, sm, qmap, s);
    }
}

// window kernel maps: every (width, height) class pair
bool make_quad_maps_w(BPParams &p, QMapsW *m)
{
    set_box_widths(p);
    for (int i = 0; i < 3; ++i)
        for (int h = 0; h < 4; ++h)
            if (!make_quad_map(p, p.gq_views, &m->m[i * 4 + h], p.box_w[i], p.box_h[h])) return false;
    return true;
}

// height classes of the row crop: the staged column and the largest odd-bank-group heights (3 or 5
// mod 8, as the staged pitch) <= 3/4, 3/5 and 3/10 of it (C5: 19, 13, 11, 5 quad rows)
inline void set_box_heights(BPParams &p, bool crop)
{
    const int nq = p.nq_s;
    p.box_h[0] = nq;
    const float frac[3] = {0.75f, 0.6f, 0.3f};
    for (int h = 1; h < 4; ++h) {
        int v = crop ? (int)(frac[h - 1] * nq) : nq;
        while (v > 3 && (v & 7) != 3 && (v & 7) != 5) --v;
        v = std::max(3, std::min(v, p.box_h[h - 1]));
        p.box_h[h] = v;
    }
}

template <int W>
void launch_window(const BPParams &q, dim3 grid, size_t sm, const QMapsW &qmap, cudaStream_t s)
{
    auto go = [&](auto kern) {
        smem_opt_in((const void *)kern, 200 * 1024);
        kern<<<grid, kWsThreads, sm, s>>>(qmap, q);
    };
    const int v = q.win_variant;
    if constexpr (W <= 8) {
        if (q.ring_bytes > 0 && v == 3) {
            if (q.poly) go(k_bp_window<true, W, 3, true>); else go(k_bp_window<false, W, 3, true>);
            return;
        }
    }
    if constexpr (W <= 16) {
        if (q.ring_bytes > 0) {                                   // row-cropped boxes in a byte ring
            if (v == 2) { if (q.poly) go(k_bp_window<true, W, 2, true>); else go(k_bp_window<false, W, 2, true>); }
            else if (v == 1) { if (q.poly) go(k_bp_window<true, W, 1, true>); else go(k_bp_window<false, W, 1, true>); }
            else { if (q.poly) go(k_bp_window<true, W, 0, true>); else go(k_bp_window<false, W, 0, true>); }
            return;
        }
        if (v == 2) {
            if (q.poly) go(k_bp_window<true, W, 2>);
            else go(k_bp_window<false, W, 2>);
            return;
        }
    }
    if (v == 1) {
        if (q.poly) go(k_bp_window<true, W, 1>);
        else go(k_bp_window<false, W, 1>);
    } else {
        if (q.poly) go(k_bp_window<true, W, 0>);
        else go(k_bp_window<false, W, 0>);
    }
}

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    return fn;
}

}  // namespace

// 2-D fp32 tensor [dim1][dim0] (row stride stride1_bytes, a multiple of 16) with a box of box1 rows x
// box0 columns, no swizzle, zero fill out of bounds (used by the filter's warp-specialized Hilbert)
bool make_tensor_map_2d_f32(CUtensorMap *map, const float *base, uint64_t dim0, uint64_t dim1,
                            uint64_t stride1_bytes, uint32_t box0, uint32_t box1)
{
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)dim0, (cuuint64_t)dim1};
    const cuuint64_t strides[1] = {(cuuint64_t)stride1_bytes};
    const cuuint32_t box[2] = {box0, box1};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the quad array as a 3-D tensor of 8-byte elements: (2 * (nr+2) per column, nc columns, n_views);
// box = full column height x fp_cols_column columns x 1 view
bool make_quad_map(const BPParams &p, int64_t n_views, CUtensorMap *map, int width, int height)
{
    if (height <= 0) height = p.nq_s;
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)2 * (p.nr + 2), (cuuint64_t)p.nc, (cuuint64_t)n_views};
    const cuuint64_t strides[2] = {(cuuint64_t)(p.nr + 2) * 16, (cuuint64_t)p.viewbytes};
    // the box's column is p.nq_s quads from quad row p.q_lo (the rows interior samples can reach, |w| <=
    // w_L); rows past the detector are zero-filled (out of bounds); the pitch is an odd number of
    // 16-B bank groups
    const cuuint32_t box[3] = {(cuuint32_t)(2 * height), (cuuint32_t)width, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<float4 *>(p.gq), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int launch_backproject_items(const BPParams &p, cudaStream_t s);

int launch_backproject(const BPParams &p, cudaStream_t s)
{
    const int zper = std::max({(p.nz + JZ - 1) / JZ, (p.nz + JZL - 1) / JZL, p.nz});   // k_bp_ends: nz per item
    return for_item_groups(p, zper, 1, [&](const BPParams &q) { return launch_backproject_items(q, s); });
}

static int launch_backproject_items(const BPParams &p, cudaStream_t s)
{
    const int nchunk = (p.nz + JZ - 1) / JZ;
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, nchunk * p.n_items);
    const int nchunk_l1 = (p.nz + JZL - 1) / JZL;
    dim3 grid_l1((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, nchunk_l1 * p.n_items);
    const int block = TX * TY;
    const char *kv = std::getenv("KATS_BP_KERNEL");
    const bool want_window = kv && std::string(kv) == "window";
    const bool want_tmem = kv && std::string(kv) == "tmem";      // A/B: the TMEM kernel for narrow windows too
    // small grids: the staged kernels run one CTA per 16x16 column tile (and item); under one CTA per
    // SM the z-chunked L1 kernel's parallelism wins (C1, 16 tiles: K5 0.262 -> 0.074 ms)
    int nsm = 148;
    nsm = device_sms();
    const int64_t staged_ctas = (int64_t)((p.nx + TX - 1) / TX) * ((p.ny + TY - 1) / TY) * p.n_items;
    const bool small_grid = staged_ctas < nsm && !want_tmem && !want_window;
    // TMEM-window kernel for wide windows (accumulators in tensor memory, 3 CTAs per SM); for
    // windows of <= 32 slices the register window is lighter and faster (C2, C5 measured)
    // (also for windows of 17-32 slices when the items pair up: the pitch-pair TMEM kernel beats the
    // register window there, C2 1.70 -> 1.48 ms, scripts/ab/gpu_c2tmem.sh)
    const bool pairs_help = p.n_items % 2 == 0 && p.max_active > 16 && !std::getenv("KATS_BP_PP");
    if (!small_grid && !want_window && (p.max_active > 32 || pairs_help || want_tmem) && p.staged && !p.checked && p.windows_monotone &&
        p.warp_span > 0 &&
        2 * p.nq_s <= 256 &&
        p.fp_cols_column <= 256 && p.gq_views > 0 && p.pad_quads <= 2048) {
        // TMEM columns, allocation and ring depth for one view (vp 1) or two views (vp 2) per pass
        int qmap44 = 1;                                           // single items, one view per pass: 4 x 4 half-warps
        if (const char *qe = std::getenv("KATS_BP_QMAP")) qmap44 = std::atoi(qe) == 44;
        auto size_tmem = [&](int vp) {
            BPParams q = p;
            q.qmap44 = qmap44;
            const int span = vp == 2 ? std::max(p.warp_span, p.warp_span2) : p.warp_span;
            if (vp == 2) q.pad_quads = p.pad_quads2;
            q.tmem_cols = 16;                                     // power of two >= span + 2 alias-free groups
            while (q.tmem_cols < ((span + 7) & ~7) + 16) q.tmem_cols *= 2;
            int alloc = 32;
            while (alloc < 2 * q.tmem_cols) alloc *= 2;           // 2 warps per TMEM lane quarter
            q.tmem_alloc = alloc;
            // deepest power-of-two ring such that 3 CTAs fit in shared memory (and TMEM: 3 x alloc <= 512)
            q.nbatch = kMaxSlots;
            while (q.nbatch > 2 && tmem_smem_bytes(q) > 74 * 1024) q.nbatch /= 2;
            return q;
        };
        // view pairs halve the per-view overhead, but not at the price of TMEM (CTAs per SM) or ring
        // depth, and only with two pairs in flight (a 2-slot ring would stall the producer; C3 measured)
        const BPParams q1 = size_tmem(1), q2 = size_tmem(2);
        int vp = q2.tmem_alloc == q1.tmem_alloc && q2.nbatch == q1.nbatch && q2.nbatch >= 4 ? 2 : 1;
        if (const char *ve = std::getenv("KATS_BP_VP")) vp = std::string(ve) == "1" ? 1 : 2;   // A/B tests
        BPParams q = vp == 2 ? q2 : q1;
        // pitch pairs (default for an even number of items; KATS_BP_PP=1|2 for A/B): two items per CTA
        // share windows, per-view geometry, group setup and flushes; TMEM and the slots double, so
        // 2 CTAs per SM (scripts/ab/gpu_pp.sh: C4 K5 48.2 -> 45.5 ms, step 50.2 -> 47.4 ms; 44.2 / 46.1 ms
        // with one view per pass)
        int pp = 2;
        if (const char *pe = std::getenv("KATS_BP_PP")) pp = std::atoi(pe) == 2 ? 2 : 1;
        if (pp == 2 && p.n_items % 2 == 0) {
            const int vp0 = vp;
            // the pair already shares the per-view work: one view per pass is faster with it (C4 K5
            // 45.5 ms with view pairs, 44.2 ms without; scripts/ab: KATS_BP_VP under pitch pairs)
            if (!std::getenv("KATS_BP_VP")) { vp = 1; q = q1; }
            q.bp_items = 2;
            int alloc2 = 32;
            while (alloc2 < 2 * 2 * q.tmem_cols) alloc2 *= 2;
            q.tmem_alloc = alloc2;
            q.nbatch = kMaxSlots;
            while (q.nbatch > 2 && tmem_smem_bytes(q) > 110 * 1024) q.nbatch /= 2;
            if (alloc2 > 256 || (vp == 2 && q.nbatch < 4)) { vp = vp0; q = vp == 2 ? q2 : q1; }   // single items
        }
        const int alloc = q.tmem_alloc;
        q.lg_nbatch = __builtin_ctz((unsigned)q.nbatch);
        q.slot_bytes = 16u * (unsigned)((p.fp_cols_column * p.nq_s + 7) & ~7);
        q.col_bytes = 16u * (unsigned)p.nq_s;
        const size_t sm = tmem_smem_bytes(q);
        QMaps qmap;
        if ((alloc <= 128 || (q.bp_items == 2 && alloc <= 256)) && sm <= 200 * 1024 && make_quad_maps(q, &qmap)) {
            // (2-D tile grid: the heaviest-first order cost this kernel registers, C4 48.5 -> 50.6 ms)
            dim3 gw((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, p.n_items / q.bp_items);
            if (q.bp_items == 2) {
                q.slot_bytes = 16u * 2u * (unsigned)((p.fp_cols_column * p.nq_s + 7) & ~7);
                if (p.poly) launch_tmem<true>(q, vp, gw, sm, qmap, s);
                else launch_tmem<false>(q, vp, gw, sm, qmap, s);
                dim3 ge((p.nx + 127) / 128, p.ny, p.nz * p.n_items);
                if (p.poly) k_bp_ends_add_t<true><<<ge, 128, 0, s>>>(q);
                else k_bp_ends_add_t<false><<<ge, 128, 0, s>>>(q);
                return KATS_BP_TMEM;
            }
            // end views ahead (k_bp_ends) except for the LSU-bound view-pair kernel, where the inline
            // gathers are hidden by other warps (C4: 48.5 inline vs 48.9 ms; C3 7.69 -> 7.49 ms ahead)
            q.ends_pre = vp == 2 ? 0 : 1;
            if (const char *e = std::getenv("KATS_BP_ENDS")) q.ends_pre = std::string(e) == "pre";
            if (q.ends_pre) launch_bp_ends(q, s);
            if (p.poly) launch_tmem<true>(q, vp, gw, sm, qmap, s);
            else launch_tmem<false>(q, vp, gw, sm, qmap, s);
            return KATS_BP_TMEM;
        }
    }
    // items kernel (KATS_BP_ITEMS=N: N slabs per CTA): a batch of slabs whose windows hold <= 8 slices
    // (C5), the CTA's slabs sharing each view's geometry.  Measured slower than the register window
    // with two slabs per CTA (C5 K5 busy 2.43-2.48 vs 2.33 ms, scripts/ab/gpu_items2.sh: 2 CTAs per
    // SM for TMEM and a 6-box ring leave the box delivery and TMEM loads exposed), so opt-in only
    {
        int ni = 0;
        const char *ie = std::getenv("KATS_BP_ITEMS");
        if (ie) ni = std::atoi(ie);
        if (ni > 0 && (!small_grid || ie) && p.staged && !p.checked && p.windows_monotone && p.max_active <= 8 &&
            p.n_items % ni == 0 && ni <= 16 && 2 * p.nq_s <= 256 && p.fp_cols_column <= 256 && p.gq_views > 0) {
            BPParams q = p;
            q.bp_items = ni;
            q.tmem_alloc = 32;
            while (q.tmem_alloc < 2 * 8 * ni) q.tmem_alloc *= 2;       // 2 warps per TMEM lane quarter
            const int vq = (p.fp_cols_column * p.nq_s + 7) & ~7;
            q.slot_bytes = 16u * (unsigned)vq;
            q.col_bytes = 16u * (unsigned)p.nq_s;
            // ring: as many one-slab slots (<= 16) as leave room for 2 CTAs per SM (and TMEM: 2 x alloc <= 512)
            q.nbatch = kMaxItemSlots;
            auto smem_of = [&](const BPParams &r) {
                return kBoxesBytes + (size_t)r.nbatch * vq * sizeof(float4) + sizeof(int) * (size_t)r.max_cta_views +
                       16 * (size_t)r.tail_quads;
            };
            while (q.nbatch > 2 && smem_of(q) > 110 * 1024) --q.nbatch;
            const size_t sm = smem_of(q);
            QMaps qmap;
            if (ni == kItemsR && !std::getenv("KATS_BP_ITEMS_TMEM")) {
                // register accumulators (4 slabs): as deep a ring as leaves room for 3 CTAs per SM
                q.nbatch = kMaxItemSlots;
                while (q.nbatch > 2 && smem_of(q) > 74 * 1024) --q.nbatch;
                const size_t smr = smem_of(q);
                if (make_quad_maps(q, &qmap)) {
                    dim3 gw = p.tile_order ? dim3(((p.nx + TX - 1) / TX) * ((p.ny + TY - 1) / TY), 1, p.n_items / ni)
                                           : dim3((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, p.n_items / ni);
                    if (p.poly) {
                        smem_opt_in((const void *)k_bp_items_reg<true>, smr);
                        k_bp_items_reg<true><<<gw, kWsThreads, smr, s>>>(qmap, q);
                    } else {
                        smem_opt_in((const void *)k_bp_items_reg<false>, smr);
                        k_bp_items_reg<false><<<gw, kWsThreads, smr, s>>>(qmap, q);
                    }
                    dim3 ge((p.nx + 127) / 128, p.ny, p.nz * p.n_items);
                    if (p.poly) k_bp_ends_add_t<true><<<ge, 128, 0, s>>>(q);
                    else k_bp_ends_add_t<false><<<ge, 128, 0, s>>>(q);
                    return KATS_BP_ITEMS;
                }
            }
            if (q.tmem_alloc <= 256 && sm <= 200 * 1024 && make_quad_maps(q, &qmap)) {
                dim3 gw = p.tile_order ? dim3(((p.nx + TX - 1) / TX) * ((p.ny + TY - 1) / TY), 1, p.n_items / ni)
                                       : dim3((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, p.n_items / ni);
                if (p.poly) {
                    smem_opt_in((const void *)k_bp_items<true>, sm);
                    k_bp_items<true><<<gw, kWsThreads, sm, s>>>(qmap, q);
                } else {
                    smem_opt_in((const void *)k_bp_items<false>, sm);
                    k_bp_items<false><<<gw, kWsThreads, sm, s>>>(qmap, q);
                }
                dim3 ge((p.nx + 127) / 128, p.ny, p.nz * p.n_items);
                if (p.poly) k_bp_ends_add_t<true><<<ge, 128, 0, s>>>(q);
                else k_bp_ends_add_t<false><<<ge, 128, 0, s>>>(q);
                return KATS_BP_ITEMS;
            }
        }
    }
    BPParams q = p;
    const int W = p.max_active <= 8 ? 8 : p.max_active <= 16 ? 16 : p.max_active <= 32 ? 32 : p.max_active <= 48 ? 48 : 0;
    // batches of an even number of items with small windows: variant 2 (two items per CTA share
    // each view's per-lane geometry); otherwise the plain kernel (KATS_BP_WINV=0|1|2: A/B tests)
    q.win_variant = W > 0 && W <= 16 && p.n_items >= 2 && p.n_items % 2 == 0 ? 2 : 0;
    if (const char *wv = std::getenv("KATS_BP_WINV")) q.win_variant = std::atoi(wv);
    // four items per CTA for batches of slabs with <= 8-slice windows (C5: K5 2.15 -> 2.07 ms, scripts/ab/gpu_ni4.sh)
    if (W > 0 && W <= 8 && p.n_items % 4 == 0 && p.nz <= kCropMaxZ && !std::getenv("KATS_BP_WINV")) q.win_variant = 3;
    if (q.win_variant == 3 && !(W > 0 && W <= 8 && p.n_items % 4 == 0 && p.nz <= kCropMaxZ)) q.win_variant = 2;
    if (q.win_variant == 2 && !(W > 0 && W <= 16 && p.n_items % 2 == 0)) q.win_variant = 1;
    q.bp_items = q.win_variant == 3 ? 4 : q.win_variant == 2 ? 2 : 1;
    // sliding-window kernel: deepest slot ring (<= kMaxSlots views) that lets 3 CTAs (W * items <= 16,
    // <= 72 registers) or 2 CTAs share an SM
    const size_t budget = (W > 0 && W * q.bp_items <= 16 ? 74 : 100) * 1024;
    q.nbatch = kMaxSlots;
    while (q.nbatch > 2 && backproject_smem_bytes(q) > budget) q.nbatch /= 2;
    size_t sm = backproject_smem_bytes(q);
    // row crop (default for short slabs, nz <= 16; KATS_BP_CROP=0|1 for A/B): each view's box holds only
    // the quad rows of the tile's open slices (C5: 11.8 -> ~7 staged B/update), in a byte ring of
    // variable-size regions (W <= 16: the 3-CTA budget, at least two of the largest views)
    q.crop = p.nz <= 16 || q.win_variant == 3;
    if (const char *ce = std::getenv("KATS_BP_CROP")) q.crop = (std::atoi(ce) != 0 || q.win_variant == 3) && p.nz <= kCropMaxZ;
    set_box_heights(q, q.crop);
    auto size_ring = [&]() {
        q.ring_bytes = 0;
        if (!(q.crop && W > 0 && W <= 16)) return;
        const size_t rest = kBoxesBytes + sizeof(int) * (size_t)p.max_cta_views + 16 * (size_t)p.tail_quads;
        const size_t maxview = (size_t)q.bp_items * (((size_t)p.fp_cols_column * p.nq_s * 16 + 127) & ~(size_t)127);
        // (3 CTAs per SM: <= ~73.8 KB of dynamic shared memory next to the kernel's ~1.2 KB static; 2: ~111 KB)
        const size_t rbudget = (size_t)(W * q.bp_items <= 16 ? 72 : 108) * 1024;
        const size_t rb = rbudget > rest ? ((rbudget - rest) & ~(size_t)127) : 0;
        if (2 * rb >= 3 * maxview) { q.ring_bytes = (int)rb; sm = rest + rb; }   // >= 1.5 of the largest views
    };
    size_ring();
    q.ring_prefetch = 0;                                             // KATS_BP_RING_PF=N: L2 prefetch N views ahead
    if (const char *pf = std::getenv("KATS_BP_RING_PF")) q.ring_prefetch = std::max(0, std::atoi(pf));
    if (q.win_variant == 3 && q.ring_bytes == 0) {                   // four items need the ring
        q.win_variant = 2; q.bp_items = 2;
        q.nbatch = kMaxSlots;
        while (q.nbatch > 2 && backproject_smem_bytes(q) > (size_t)74 * 1024) q.nbatch /= 2;
        sm = backproject_smem_bytes(q);
        size_ring();
    }
    QMapsW qmap;
    if (!small_grid && p.staged && !p.checked && p.windows_monotone && W > 0 && sm <= 200 * 1024 && 2 * p.nq_s <= 256 &&
        p.tail_quads <= 4096 &&
        p.fp_cols_column <= 256 && p.gq_views > 0 && make_quad_maps_w(q, &qmap)) {
        dim3 gw = p.tile_order ? dim3(((p.nx + TX - 1) / TX) * ((p.ny + TY - 1) / TY), 1, p.n_items / q.bp_items)
                               : dim3((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY, p.n_items / q.bp_items);
        // the window kernel always finishes slices from end views written ahead (C5 2.55 -> 2.35 ms,
        // C2 1.43 -> 1.38 ms)
        q.ends_pre = 1;
        launch_bp_ends(q, s);
        switch (W) {
        case 8: launch_window<8>(q, gw, sm, qmap, s); break;
        case 16: launch_window<16>(q, gw, sm, qmap, s); break;
        case 32: launch_window<32>(q, gw, sm, qmap, s); break;
        default: launch_window<48>(q, gw, sm, qmap, s); break;
        }
        return KATS_BP_WINDOW;
    }
    if (p.poly) {
        if (p.checked) k_backproject<true, true><<<grid_l1, block, 0, s>>>(p);
        else k_backproject<true, false><<<grid_l1, block, 0, s>>>(p);
    } else {
        if (p.checked) k_backproject<false, true><<<grid_l1, block, 0, s>>>(p);
        else k_backproject<false, false><<<grid_l1, block, 0, s>>>(p);
    }
    return KATS_BP_L1;
}

}  // namespace kats
