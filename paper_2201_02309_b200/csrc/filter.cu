// filter.cu — filtering steps 1-6 of the Katsevich implementation of
// PAPER.md §II (l.117-154) as sm_100a kernels.  Each filtered view depends
// only on raw views v-1, v, v+1, so the same kernels serve the per-pitch slab
// (P:l.250) and the filter-once long-scan path.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>

#include "kernels.cuh"

namespace kats {

bool make_tensor_map_2d_f32(CUtensorMap *map, const float *base, uint64_t dim0, uint64_t dim1,
                            uint64_t stride1_bytes, uint32_t box0, uint32_t box1);   // backproject.cu

// ---------------------------------------------------------------------------
// K12: g3[v][i][l] = lerp_w(g2[v][·][l], w_κ(α_l, ψ_i)),  g2 = D/sqrt(D²+w²)·g1,
//      g1 = (∂_q + ∂_α) g   (Eqs. 8-11).  g2 is never materialised: the two
//      rows the κ-line sample needs are differentiated on the fly (centred
//      differences, one-sided at the α edges; reading A5).
// Grid: x over α (coalesced), y over ψ, z over views.
// ---------------------------------------------------------------------------
// K3 input element (line, column l): plain lines of nc floats, or parity-split lines (p.k3_in_split)
__device__ __forceinline__ size_t k3in_off(const FilterParams &p, size_t line, int l)
{
    return p.k3_in_split ? line * (size_t)(2 * p.hp) + (size_t)((l & 1) * p.hp + (l >> 1)) : line * (size_t)p.nc + l;
}

__device__ __forceinline__ float g2_at(const FilterParams &p, const float *__restrict__ gv, int m, int l)
{
    const int rs = p.nr * p.nc, vs = rs;
    const float *r = gv + m * p.nc;
    float dq = (__ldg(r + l + vs) - __ldg(r + l - vs)) * p.inv_2dlam;
    float da;
    if (l == 0) da = (__ldg(r + 1) - __ldg(r)) * p.inv_dalpha;
    else if (l == p.nc - 1) da = (__ldg(r + l) - __ldg(r + l - 1)) * p.inv_dalpha;
    else da = (__ldg(r + l + 1) - __ldg(r + l - 1)) * p.inv_2dalpha;
    return __ldg(p.wlen + m) * (dq + da);
}

// Flat detector (NEXT-4, reading A27): g2 = D/sqrt(D²+u²+w²) (∂_q + (u²+D²)/D ∂_u + uw/D ∂_w) g,
// the u and w differences centred, one-sided at the edges (as the α difference above).
__device__ __forceinline__ float g2_at_flat(const FilterParams &p, const float *__restrict__ gv, int m, int l)
{
    const int vs = p.nr * p.nc, nc = p.nc;
    const float *r = gv + m * nc;
    const float dq = (__ldg(r + l + vs) - __ldg(r + l - vs)) * p.inv_2dlam;
    float du, dw;
    if (l == 0) du = (__ldg(r + 1) - __ldg(r)) * p.inv_dalpha;
    else if (l == nc - 1) du = (__ldg(r + l) - __ldg(r + l - 1)) * p.inv_dalpha;
    else du = (__ldg(r + l + 1) - __ldg(r + l - 1)) * p.inv_2dalpha;
    if (m == 0) dw = (__ldg(r + nc + l) - __ldg(r + l)) * p.inv_dw;
    else if (m == p.nr - 1) dw = (__ldg(r + l) - __ldg(r - nc + l)) * p.inv_dw;
    else dw = (__ldg(r + nc + l) - __ldg(r - nc + l)) * p.inv_2dw;
    const float a = __ldg(p.flat_a + l);                                   // u / D
    const float wd = ((float)m - 0.5f * (float)(p.nr - 1)) * p.dw_over_D;   // w / D
    const float g1 = dq + p.D * fmaf(a, a, 1.f) * du + a * (wd * p.D) * dw;
    return rsqrtf(1.f + fmaf(a, a, wd * wd)) * g1;
}

// one thread per (view, column, kPsiPer κ-lines), as k_deriv_fwd_rebin below, with the flat g2
constexpr int kPsiPerFlat = 8;
__global__ void __launch_bounds__(256) k_deriv_fwd_rebin_flat(FilterParams p)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const int i0 = blockIdx.y * kPsiPerFlat;
    const int v = blockIdx.z;
    if (l >= p.nc) return;
    const int64_t g = p.view0 + v;
    const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
    const float *gv = p.sino + (size_t)raw * p.nr * p.nc;
    const size_t line0 = (size_t)v * p.npsi + i0;
#pragma unroll
    for (int j = 0; j < kPsiPerFlat; ++j) {
        if (i0 + j >= p.npsi) break;
        const RebinEntry e = p.fr[(i0 + j) * p.nc + l];
        float o = 0.f;
        if (e.idx >= 0) {
            const float a = g2_at_flat(p, gv, e.idx, l);
            const float b = g2_at_flat(p, gv, e.idx + 1, l);
            o = fmaf(e.frac, b - a, a);
        }
        p.g3[k3in_off(p, line0 + j, l)] = o;
    }
}

// A CTA spans a whole detector row (narrow detectors) and kPsiPer κ-lines of one view: each
// thread computes kPsiPer independent samples (loads in flight together); few, fat CTAs instead
// of one per (view, κ-line) (C4: 66K CTAs of 128 threads per chunk were launch-rate bound).
constexpr int kPsiPer = 8;

__global__ void __launch_bounds__(256) k_deriv_fwd_rebin(FilterParams p)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const int i0 = blockIdx.y * kPsiPer;
    const int v = blockIdx.z;
    if (l >= p.nc) return;
    const int64_t g = p.view0 + v;
    const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
    const float *gv = p.sino + (size_t)raw * p.nr * p.nc;
    const size_t line0 = (size_t)v * p.npsi + i0;
#pragma unroll
    for (int j = 0; j < kPsiPer; ++j) {
        if (i0 + j >= p.npsi) break;
        const RebinEntry e = p.fr[(i0 + j) * p.nc + l];
        float o = 0.f;
        if (e.idx >= 0) {
            const float a = g2_at(p, gv, e.idx, l);
            const float b = g2_at(p, gv, e.idx + 1, l);
            o = fmaf(e.frac, b - a, a);
        }
        p.g3[k3in_off(p, line0 + j, l)] = o;
    }
}

// Same computation, one thread per (view, column, <= 32 κ-lines) walking the κ-lines in ψ
// order: neighbouring κ-lines cross the same or adjacent detector rows, so the
// two g2 rows a sample needs are mostly already in hand (two-row cache);
// identical arithmetic to g2_at, coalesced along α for the table reads and the
// g3 stores.
__global__ void __launch_bounds__(128) k_deriv_fwd_rebin_col(FilterParams p, int seg)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
    const int i0 = blockIdx.z * seg, i1 = min(i0 + seg, p.npsi);   // this thread's κ-lines
    if (l >= p.nc) return;
    const int64_t g = p.view0 + v;
    const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
    const float *gv = p.sino + (size_t)raw * p.nr * p.nc;
    const size_t line0 = (size_t)v * p.npsi;
    int r0 = -2, r1 = -2;                                          // cached rows and their g2
    float c0 = 0.f, c1 = 0.f;
    for (int i = i0; i < i1; ++i) {
        const RebinEntry e = p.fr[i * p.nc + l];
        float o = 0.f;
        if (e.idx >= 0) {
            const int m = e.idx;
            float a, b;
            if (m == r0) { a = c0; b = (m + 1 == r1) ? c1 : g2_at(p, gv, m + 1, l); }
            else if (m == r1) { a = c1; b = g2_at(p, gv, m + 1, l); }
            else { a = g2_at(p, gv, m, l); b = g2_at(p, gv, m + 1, l); }
            r0 = m; c0 = a; r1 = m + 1; c1 = b;
            o = fmaf(e.frac, b - a, a);
        }
        p.g3[k3in_off(p, line0 + i, l)] = o;
    }
}

// Column walk over VPB views per thread (KATS_K12=colv2 / colv4): the view-independent rebin
// entries are loaded once for the VPB views and their stencil loads are issued together.
template <int VPB>
__global__ void __launch_bounds__(128) k_deriv_fwd_rebin_colv(FilterParams p, int seg)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, vb = blockIdx.y * VPB;
    const int i0 = blockIdx.z * seg, i1 = min(i0 + seg, p.npsi);   // this thread's κ-lines
    if (l >= p.nc) return;
    const int nv = min(VPB, p.n_views - vb);
    const float *gv[VPB];
#pragma unroll
    for (int j = 0; j < VPB; ++j) {
        const int64_t g = p.view0 + vb + min(j, nv - 1);
        const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
        gv[j] = p.sino + (size_t)raw * p.nr * p.nc;
    }
    int r0 = -2, r1 = -2;                                          // cached rows and their g2
    float c0[VPB], c1[VPB];
#pragma unroll
    for (int j = 0; j < VPB; ++j) c0[j] = c1[j] = 0.f;
    for (int i = i0; i < i1; ++i) {
        const RebinEntry e = p.fr[i * p.nc + l];
        float o[VPB];
        if (e.idx >= 0) {
            const int m = e.idx;
            float a[VPB], b[VPB];
            if (m == r0) {
                const bool hit = m + 1 == r1;
#pragma unroll
                for (int j = 0; j < VPB; ++j) { a[j] = c0[j]; b[j] = hit ? c1[j] : g2_at(p, gv[j], m + 1, l); }
            } else if (m == r1) {
#pragma unroll
                for (int j = 0; j < VPB; ++j) { a[j] = c1[j]; b[j] = g2_at(p, gv[j], m + 1, l); }
            } else {
#pragma unroll
                for (int j = 0; j < VPB; ++j) { a[j] = g2_at(p, gv[j], m, l); b[j] = g2_at(p, gv[j], m + 1, l); }
            }
            r0 = m; r1 = m + 1;
#pragma unroll
            for (int j = 0; j < VPB; ++j) { c0[j] = a[j]; c1[j] = b[j]; o[j] = fmaf(e.frac, b[j] - a[j], a[j]); }
        } else {
#pragma unroll
            for (int j = 0; j < VPB; ++j) o[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < VPB; ++j)
            if (j < nv) p.g3[k3in_off(p, (size_t)(vb + j) * p.npsi + i, l)] = o[j];
    }
}

// Same computation in two phases per (view, K12_TL-column tile): the CTA first computes g2 of the
// tile's nr x K12_TL samples (Eqs. 8-9) into shared memory, then the tile's npsi x K12_TL κ-line
// samples (Eqs. 10-11) read their two g2 rows from there.  A thread keeps one column and walks
// rows (phase 1) / κ-lines (phase 2) K12_RS apart with pointer increments: no per-item index
// division, unconditional unrolled loads (ncu, C4: the column walk spends ~77 instructions per
// sample on index math and a dependent table -> stencil chain, 34 us per 256-view chunk).
// α-derivative at the edges as g2_at: lp = min(l+1, nc-1), lm = max(l-1, 0), scale 1/((lp-lm)Δα).
constexpr int K12_TL = 64, K12_THREADS = 256, K12_RS = K12_THREADS / K12_TL;

__global__ void __launch_bounds__(K12_THREADS) k_deriv_fwd_rebin_tile(FilterParams p)
{
    extern __shared__ float g2s[];   // [nr][K12_TL]
    const int lt = threadIdx.x % K12_TL, r0 = threadIdx.x / K12_TL;
    const int nc = p.nc, l = blockIdx.x * K12_TL + lt, v = blockIdx.y;
    const bool col_ok = l < nc;
    const int lc = col_ok ? l : nc - 1;
    const int lp = min(lc + 1, nc - 1), lm = max(lc - 1, 0);
    const float sa = (lp - lm == 2) ? p.inv_2dalpha : p.inv_dalpha, sq = p.inv_2dlam;
    const int64_t g = p.view0 + v;
    const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
    const int vs = p.nr * nc;
    const float *r = p.sino + (size_t)raw * vs + (size_t)r0 * nc;
    float *gs = g2s + r0 * K12_TL + lt;
#pragma unroll 4
    for (int m = r0; m < p.nr; m += K12_RS) {
        const float dq = (__ldg(r + lc + vs) - __ldg(r + lc - vs)) * sq;
        const float da = (__ldg(r + lp) - __ldg(r + lm)) * sa;
        *gs = __ldg(p.wlen + m) * (dq + da);
        r += K12_RS * nc;
        gs += K12_RS * K12_TL;
    }
    __syncthreads();
    if (!col_ok) return;
    const size_t pitch = p.k3_in_split ? (size_t)(2 * p.hp) : (size_t)nc;
    const int co = p.k3_in_split ? (l & 1) * p.hp + (l >> 1) : l;
    float *out = p.g3 + ((size_t)v * p.npsi + r0) * pitch + co;
    const RebinEntry *t = p.fr + (size_t)r0 * nc + l;
    const float *gcol = g2s + lt;
#pragma unroll 4
    for (int i = r0; i < p.npsi; i += K12_RS) {
        const RebinEntry en = *t;
        const int ia = max(en.idx, 0);
        const float a = gcol[ia * K12_TL], b = gcol[(ia + 1) * K12_TL];
        *out = en.idx >= 0 ? fmaf(en.frac, b - a, a) : 0.f;
        t += K12_RS * nc;
        out += K12_RS * pitch;
    }
}


// Row form (default): a CTA = 8 warps on one 32-column block (lane = column) and a run of nvb
// consecutive views.  Per view, the warps first form g2 = D/sqrt(D²+w²)·(∂_q + ∂_α)g of the block's
// nr rows in shared memory (Eqs. 8-9; coalesced raw rows, the ±1-view and ±1-column stencil reads
// hit L1/L2), then its npsi κ-line samples (Eqs. 10-11) from there, with the block's rebin entries
// staged in shared memory once for all the CTA's views.  The raw stencil values of view j+1 are
// loaded into registers before view j's κ-line samples, so their latency overlaps that work; the
// g2 tile is double-buffered (one barrier per view).  Warps walk rows / κ-lines: no index
// division.  Same fp32 arithmetic as g2_at.
constexpr int K12R_WARPS = 8, K12R_MAXR = 8;   // rows per warp: nr <= 64

template <int MINB>
__global__ void __launch_bounds__(32 * K12R_WARPS, MINB) k_deriv_fwd_rebin_rows(FilterParams p, int nvb)
{
    extern __shared__ float k12s[];
    const int nr = p.nr, nc = p.nc, npsi = p.npsi, rs = nr * nc;
    float2 *tab = reinterpret_cast<float2 *>(k12s);                // [npsi][32]: (idx bits, frac)
    float *g2s = k12s + 2 * npsi * 32;                              // [2][nr][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int l = blockIdx.x * 32 + lane;
    const bool col_ok = l < nc;
    const int lc = col_ok ? l : nc - 1;
    const int lp = min(lc + 1, nc - 1), lm = max(lc - 1, 0);
    const float sa = (lp - lm == 2) ? p.inv_2dalpha : p.inv_dalpha, sq = p.inv_2dlam;
    for (int i = warp; i < npsi; i += K12R_WARPS) {
        const RebinEntry e = p.fr[(size_t)i * nc + lc];
        tab[i * 32 + lane] = make_float2(__int_as_float(e.idx), e.frac);
    }
    const int v0 = blockIdx.y * nvb, nv = min(nvb, p.n_views - v0);
    const size_t pitch = p.k3_in_split ? (size_t)(2 * p.hp) : (size_t)nc;
    const int co = p.k3_in_split ? (l & 1) * p.hp + (l >> 1) : l;
    float nx_[K12R_MAXR], pv_[K12R_MAXR], rt_[K12R_MAXR], lt_[K12R_MAXR];   // view j's stencil reads
    auto load_view = [&](int j) {
        const int64_t g = p.view0 + v0 + j;
        const int64_t raw = p.slab_views ? g + 2 * (g / p.slab_views) : g;
        const float *gv = p.sino + (size_t)raw * rs;
#pragma unroll
        for (int q = 0; q < K12R_MAXR; ++q) {
            const int m = warp + q * K12R_WARPS;
            if (m < nr) {
                const float *r = gv + (size_t)m * nc;
                nx_[q] = __ldg(r + lc + rs);
                pv_[q] = __ldg(r + lc - rs);
                rt_[q] = __ldg(r + lp);
                lt_[q] = __ldg(r + lm);
            }
        }
    };
    if (nv > 0) load_view(0);
    for (int j = 0; j < nv; ++j) {
        float *buf = g2s + (j & 1) * nr * 32;
#pragma unroll
        for (int q = 0; q < K12R_MAXR; ++q) {
            const int m = warp + q * K12R_WARPS;
            if (m < nr) {
                const float dq = (nx_[q] - pv_[q]) * sq;
                const float da = (rt_[q] - lt_[q]) * sa;
                buf[m * 32 + lane] = __ldg(p.wlen + m) * (dq + da);
            }
        }
        if (j + 1 < nv) load_view(j + 1);                          // in flight through the samples below
        // (view j+2 rewrites this buffer only after every thread passed view j+1's barrier, i.e.
        // after its reads of view j below)
        __syncthreads();
        if (col_ok) {
            float *out = p.g3 + (size_t)(v0 + j) * npsi * pitch + co;
            for (int i = warp; i < npsi; i += K12R_WARPS) {
                const float2 e = tab[i * 32 + lane];
                const int ia = __float_as_int(e.x);
                float o = 0.f;
                if (ia >= 0) {
                    const float a = buf[ia * 32 + lane], b = buf[(ia + 1) * 32 + lane];
                    o = fmaf(e.y, b - a, a);
                }
                out[(size_t)i * pitch] = o;
            }
        }
    }
}

// Warp-per-view form: each warp of a CTA owns one view (of a run of vpw views) on one 32-column
// block (lane = column): g2 of the block's rows into a warp-private shared-memory tile, then the
// npsi κ-line samples from it — no CTA barrier in the view loop; the block's rebin entries are
// staged once per CTA.  HALF (NEXT-4, reading A25): Noo's 2x2x2 half-sample derivative
// on the half-shifted grid (the plan's effective geometry: nr, nc are the shifted grid's sizes,
// raw views have nr + 1 rows and nc + 1 columns; effective view g reads raw views raw(g), raw(g)+1).
template <bool HALF, int UR = 4>
__global__ void __launch_bounds__(256) k_deriv_fwd_rebin_wv(FilterParams p, int vpw)
{
    extern __shared__ float k12s[];
    const int nr = p.nr, nc = p.nc, npsi = p.npsi;
    const int rnc = HALF ? nc + 1 : nc, rs = HALF ? (nr + 1) * (nc + 1) : nr * nc;   // raw row / view
    float2 *tab = reinterpret_cast<float2 *>(k12s);                // [npsi][32]: (idx bits, frac)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *g2w = k12s + 2 * npsi * 32 + warp * nr * 32;            // this warp's [nr][32]
    const int l = blockIdx.x * 32 + lane;
    const bool col_ok = l < nc;
    const int lc = col_ok ? l : nc - 1;
    for (int i = warp; i < npsi; i += 8) {
        const RebinEntry e = p.fr[(size_t)i * nc + lc];
        tab[i * 32 + lane] = make_float2(__int_as_float(e.idx), e.frac);
    }
    __syncthreads();
    const size_t pitch = p.k3_in_split ? (size_t)(2 * p.hp) : (size_t)nc;
    const int co = p.k3_in_split ? (l & 1) * p.hp + (l >> 1) : l;
    for (int jj = 0; jj < vpw; ++jj) {
        const int j = (blockIdx.y * 8 + warp) * vpw + jj;
        if (j >= p.n_views) break;
        const int64_t g = p.view0 + j;
        const int64_t raw = p.slab_views ? g + (HALF ? 1 : 2) * (g / p.slab_views) : g;
        const float *gv = p.sino + (size_t)raw * rs;
        if constexpr (HALF) {
            // rolling rows: raw row m of views k, k+1 at columns l, l+1
            const float sq = 0.25f * p.inv_2dlam * 2.f, sa = 0.25f * p.inv_dalpha;    // 1/(4Δλ), 1/(4Δα)
            const float *r0 = gv + lc, *r1 = gv + rs + lc;
            float a0 = __ldg(r0), a1 = __ldg(r0 + 1), b0 = __ldg(r1), b1 = __ldg(r1 + 1);
#pragma unroll 4
            for (int m = 0; m < nr; ++m) {
                r0 += rnc; r1 += rnc;
                const float c0 = __ldg(r0), c1 = __ldg(r0 + 1), d0 = __ldg(r1), d1 = __ldg(r1 + 1);
                // view differences (k+1) - k over the 2x2 (row, column) face, column differences over (view, row)
                const float dq = ((b0 - a0) + (b1 - a1)) + ((d0 - c0) + (d1 - c1));
                const float da = ((a1 - a0) + (b1 - b0)) + ((c1 - c0) + (d1 - d0));
                g2w[m * 32 + lane] = __ldg(p.wlen + m) * fmaf(dq, sq, da * sa);
                a0 = c0; a1 = c1; b0 = d0; b1 = d1;
            }
        } else {
            const int lp = min(lc + 1, nc - 1), lm = max(lc - 1, 0);
            const float sa = (lp - lm == 2) ? p.inv_2dalpha : p.inv_dalpha, sq = p.inv_2dlam;
#pragma unroll UR
            for (int m = 0; m < nr; ++m) {
                const float *r = gv + (size_t)m * nc;
                const float dq = (__ldg(r + lc + rs) - __ldg(r + lc - rs)) * sq;
                const float da = (__ldg(r + lp) - __ldg(r + lm)) * sa;
                g2w[m * 32 + lane] = __ldg(p.wlen + m) * (dq + da);
            }
        }
        __syncwarp();
        if (col_ok) {
            float *out = p.g3 + (size_t)j * npsi * pitch + co;
#pragma unroll 4
            for (int i = 0; i < npsi; ++i) {
                const float2 e = tab[i * 32 + lane];
                const int ia = __float_as_int(e.x);
                float o = 0.f;
                if (ia >= 0) {
                    const float a = g2w[ia * 32 + lane], b = g2w[(ia + 1) * 32 + lane];
                    o = fmaf(e.y, b - a, a);
                }
                out[(size_t)i * pitch] = o;
            }
        }
        __syncwarp();                                               // before the next view's g2
    }
}

// NEXT-4, reading A26 (Hann-apodised Hilbert): each κ-line smoothed in place by [1/4, 1/2, 1/4] along
// α (zeros beyond the detector columns) before K3; the same symmetric smoothing after K3^T in the
// adjoint.  A warp per line, the line staged in shared memory (plain or parity-split layout).
__global__ void __launch_bounds__(256) k_hann_smooth(FilterParams p, float *lines, int64_t n_lines, int split)
{
    extern __shared__ float hs[];
    const int nc = p.nc, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *t = hs + warp * nc;
    const size_t pitch = split ? (size_t)(2 * p.hp) : (size_t)nc;
    for (int64_t ln = (int64_t)blockIdx.x * 8 + warp; ln < n_lines; ln += (int64_t)gridDim.x * 8) {
        float *L = lines + (size_t)ln * pitch;
        for (int l = lane; l < nc; l += 32) t[l] = L[split ? (l & 1) * p.hp + (l >> 1) : l];
        __syncwarp();
        for (int l = lane; l < nc; l += 32) {
            const float o = 0.5f * t[l] + 0.25f * ((l > 0 ? t[l - 1] : 0.f) + (l + 1 < nc ? t[l + 1] : 0.f));
            L[split ? (l & 1) * p.hp + (l >> 1) : l] = o;
        }
        __syncwarp();
    }
}

void launch_hann_smooth(const FilterParams &p, float *lines, int64_t n_lines, int split, cudaStream_t s)
{
    const size_t smem = sizeof(float) * 8 * (size_t)p.nc;
    smem_opt_in((const void *)k_hann_smooth, smem);
    const int64_t blocks = std::min<int64_t>((n_lines + 7) / 8, 16 * (int64_t)device_sms());
    k_hann_smooth<<<(unsigned)std::max<int64_t>(blocks, 1), 256, smem, s>>>(p, lines, n_lines, split);
}

// ---------------------------------------------------------------------------
// K3: g4 = Σ_l' K[l-l'] g3[l'] along each κ-line (Eq. 12, h_H = 1/(πs) of
//     Eq. e4, band-limited kernel of DESIGN.md reading A10: only odd
//     distances contribute, so an output of parity p sums the inputs of
//     parity 1-p).  Direct convolution, register-tiled: a thread owns HR
//     consecutive same-parity outputs l0, l0+2, ..., keeps the HR kernel taps
//     they need in a register window that slides by one tap per input, so
//     each input costs 2 shared-memory loads for HR FMAs.  A CTA holds
//     several κ-lines (and the kernel) in shared memory.
// ---------------------------------------------------------------------------
constexpr int HR = 8;

__device__ __forceinline__ int hilbert_threads_per_line(int nc) { return 2 * (((nc + 1) / 2 + HR - 1) / HR); }

__global__ void __launch_bounds__(256) k_hilbert(FilterParams p, int64_t n_lines, int lines_per_block)
{
    extern __shared__ float smem[];
    const int nc = p.nc;
    constexpr int PAD = 2 * HR + 4;            // zero taps beyond |d| = nc-1 (windows of discarded outputs)
    float *ks = smem + PAD;                    // K[d] at ks[d + nc - 1], d = -(nc-1) .. nc-1
    float *gl = smem + 2 * nc - 1 + 2 * PAD;   // lines_per_block x nc
    const int64_t line0 = (int64_t)blockIdx.x * lines_per_block;
    const int nl = (n_lines - line0 < lines_per_block) ? (int)(n_lines - line0) : lines_per_block;
    for (int t = threadIdx.x; t < 2 * nc - 1 + 2 * PAD; t += blockDim.x)
        smem[t] = (t >= PAD && t < PAD + 2 * nc - 1) ? __ldg(p.hilbert + t - PAD) : 0.f;
    const float *src = p.g3 + line0 * nc;
    for (int t = threadIdx.x; t < nl * nc; t += blockDim.x) gl[t] = src[t];
    __syncthreads();
    const int tpl = hilbert_threads_per_line(nc);
    const int li = threadIdx.x / tpl, r = threadIdx.x - li * tpl;
    if (li >= nl) return;
    const int half = tpl / 2;
    const int par = r / half;                  // output parity
    const int l0 = par + 2 * HR * (r - par * half);
    if (l0 >= nc) return;
    const float *g = gl + li * nc;
    // inputs l' = 1-par, 3-par, ...; tap for output l0+2j and input l' is K[l0 + 2j - l']
    float acc[HR];
#pragma unroll
    for (int j = 0; j < HR; ++j) acc[j] = 0.f;
    const float *kk = ks + nc - 1 + l0;        // kk[2j - l'] = K[l0 + 2j - l']
    int lp = 1 - par;
    // window w[j] = K[l0 + 2j - lp]
    float w[HR];
#pragma unroll
    for (int j = 0; j < HR; ++j) w[j] = kk[2 * j - lp];
    for (; lp + 2 * (HR - 1) < nc; lp += 2 * HR) {
#pragma unroll
        for (int s = 0; s < HR; ++s) {
            const float gv = g[lp + 2 * s];
            // window for input lp + 2s: w[(j - s) mod HR] holds K[l0 + 2j - lp - 2s]
#pragma unroll
            for (int j = 0; j < HR; ++j) acc[j] = fmaf(w[(j - s + HR) % HR], gv, acc[j]);
            // slide: input lp+2s+2 needs slot i = -s-1, i.e. K[l0 - 2s - 2 - lp], in the slot
            // ((-s-1) mod HR) that held the tap of output HR-1-s just consumed
            w[(HR - 1 - s) % HR] = kk[-2 * s - 2 - lp];
        }
    }
    // remainder inputs (at most HR-1 of them)
    for (; lp < nc; lp += 2) {
        const float gv = g[lp];
#pragma unroll
        for (int j = 0; j < HR; ++j) acc[j] = fmaf(kk[2 * j - lp], gv, acc[j]);
    }
    float *dst = p.g4 + (line0 + li) * nc;
#pragma unroll
    for (int j = 0; j < HR; ++j)
        if (l0 + 2 * j < nc) dst[l0 + 2 * j] = p.sign * acc[j];
}

// ---------------------------------------------------------------------------
// K3 on the tensor cores (default when the taps fit): split by
// output parity the odd-tap convolution is a dense GEMM per parity,
//   g4[line][2n + par] = Σ_k g3[line][2k + 1 - par] · K[2(n - k) + 2 par - 1],
// M = κ-lines, N = K = ⌈n_α/2⌉ (padded to NH, a multiple of 32).  fp32
// accuracy from 3xTF32: A = A_h + A_l, B = B_h + B_l (A_h, B_h: fp32 with the
// low 13 mantissa bits cleared, exactly representable in TF32; the remainders
// are exact in fp32), D = A_h B_h + A_h B_l + A_l B_h accumulated in fp32 in
// TMEM (the dropped A_l B_l is ~2^-20 relative).  One CTA = 128 lines x one
// parity; 4 warps stage each 32-wide K chunk of A (split on the fly) and of the
// precomputed tap matrix (hi/lo, plan table) into shared memory in the
// canonical no-swizzle K-major UMMA layout (8-row x 16-byte core matrices:
// LBO = 128 B along K, SBO = 1024 B along M/N), one thread issues
// tcgen05.mma.kind::tf32 (M = 128, N <= 256 per instruction, K = 8) and
// commits to an mbarrier; the epilogue reads the accumulator with tcgen05.ld.
// ---------------------------------------------------------------------------
// operand staging is latency-bound: the per-parity kernel (one CTA per SM, TMEM-limited) stages with
// 16 warps, the two-parity kernel (two CTAs per SM) with 8; warps w, w+4, ... share a TMEM lane quarter
constexpr int TC_M = 128, TC_KC = 32, TC_THREADS = 512, TC2_THREADS = 256;

__host__ __device__ inline int hilbert_tc_nh(int nc) { return ((nc + 1) / 2 + 31) / 32 * 32; }

// canonical K-major offset (bytes) of element (row, k) in a [rows][32] chunk
__device__ __forceinline__ unsigned tc_off(int row, int k)
{
    return (unsigned)((row >> 3) * 1024 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t tc_desc(unsigned saddr)
{
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           (1ull << 46);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void __launch_bounds__(TC_THREADS, 1) k_hilbert_tc(FilterParams p, int64_t n_lines, int nstage)
{
    extern __shared__ __align__(1024) unsigned char tsm[];
    const int nc = p.nc, NH = hilbert_tc_nh(nc), NK = NH / TC_KC;
    const int par = blockIdx.y;                                  // output parity
    const int nin = (nc - (1 - par) + 1) / 2, nout = (nc - par + 1) / 2;
    const int64_t line0 = (int64_t)blockIdx.x * TC_M;
    // nstage = 2: chunk kc+1 is staged while the tensor core works on chunk kc (one mbarrier per stage)
    const unsigned stage_bytes = (unsigned)(2 * TC_M * TC_KC * 4 + 2 * NH * TC_KC * 4);
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ unsigned s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&s_bar[0]);
    if (warp == 0) {
        unsigned cols = 32;
        while (cols < (unsigned)NH) cols <<= 1;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    // instruction descriptor: D f32, A/B tf32, both K-major, M = 128
    const unsigned idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(TC_M >> 4) << 24);
    const float4 *btab = reinterpret_cast<const float4 *>(p.hilbert_tc) + (size_t)par * NK * 2 * NH * TC_KC / 4;
    for (int kc = 0; kc < NK; ++kc) {
        const int st = kc % nstage;
        if (kc >= nstage) {                                       // the MMAs of chunk kc - nstage read this stage
            asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                         "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                         "@!d bra WAIT_%=;\n\t}" ::"r"(bar0 + 8u * st), "r"((unsigned)(((kc - nstage) / nstage) & 1))
                         : "memory");
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        unsigned char *Ah = tsm + st * stage_bytes, *Al = Ah + TC_M * TC_KC * 4;
        unsigned char *Bh = Al + TC_M * TC_KC * 4, *Bl = Bh + NH * TC_KC * 4;
        const unsigned sAh = (unsigned)__cvta_generic_to_shared(Ah), sAl = (unsigned)__cvta_generic_to_shared(Al);
        const unsigned sBh = (unsigned)__cvta_generic_to_shared(Bh), sBl = (unsigned)__cvta_generic_to_shared(Bl);
        // A chunk: lane = (row within an 8-row group, k quad); a warp stores 512 contiguous bytes
        const int rr = lane & 7, kq = lane >> 3;
        for (int g = warp; g < TC_M / 8; g += TC_THREADS / 32) {
            const int row = g * 8 + rr;
            const int64_t line = line0 + row;
            const float *src = p.g3 + line * nc + (1 - par);
#pragma unroll
            for (int qb = 0; qb < 2; ++qb) {
                const int k0 = kc * TC_KC + (qb * 4 + kq) * 4;
                float v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    v[i] = (line < n_lines && k0 + i < nin) ? __ldg(src + 2 * (k0 + i)) : 0.f;
                const float4 h = make_float4(tf32_hi(v[0]), tf32_hi(v[1]), tf32_hi(v[2]), tf32_hi(v[3]));
                const unsigned o = tc_off(row, (qb * 4 + kq) * 4);
                *reinterpret_cast<float4 *>(Ah + o) = h;
                *reinterpret_cast<float4 *>(Al + o) = make_float4(v[0] - h.x, v[1] - h.y, v[2] - h.z, v[3] - h.w);
            }
        }
        // B chunk (hi, lo): already in the canonical layout in the plan table
        const float4 *bsrc = btab + (size_t)kc * 2 * NH * TC_KC / 4;
        float4 *bdst = reinterpret_cast<float4 *>(Bh);
        for (int i = tid; i < 2 * NH * TC_KC / 4; i += TC_THREADS) bdst[i] = __ldg(bsrc + i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int n0 = 0; n0 < NH; n0 += 256) {
                const int nn = NH - n0 < 256 ? NH - n0 : 256;
                const unsigned idesc = idesc_base | ((unsigned)(nn >> 3) << 17);
                const unsigned boff = (unsigned)(n0 / 8) * 1024u;
#pragma unroll
                for (int kk = 0; kk < TC_KC / 8; ++kk) {
                    const unsigned ko = (unsigned)kk * 256u;
                    const uint64_t a_h = tc_desc(sAh + ko), a_l = tc_desc(sAl + ko);
                    const uint64_t b_h = tc_desc(sBh + boff + ko), b_l = tc_desc(sBl + boff + ko);
                    const unsigned first = (kc == 0 && kk == 0) ? 0u : 1u;
                    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}"
                                 ::"r"(tmem + (unsigned)n0), "l"(a_h), "l"(b_h), "r"(idesc), "r"(first));
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                 ::"r"(tmem + (unsigned)n0), "l"(a_h), "l"(b_l), "r"(idesc));
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                 ::"r"(tmem + (unsigned)n0), "l"(a_l), "l"(b_h), "r"(idesc));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(bar0 + 8u * st) : "memory");
        }
    }
    {   // the last commit covers every MMA issued before it
        const int kl = NK - 1;
        asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                     "@!d bra WAIT_%=;\n\t}" ::"r"(bar0 + 8u * (kl % nstage)), "r"((unsigned)((kl / nstage) & 1))
                     : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // epilogue: warp w owns accumulator rows (lines) 32w .. 32w+31 = TMEM lanes.  32 lines x 32
    // outputs at a time go through padded shared memory (the A tiles are free now), so each line's
    // outputs leave as one store spanning 256 bytes instead of 32 lines' scattered words.
    const int q4 = warp & 3;                                      // TMEM lane quarter = lines 32 q4 ..
    float *stg = reinterpret_cast<float *>(tsm) + warp * 32 * 33;
    const unsigned trow = tmem + ((unsigned)(q4 * 32) << 16);
    for (int c = 32 * (warp >> 2); c < NH; c += 32 * (TC_THREADS / 128)) {
        float v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                       "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                     : "r"(trow + (unsigned)c));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]),
                       "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
                     : "r"(trow + (unsigned)(c + 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = v[i];
        __syncwarp();
        const int n = c + lane;                                   // output n of this parity: column 2n + par
        for (int r = 0; r < 32; ++r) {
            const int64_t line = line0 + q4 * 32 + r;
            if (line < n_lines && n < nout) p.g4[line * nc + 2 * n + par] = p.sign * stg[r * 33 + lane];
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        unsigned cols = 32;
        while (cols < (unsigned)NH) cols <<= 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
    }
}

// ---------------------------------------------------------------------------
// K3 on the tensor cores with the tap matrix held as Hankel core matrices (default for wide
// detectors).  Per parity the tap matrix is Toeplitz, B[n][k] = T(n - k).  With the K index
// reversed in both operands (k' = NH - 1 - k) it is Hankel, B'[n][k'] = T(n + k' - NH + 1), so
// the canonical K-major core matrix (8 rows n x 4 columns k') at row group ng and K quad kq'
// depends only on s = 2 ng + kq'.  The NH/2 distinct cores are stored consecutively (128 B
// each) and the UMMA descriptor walks them with LBO = 128 B (next K quad = next core) and
// SBO = 256 B (next row group = two cores on): the whole B operand of one parity is 64 NH
// bytes per TF32 half, loaded once per CTA instead of streamed per K chunk.  The A chunks
// (κ-line samples of the parity's inputs, K reversed, split hi/lo) go through an
// nstage-deep ring; one thread issues the 3xTF32 MMAs of a chunk and commits them to the
// stage's mbarrier, so staging chunk kc+1.. overlaps the tensor core on chunk kc.
// ---------------------------------------------------------------------------
// Persistent: 2 CTAs per SM, each fixed to one parity (its taps loaded once), loop over work items
// (128-line block, output half).  nsplit = 2 (NH > 256): an item covers one half of the outputs
// (N = NH/2) so the accumulator fits 256 TMEM columns and two CTAs share an SM (one's staging and
// epilogue overlap the other's MMAs).
constexpr int HK_THREADS = 512;

__device__ __forceinline__ uint64_t hk_desc(unsigned saddr)
{
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           (1ull << 46);
}

__global__ void __launch_bounds__(HK_THREADS, 2) k_hilbert_hk(FilterParams p, int64_t n_lines, int nstage, int nsplit)
{
    extern __shared__ __align__(1024) unsigned char tsm[];
    const int nc = p.nc, NH = hilbert_tc_nh(nc), NK = NH / TC_KC, NS = NH / 2;
    const int NN = NH / nsplit;                                  // outputs of an item: [n_lo, n_lo + NN)
    const int par = blockIdx.x & 1, cta = blockIdx.x >> 1, ncta = gridDim.x >> 1;
    const int nin = (nc - (1 - par) + 1) / 2, nout = (nc - par + 1) / 2;
    const int64_t n_items = (n_lines + TC_M - 1) / TC_M * nsplit;
    unsigned char *Bh = tsm, *Bl = tsm + NS * 128;               // Hankel cores, hi / lo
    unsigned char *A0 = tsm + 2 * NS * 128;
    const unsigned stage_bytes = (unsigned)(2 * TC_M * TC_KC * 4);   // A hi + lo of one K chunk
    // epilogue staging: the A ring (idle between an item's last MMA and the next item's first chunk)
    float *stg_all = reinterpret_cast<float *>(A0);
    __shared__ __align__(8) unsigned long long s_bar[4];
    __shared__ unsigned s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&s_bar[0]);
    unsigned cols = 32;
    while (cols < (unsigned)NN) cols <<= 1;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < nstage; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * i));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {   // the parity's tap cores (hi then lo, 8 float4 per core)
        const float4 *src = reinterpret_cast<const float4 *>(p.hilbert_hk) + (size_t)par * 2 * NS * 8;
        float4 *dst = reinterpret_cast<float4 *>(Bh);
        for (int i = tid; i < 2 * NS * 8; i += HK_THREADS) dst[i] = __ldg(src + i);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    const unsigned idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(TC_M >> 4) << 24);
    const unsigned sBh = (unsigned)__cvta_generic_to_shared(Bh), sBl = (unsigned)__cvta_generic_to_shared(Bl);
    const int rr = lane & 7, kq = lane >> 3;
    // a thread's samples of one A chunk: row warp * 8 + rr, K quads kq and 4 + kq; element (row, j)
    // is input k = NH - 1 - (32 kc + j) of the line
    static_assert(HK_THREADS / 32 == TC_M / 8, "one 8-row group per warp");
    const int row = warp * 8 + rr;
    const int q4 = warp & 3;                                     // epilogue: TMEM lane quarter
    const unsigned trow = tmem + ((unsigned)(q4 * 32) << 16);
    float *stg = stg_all + warp * 32 * 17;
    int g = 0;                                                   // chunks issued by this CTA (ring phase)
    for (int64_t item = cta; item < n_items; item += ncta) {
        const int64_t line0 = item / nsplit * TC_M;
        const int n_lo = (int)(item % nsplit) * NN;
        const int64_t line = line0 + row;
        const float *src = p.g3 + line * nc + (1 - par);
        auto load_chunk = [&](int kc, float (&v)[2][4]) {
#pragma unroll
            for (int qb = 0; qb < 2; ++qb)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int k = NH - 1 - (kc * TC_KC + (qb * 4 + kq) * 4 + i);
                    v[qb][i] = (line < n_lines && k < nin) ? __ldg(src + 2 * k) : 0.f;
                }
        };
        float cur[2][4];
        load_chunk(0, cur);
        for (int kc = 0; kc < NK; ++kc, ++g) {
            const int st = g % nstage;
            float nxt[2][4];                                      // next chunk's loads fly over this one
            if (kc + 1 < NK) load_chunk(kc + 1, nxt);
            if (g >= nstage) {                                    // the MMAs of chunk g - nstage read this stage
                asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                             "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                             "@!d bra WAIT_%=;\n\t}" ::"r"(bar0 + 8u * st), "r"((unsigned)(((g - nstage) / nstage) & 1))
                             : "memory");
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            unsigned char *Ah = A0 + st * stage_bytes, *Al = Ah + TC_M * TC_KC * 4;
#pragma unroll
            for (int qb = 0; qb < 2; ++qb) {
                const float *v = cur[qb];
                const float4 h = make_float4(tf32_hi(v[0]), tf32_hi(v[1]), tf32_hi(v[2]), tf32_hi(v[3]));
                const unsigned o = tc_off(row, (qb * 4 + kq) * 4);
                *reinterpret_cast<float4 *>(Ah + o) = h;
                *reinterpret_cast<float4 *>(Al + o) = make_float4(v[0] - h.x, v[1] - h.y, v[2] - h.z, v[3] - h.w);
            }
#pragma unroll
            for (int qb = 0; qb < 2; ++qb)
#pragma unroll
                for (int i = 0; i < 4; ++i) cur[qb][i] = nxt[qb][i];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned sAh = (unsigned)__cvta_generic_to_shared(Ah), sAl = (unsigned)__cvta_generic_to_shared(Al);
                for (int n0 = n_lo; n0 < n_lo + NN; n0 += 256) {
                    const int nn = n_lo + NN - n0 < 256 ? n_lo + NN - n0 : 256;
                    const unsigned idesc = idesc_base | ((unsigned)(nn >> 3) << 17);
                    const unsigned tcol = tmem + (unsigned)(n0 - n_lo);
#pragma unroll
                    for (int kk = 0; kk < TC_KC / 8; ++kk) {
                        const unsigned core = (unsigned)(2 * (n0 >> 3) + kc * 8 + kk * 2) * 128u;   // s of (n0, k' = 32 kc + 8 kk)
                        const uint64_t a_h = tc_desc(sAh + (unsigned)kk * 256u), a_l = tc_desc(sAl + (unsigned)kk * 256u);
                        const uint64_t b_h = hk_desc(sBh + core), b_l = hk_desc(sBl + core);
                        const unsigned first = (kc == 0 && kk == 0) ? 0u : 1u;
                        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}"
                                     ::"r"(tcol), "l"(a_h), "l"(b_h), "r"(idesc), "r"(first));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                     ::"r"(tcol), "l"(a_h), "l"(b_l), "r"(idesc));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                     ::"r"(tcol), "l"(a_l), "l"(b_h), "r"(idesc));
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(bar0 + 8u * st) : "memory");
            }
        }
        {   // the item's last commit covers every MMA issued before it
            const int gl = g - 1;
            asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                         "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                         "@!d bra WAIT_%=;\n\t}" ::"r"(bar0 + 8u * (gl % nstage)), "r"((unsigned)((gl / nstage) & 1))
                         : "memory");
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        // epilogue: warp w owns accumulator rows (lines) 32 (w & 3) .. = TMEM lane quarter; 32 lines x 16
        // outputs at a time go through padded shared memory
        for (int c = 16 * (warp >> 2); c < NN; c += 16 * (HK_THREADS / 128)) {
            float v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                           "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                         : "r"(trow + (unsigned)c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) stg[lane * 17 + i] = v[i];
            __syncwarp();
            const int cl = lane & 15, rh = lane >> 4;               // half-warps take alternate lines
            const int n = n_lo + c + cl;                            // output n of this parity: column 2n + par
            for (int r = rh; r < 32; r += 2) {
                const int64_t ln = line0 + q4 * 32 + r;
                if (ln < n_lines && n < nout && c + cl < NN) p.g4[ln * nc + 2 * n + par] = p.sign * stg[r * 17 + cl];
            }
            __syncwarp();
        }
        // the next item's first MMA overwrites the accumulator: every warp's reads must be done
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

// ---------------------------------------------------------------------------
// Warp-specialized Hankel-core K3 (default for wide detectors).  One persistent CTA per SM, fixed
// to one parity, walks work items (128-line block, output half with N = NN <= 256):
//   warps 0-7   producers: load an A chunk (128 lines x 32 inputs, K reversed), split hi/lo, store
//               it in the canonical layout into a 4-deep ring, one mbarrier arrive per warp;
//   warp 8      MMA: one thread issues the chunk's 3xTF32 MMAs (B = the resident Hankel cores)
//               into one of two TMEM accumulators and commits the ring slot back to the producers;
//               after an item's last chunk it commits the accumulator to the epilogue;
//   warps 9-12  epilogue: one TMEM lane quarter each, accumulator -> padded smem -> g4, then free
//               the accumulator, while the tensor core already works on the next item.
// ---------------------------------------------------------------------------
// warps 0-7 convert, 8 issues MMAs, 9-12 epilogue, 13 issues the A chunk TMAs
constexpr int WS_PROD = 8, WS_EPI = 4, WS_THREADS = 32 * (WS_PROD + 1 + WS_EPI + 1);
constexpr unsigned WS_RAWB = TC_M * TC_KC * 4;                    // one raw A chunk: 128 lines x 32 inputs
// A tiles of this kernel: K-major core matrices with LBO = 144 B (K quads 9 bank groups apart) and
// SBO = 1152 B, so the 8 K quads of one line a quarter-warp stores hit 8 different 16-B bank groups
constexpr unsigned WS_LBO = 144, WS_SBO = 1152, WS_ATILE = (TC_M / 8) * WS_SBO;
__device__ __forceinline__ unsigned ws_off(int row, int k)
{
    return (unsigned)((row >> 3) * WS_SBO + (k >> 2) * WS_LBO + (row & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t ws_desc(unsigned saddr)
{
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(WS_LBO >> 4) << 16) | ((uint64_t)(WS_SBO >> 4) << 32) |
           (1ull << 46);
}

__device__ __forceinline__ void ws_wait(unsigned bar, unsigned parity)
{
    asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                 "@!d bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void ws_arrive(unsigned bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// (the tensor map is the first parameter: it must sit 64-byte aligned in the parameter space)
// WS_NST converted A stages (hi/lo tiles), WS_RAW raw TMA chunks in flight
template <int WS_NST, int WS_RAW>
__global__ void __launch_bounds__(WS_THREADS, 1) k_hilbert_ws(const __grid_constant__ CUtensorMap amap, FilterParams p,
                                                              int64_t n_lines, int nsplit)
{
    extern __shared__ __align__(1024) unsigned char tsm[];
    const int nc = p.nc, NH = hilbert_tc_nh(nc), NK = NH / TC_KC, NS = NH / 2;
    const int NN = NH / nsplit;
    const int par = blockIdx.x & 1, cta = blockIdx.x >> 1, ncta = gridDim.x >> 1;
    const int nin = (nc - (1 - par) + 1) / 2, nout = (nc - par + 1) / 2;
    const int64_t n_items = (n_lines + TC_M - 1) / TC_M * nsplit;
    unsigned char *Bh = tsm, *Bl = tsm + NS * 128;
    unsigned char *A0 = tsm + 2 * NS * 128;
    constexpr unsigned kStage = 2 * WS_ATILE;
    unsigned char *R0 = A0 + WS_NST * kStage;                    // raw chunks (TMA): [WS_RAW][128][32] floats
    float *stg_all = reinterpret_cast<float *>(R0 + WS_RAW * WS_RAWB);   // epilogue: 4 warps x 32 x 17
    __shared__ __align__(8) unsigned long long s_full[WS_NST], s_empty[WS_NST], s_afull[2], s_aempty[2];
    __shared__ __align__(8) unsigned long long s_rfull[WS_RAW], s_rempty[WS_RAW];
    __shared__ unsigned s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&s_full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&s_empty[0]);
    const unsigned afull0 = (unsigned)__cvta_generic_to_shared(&s_afull[0]);
    const unsigned aempty0 = (unsigned)__cvta_generic_to_shared(&s_aempty[0]);
    const unsigned rfull0 = (unsigned)__cvta_generic_to_shared(&s_rfull[0]);
    const unsigned rempty0 = (unsigned)__cvta_generic_to_shared(&s_rempty[0]);
    if (warp == WS_PROD) {                                       // two accumulators of 256 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < WS_NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(full0 + 8u * i), "r"(WS_PROD));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8u * i));
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(afull0 + 8u * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(aempty0 + 8u * i), "r"(WS_EPI));
        }
        for (int i = 0; i < WS_RAW; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rfull0 + 8u * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rempty0 + 8u * i), "r"(WS_PROD));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {   // the parity's tap cores (hi then lo)
        const float4 *src = reinterpret_cast<const float4 *>(p.hilbert_hk) + (size_t)par * 2 * NS * 8;
        float4 *dst = reinterpret_cast<float4 *>(Bh);
        for (int i = tid; i < 2 * NS * 8; i += WS_THREADS) dst[i] = __ldg(src + i);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;

    if (warp < WS_PROD) {
        // ---- converters: raw chunk (TMA, inputs k = NH - 32 - 32 kc + j ascending in j) -> reversed,
        //      hi/lo-split canonical A tile; thread -> K quad q of the raw row, rows rs + 32 j ----
        const int q = tid & 7, rs = tid >> 3;
        int g = 0;
        for (int64_t item = cta; item < n_items; item += ncta) {
            for (int kc = 0; kc < NK; ++kc, ++g) {
                const int rst = g % WS_RAW, st = g % WS_NST;
                ws_wait(rfull0 + 8u * rst, (unsigned)(g / WS_RAW) & 1u);
                if (g >= WS_NST) ws_wait(empty0 + 8u * st, (unsigned)((g / WS_NST) - 1) & 1u);
                const float *raw = reinterpret_cast<const float *>(R0 + rst * WS_RAWB);
                unsigned char *Ah = A0 + st * kStage, *Al = Ah + WS_ATILE;
                const int k0 = NH - 32 - 32 * kc + 4 * q;            // inputs k0 .. k0 + 3 of this quad
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int row = rs + 32 * j;
                    const float4 r4 = *reinterpret_cast<const float4 *>(raw + row * 32 + 4 * q);
                    // k' order (K reversed): k0 + 3, k0 + 2, k0 + 1, k0; inputs k >= nin are not this parity's
                    const float v0 = k0 + 3 < nin ? r4.w : 0.f, v1 = k0 + 2 < nin ? r4.z : 0.f;
                    const float v2 = k0 + 1 < nin ? r4.y : 0.f, v3 = k0 < nin ? r4.x : 0.f;
                    const float4 h = make_float4(tf32_hi(v0), tf32_hi(v1), tf32_hi(v2), tf32_hi(v3));
                    const unsigned o = ws_off(row, 4 * (7 - q));
                    *reinterpret_cast<float4 *>(Ah + o) = h;
                    *reinterpret_cast<float4 *>(Al + o) = make_float4(v0 - h.x, v1 - h.y, v2 - h.z, v3 - h.w);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
                __syncwarp();
                if (lane == 0) { ws_arrive(rempty0 + 8u * rst); ws_arrive(full0 + 8u * st); }
            }
        }
    } else if (warp == WS_PROD) {
        // ---- MMA issuer ----
        if (lane == 0) {
            const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(TC_M >> 4) << 24) |
                                   ((unsigned)(NN >> 3) << 17);
            const unsigned sBh = (unsigned)__cvta_generic_to_shared(Bh), sBl = (unsigned)__cvta_generic_to_shared(Bl);
            int g = 0, it = 0;
            for (int64_t item = cta; item < n_items; item += ncta, ++it) {
                const int acc = it & 1;
                const int n_lo = (int)(item % nsplit) * NN;
                if (it >= 2) ws_wait(aempty0 + 8u * acc, (unsigned)((it >> 1) - 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned tcol = tmem + (unsigned)(acc * 256);
                for (int kc = 0; kc < NK; ++kc, ++g) {
                    const int st = g % WS_NST;
                    ws_wait(full0 + 8u * st, (unsigned)(g / WS_NST) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned sAh = (unsigned)__cvta_generic_to_shared(A0 + st * kStage);
                    const unsigned sAl = sAh + WS_ATILE;
#pragma unroll
                    for (int kk = 0; kk < TC_KC / 8; ++kk) {
                        const unsigned core = (unsigned)(2 * (n_lo >> 3) + kc * 8 + kk * 2) * 128u;
                        const uint64_t a_h = ws_desc(sAh + (unsigned)kk * 2u * WS_LBO), a_l = ws_desc(sAl + (unsigned)kk * 2u * WS_LBO);
                        const uint64_t b_h = hk_desc(sBh + core), b_l = hk_desc(sBl + core);
                        const unsigned first = (kc == 0 && kk == 0) ? 0u : 1u;
                        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}"
                                     ::"r"(tcol), "l"(a_h), "l"(b_h), "r"(idesc), "r"(first));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                     ::"r"(tcol), "l"(a_h), "l"(b_l), "r"(idesc));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                                     ::"r"(tcol), "l"(a_l), "l"(b_h), "r"(idesc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 ::"r"(empty0 + 8u * st) : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             ::"r"(afull0 + 8u * acc) : "memory");
            }
        }
        __syncwarp();
    } else if (warp == WS_PROD + 1 + WS_EPI) {
        // ---- A chunk TMA issuer: box of 32 inputs x 128 lines of the parity's half-lines ----
        if (lane == 0) {
            const int colbase = (1 - par) * p.hp + NH - 32;
            int g = 0;
            for (int64_t item = cta; item < n_items; item += ncta) {
                const int line0 = (int)(item / nsplit * TC_M);
                for (int kc = 0; kc < NK; ++kc, ++g) {
                    const int rst = g % WS_RAW;
                    if (g >= WS_RAW) ws_wait(rempty0 + 8u * rst, (unsigned)((g / WS_RAW) - 1) & 1u);
                    const unsigned full = rfull0 + 8u * rst;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(WS_RAWB) : "memory");
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                                 ::"r"((unsigned)__cvta_generic_to_shared(R0 + rst * WS_RAWB)),
                                   "l"(reinterpret_cast<uint64_t>(&amap)), "r"(colbase - 32 * kc), "r"(line0), "r"(full)
                                 : "memory");
                }
            }
        }
        __syncwarp();
    } else {
        // ---- epilogue: TMEM lane quarter q4 = lines 32 q4 .. of the item ----
        const int ew = warp - WS_PROD - 1, q4 = warp & 3;
        float *stg = stg_all + ew * 32 * 17;
        int it = 0;
        for (int64_t item = cta; item < n_items; item += ncta, ++it) {
            const int acc = it & 1;
            const int64_t line0 = item / nsplit * TC_M;
            const int n_lo = (int)(item % nsplit) * NN;
            ws_wait(afull0 + 8u * acc, (unsigned)(it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned trow = tmem + ((unsigned)(q4 * 32) << 16) + (unsigned)(acc * 256);
            for (int c = 0; c < NN; c += 16) {
                float v[16];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                               "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                             : "r"(trow + (unsigned)c));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; ++i) stg[lane * 17 + i] = v[i];
                __syncwarp();
                const int cl = lane & 15, rh = lane >> 4;
                const int n = n_lo + c + cl;
                for (int r = rh; r < 32; r += 2) {
                    const int64_t ln = line0 + q4 * 32 + r;
                    if (ln < n_lines && n < nout && c + cl < NN) p.g4[ln * nc + 2 * n + par] = p.sign * stg[r * 17 + cl];
                }
                __syncwarp();
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) ws_arrive(aempty0 + 8u * acc);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == WS_PROD) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

// Both parities per CTA (NH <= 256: two accumulators fit TMEM's 512 columns).
// A K chunk covers inputs l in [64 kc, 64 kc + 64) of each line (coalesced
// loads), de-interleaved into the even- and odd-input tiles; output parity 0
// takes the odd inputs, parity 1 the even ones.  The epilogue stages 32 lines x
// 32 outputs per warp in padded shared memory so every line is written as
// contiguous 128-byte runs.
__global__ void __launch_bounds__(TC2_THREADS, 1) k_hilbert_tc2(FilterParams p, int64_t n_lines)
{
    extern __shared__ __align__(1024) unsigned char tsm[];
    const int nc = p.nc, NH = hilbert_tc_nh(nc), NK = NH / TC_KC;
    const int64_t line0 = (int64_t)blockIdx.x * TC_M;
    constexpr int AT = TC_M * TC_KC * 4;                         // one A tile (16 KB)
    unsigned char *Aeh = tsm, *Ael = tsm + AT, *Aoh = tsm + 2 * AT, *Aol = tsm + 3 * AT;
    unsigned char *B = tsm + 4 * AT;                             // [par][hi, lo][NH x 32]
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar);
    unsigned cols = 32;
    while (cols < 2u * (unsigned)NH) cols <<= 1;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(&s_tmem)), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NH >> 3) << 17) | ((unsigned)(TC_M >> 4) << 24);
    const unsigned sA[4] = {(unsigned)__cvta_generic_to_shared(Aeh), (unsigned)__cvta_generic_to_shared(Ael),
                            (unsigned)__cvta_generic_to_shared(Aoh), (unsigned)__cvta_generic_to_shared(Aol)};
    const unsigned sB = (unsigned)__cvta_generic_to_shared(B);
    const unsigned bt = (unsigned)NH * TC_KC * 4;                 // one B tile

    for (int kc = 0; kc < NK; ++kc) {
        // A: lane = (row in an 8-row group, k quad); 8 consecutive inputs per lane = 4 (even, odd) pairs
        const int rr = lane & 7, kq = lane >> 3;
        for (int g = warp; g < TC_M / 8; g += TC2_THREADS / 32) {
            const int row = g * 8 + rr;
            const int64_t line = line0 + row;
            const float *src = p.g3 + line * nc;
            const bool ok = line < n_lines;
#pragma unroll
            for (int qb = 0; qb < 2; ++qb) {
                const int kl = (qb * 4 + kq) * 4;                   // k within the chunk
                const int l0 = 2 * (kc * TC_KC + kl);               // first input column
                float e[4], o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    e[i] = (ok && l0 + 2 * i < nc) ? __ldg(src + l0 + 2 * i) : 0.f;
                    o[i] = (ok && l0 + 2 * i + 1 < nc) ? __ldg(src + l0 + 2 * i + 1) : 0.f;
                }
                const unsigned off = tc_off(row, kl);
                const float4 eh = make_float4(tf32_hi(e[0]), tf32_hi(e[1]), tf32_hi(e[2]), tf32_hi(e[3]));
                const float4 oh = make_float4(tf32_hi(o[0]), tf32_hi(o[1]), tf32_hi(o[2]), tf32_hi(o[3]));
                *reinterpret_cast<float4 *>(Aeh + off) = eh;
                *reinterpret_cast<float4 *>(Ael + off) = make_float4(e[0] - eh.x, e[1] - eh.y, e[2] - eh.z, e[3] - eh.w);
                *reinterpret_cast<float4 *>(Aoh + off) = oh;
                *reinterpret_cast<float4 *>(Aol + off) = make_float4(o[0] - oh.x, o[1] - oh.y, o[2] - oh.z, o[3] - oh.w);
            }
        }
        // B chunk kc of both parities (hi, lo each), canonical layout in the plan table
        const float4 *tab = reinterpret_cast<const float4 *>(p.hilbert_tc);
        for (int par = 0; par < 2; ++par) {
            const float4 *bsrc = tab + (((size_t)par * NK + kc) * 2) * NH * TC_KC / 4;
            float4 *bdst = reinterpret_cast<float4 *>(B + (size_t)par * 2 * bt);
            for (int i = tid; i < 2 * NH * TC_KC / 4; i += TC2_THREADS) bdst[i] = __ldg(bsrc + i);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int par = 0; par < 2; ++par) {
                const unsigned ah = sA[par == 0 ? 2 : 0], al = sA[par == 0 ? 3 : 1];   // parity 0 <- odd inputs
                const unsigned bh = sB + (unsigned)par * 2u * bt, bl = bh + bt;
                const unsigned d = tmem + (unsigned)(par * NH);
#pragma unroll
                for (int kk = 0; kk < TC_KC / 8; ++kk) {
                    const unsigned ko = (unsigned)kk * 256u;
                    const uint64_t a_h = tc_desc(ah + ko), a_l = tc_desc(al + ko);
                    const uint64_t b_h = tc_desc(bh + ko), b_l = tc_desc(bl + ko);
                    const unsigned acc = (kc == 0 && kk == 0) ? 0u : 1u;
                    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}"
                                 ::"r"(d), "l"(a_h), "l"(b_h), "r"(idesc), "r"(acc));
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a_h),
                                 "l"(b_l), "r"(idesc));
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a_l),
                                 "l"(b_h), "r"(idesc));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                         : "memory");
        }
        asm volatile("{\n\t.reg .pred d;\n\tWAIT_%=:\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t"
                     "@!d bra WAIT_%=;\n\t}" ::"r"(bar), "r"((unsigned)(kc & 1)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // epilogue: per warp, 32 lines (its TMEM lanes) x 32 output columns at a time through smem
    const int q4 = warp & 3;                                      // TMEM lane quarter = lines 32 q4 ..
    float *stg = reinterpret_cast<float *>(tsm) + warp * 32 * 33;
    const unsigned trow = tmem + ((unsigned)(q4 * 32) << 16);
    for (int c = 16 * (warp >> 2); c < NH; c += 16 * (TC2_THREADS / 128)) {
        float v0[16], v1[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=f"(v0[0]), "=f"(v0[1]), "=f"(v0[2]), "=f"(v0[3]), "=f"(v0[4]), "=f"(v0[5]), "=f"(v0[6]), "=f"(v0[7]),
                       "=f"(v0[8]), "=f"(v0[9]), "=f"(v0[10]), "=f"(v0[11]), "=f"(v0[12]), "=f"(v0[13]), "=f"(v0[14]), "=f"(v0[15])
                     : "r"(trow + (unsigned)c));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=f"(v1[0]), "=f"(v1[1]), "=f"(v1[2]), "=f"(v1[3]), "=f"(v1[4]), "=f"(v1[5]), "=f"(v1[6]), "=f"(v1[7]),
                       "=f"(v1[8]), "=f"(v1[9]), "=f"(v1[10]), "=f"(v1[11]), "=f"(v1[12]), "=f"(v1[13]), "=f"(v1[14]), "=f"(v1[15])
                     : "r"(trow + (unsigned)(NH + c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // lane = line; output columns 2c .. 2c+31 (parity 0 at even, parity 1 at odd)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            stg[lane * 33 + 2 * i] = v0[i];
            stg[lane * 33 + 2 * i + 1] = v1[i];
        }
        __syncwarp();
        const int l = 2 * c + lane;
        for (int r = 0; r < 32; ++r) {
            const int64_t line = line0 + q4 * 32 + r;
            if (line < n_lines && l < nc) p.g4[line * nc + l] = p.sign * stg[r * 33 + lane];
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

// ---------------------------------------------------------------------------
// K4: gF[v][m][l] = cos α_l · lerp_ψ(g4[v][·][l], ψ̂(α_l, w_m))   (Eqs. 13-15)
//
// Output for the backprojection: per view, column-major 2x2 tap quads in
// sum/difference form
//   Q[v][l][r] = (s_0 - ρ d_0, s_1 - ρ d_1, d_0, d_1),   ρ = r - c,  c = (nr + 2) / 2,
//   s_j = ½(g[m][l+j] + g[m+1][l+j]),  d_j = g[m+1][l+j] - g[m][l+j],  m = r - 2,
// r = 0 .. nr+1 (two zero rows below the detector; taps beyond the last row or
// column are 0).  With the centred quad-row position P = (m + f) + 1.5 - c of a
// sample at (l + fa, m + f) and r = round(P + c), the bilinear sample is
//   w0 (Q.x + P Q.z) + w1 (Q.y + P Q.w),   w0 = 1 - fa, w1 = fa,
// i.e. one 128-bit load and two paired FMAs (FFMA2) in the BP, no fraction.
// Optionally also the plain gF (debug / parity entry point).
// One CTA per (view, 32-column block): the block's (nr + 3) x 33 gF values are
// formed in shared memory, then written as contiguous quad columns.
// ---------------------------------------------------------------------------
constexpr int K4_COLS = 32;

// VPB views per CTA (grid.y = ceil(n_views / VPB)): the view-independent rebin entry and cos α_l
// are loaded once per (row, column) and the VPB views' g4 gathers are issued back to back.
template <int VPB>
__global__ void __launch_bounds__(256) k_bwd_rebin_cos(FilterParams p)
{
    extern __shared__ float tile[];            // [VPB][nr + 3][K4_COLS + 1], rows m = -2 .. nr
    const int nc = p.nc, nr = p.nr, nq = nr + 2;
    const int l0 = blockIdx.x * K4_COLS;
    const int v0 = blockIdx.y * VPB;
    const int nv = min(VPB, p.n_views - v0);
    const int cols = min(K4_COLS, nc - l0);
    const int ld = K4_COLS + 1, tsz = (nr + 3) * ld;
    for (int e = threadIdx.x; e < tsz; e += blockDim.x) {
        const int mm = e / ld, ll = e - mm * ld, m = mm - 2, l = l0 + ll;
        float out[VPB];
#pragma unroll
        for (int j = 0; j < VPB; ++j) out[j] = 0.f;
        if (m >= 0 && m < nr && l < nc && ll <= cols) {
            const RebinEntry r = p.br[m * nc + l];
            if (r.idx >= 0) {
                const float ca = __ldg(p.cos_alpha + l);
                const float *g = p.g4 + ((size_t)v0 * p.npsi + r.idx) * nc + l;
                const size_t vs = (size_t)p.npsi * nc;
                float a[VPB], b[VPB];
#pragma unroll
                for (int j = 0; j < VPB; ++j)
                    if (j < nv) { a[j] = g[j * vs]; b[j] = g[j * vs + nc]; }
#pragma unroll
                for (int j = 0; j < VPB; ++j)
                    if (j < nv) out[j] = ca * fmaf(r.frac, b[j] - a[j], a[j]);
            }
            if (p.gF && ll < cols)
#pragma unroll
                for (int j = 0; j < VPB; ++j)
                    if (j < nv) p.gF[((size_t)(v0 + j) * nr + m) * nc + l] = out[j];
        }
#pragma unroll
        for (int j = 0; j < VPB; ++j) tile[j * tsz + e] = out[j];
    }
    __syncthreads();
    const int per = cols * nq;
    for (int e = threadIdx.x; e < nv * per; e += blockDim.x) {
        const int j = e / per, e1 = e - j * per;
        const int ll = e1 / nq, r = e1 - ll * nq;       // r = quad row; taps rows r-2, r-1
        const float *t0 = tile + j * tsz + r * ld + ll;
        const float a0 = t0[0], a1 = t0[1], c0 = t0[ld], c1 = t0[ld + 1];
        const float rc = (float)(r - (nr + 2) / 2);      // centred quad row
        p.gq[((size_t)(v0 + j) * nc + l0) * nq + e1] =
            make_float4(fmaf(-rc, c0 - a0, 0.5f * (a0 + c0)), fmaf(-rc, c1 - a1, 0.5f * (a1 + c1)), c0 - a0, c1 - a1);
    }
}


// Row form (default): a CTA = 256 threads on one 32-column block and a run of view groups of VPB
// views.  A thread owns the same (row, column) entries of the [nr + 3][33] g5·cos α tile in every
// group (rows m = -2 .. nr, columns c0 .. c0+32; index advanced incrementally, no division), so their
// rebin entries and cos α stay in registers for the whole run; the g4 gathers of group i+1 are
// issued before group i's quads are written.  Phase 2 writes the block's quads in their global order
// (column-major, rows contiguous).  Same fp32 arithmetic as k_bwd_rebin_cos.
// K4R_E: tile entries per thread, (nr + 3) * 33 <= 256 * K4R_E (4: nr <= 28, 9: nr <= 66)
template <int VPB, int K4R_E>
__global__ void __launch_bounds__(256) k_bwd_rebin_cos_rows(FilterParams p, int ngroups)
{
    extern __shared__ float tile[];            // [2][VPB][nr + 3][33], rows m = -2 .. nr
    const int nc = p.nc, nr = p.nr, nq = nr + 2, ld = K4_COLS + 1, tsz = (nr + 3) * ld;
    const int tid = threadIdx.x;
    const int l0 = blockIdx.x * K4_COLS;
    const int cols = min(K4_COLS, nc - l0);
    const size_t vs = (size_t)p.npsi * nc;
    // this thread's tile entries e = tid + 256 i: rebin entry (idx < 0: zero), cos α, column
    int eidx[K4R_E], eoff[K4R_E];
    float efr[K4R_E], eca[K4R_E];
    {
        int mm = tid / ld, ll = tid - mm * ld;
        const int DM = 256 / ld, DL = 256 - DM * ld;
#pragma unroll
        for (int i = 0; i < K4R_E; ++i) {
            const int m = mm - 2, l = l0 + ll;
            eidx[i] = -1; efr[i] = 0.f; eca[i] = 0.f; eoff[i] = mm * ld + ll;
            if (mm >= nr + 3) eoff[i] = -1;
            else if (m >= 0 && m < nr && l < nc) {
                const RebinEntry r = p.br[m * nc + l];
                eidx[i] = r.idx;
                efr[i] = r.frac;
                eca[i] = __ldg(p.cos_alpha + l);
            }
            mm += DM; ll += DL;
            if (ll >= ld) { ll -= ld; ++mm; }
        }
    }
    const int ll0 = tid / nq, r0 = tid - ll0 * nq, DL2 = 256 / nq, DR2 = 256 - DL2 * nq;
    const float rcen = (float)((nr + 2) / 2);
    const int per = cols * nq;
    float ga[K4R_E][VPB], gb[K4R_E][VPB];
    auto gather = [&](int grp) {
        const int v0 = (blockIdx.y * ngroups + grp) * VPB;
#pragma unroll
        for (int i = 0; i < K4R_E; ++i)
            if (eidx[i] >= 0) {
                const float *g = p.g4 + ((size_t)v0 * p.npsi + eidx[i]) * nc + l0 + (eoff[i] % ld);
#pragma unroll
                for (int j = 0; j < VPB; ++j)
                    if (v0 + j < p.n_views) { ga[i][j] = g[j * vs]; gb[i][j] = g[j * vs + nc]; }
            }
    };
    const int g_end = min(ngroups, (p.n_views - blockIdx.y * ngroups * VPB + VPB - 1) / VPB);
    if (g_end > 0) gather(0);
    for (int grp = 0; grp < g_end; ++grp) {
        const int v0 = (blockIdx.y * ngroups + grp) * VPB;
        const int nv = min(VPB, p.n_views - v0);
        float *tb = tile + (grp & 1) * VPB * tsz;
#pragma unroll
        for (int i = 0; i < K4R_E; ++i) {
            if (eoff[i] < 0) continue;
#pragma unroll
            for (int j = 0; j < VPB; ++j) {
                const float out = eidx[i] >= 0 && j < nv ? eca[i] * fmaf(efr[i], gb[i][j] - ga[i][j], ga[i][j]) : 0.f;
                tb[j * tsz + eoff[i]] = out;
                if (p.gF && j < nv) {                                   // debug path only
                    const int mm = eoff[i] / ld, ll = eoff[i] - mm * ld;
                    if (mm >= 2 && mm < nr + 2 && ll < cols) p.gF[((size_t)(v0 + j) * nr + mm - 2) * nc + l0 + ll] = out;
                }
            }
        }
        if (grp + 1 < g_end) gather(grp + 1);                    // in flight through the quads below
        __syncthreads();
        for (int j = 0; j < nv; ++j) {
            float4 *dst = p.gq + ((size_t)(v0 + j) * nc + l0) * nq;
            const float *tj = tb + j * tsz;
            int ll = ll0, r = r0;
            for (int e = tid; e < per; e += 256) {
                const float *t0 = tj + r * ld + ll;       // r = quad row; taps rows r-2, r-1
                const float a0 = t0[0], a1 = t0[1], c0 = t0[ld], c1 = t0[ld + 1];
                const float rc = (float)r - rcen;         // centred quad row
                dst[e] = make_float4(fmaf(-rc, c0 - a0, 0.5f * (a0 + c0)), fmaf(-rc, c1 - a1, 0.5f * (a1 + c1)),
                                     c0 - a0, c1 - a1);
                ll += DL2;
                r += DR2;
                if (r >= nq) { r -= nq; ++ll; }
            }
        }
        // (group grp+2 rewrites this tile buffer only after every thread passed group grp+1's barrier)
    }
}

void launch_deriv_fwd_rebin(const FilterParams &p, cudaStream_t s)
{
    // column walk, 8 κ-lines per thread (two-row g2 cache; measured best on every config: C4 1.69 ->
    // 1.42 ms vs the per-sample kernel, C3 0.67 -> 0.65, C5 0.72 -> 0.71 vs 32-line segments);
    // KATS_K12=sample: one thread per sample (8 κ-lines unrolled); colN: N κ-lines per thread
    if (p.flat) {                                               // flat detector (A27): its own K12
        const int bx = std::min(256, (p.nc + 31) / 32 * 32);
        k_deriv_fwd_rebin_flat<<<dim3((p.nc + bx - 1) / bx, (p.npsi + kPsiPerFlat - 1) / kPsiPerFlat, p.n_views), bx, 0,
                                 s>>>(p);
        return;
    }
    const char *ke = std::getenv("KATS_K12");
    const std::string k12 = ke ? ke : "";
    const size_t wv_smem = sizeof(float) * (2 * (size_t)p.npsi * 32 + 8 * (size_t)p.nr * 32);
    // default: warp per view for detectors of <= 32 rows, the row form above (scripts/ab/gpu_k12wv.sh,
    // steps: C5 4.08 (round-1 column walk) / 4.32 (rows) / 3.95 ms (wv), C2 1.70 / 1.68 / 1.68,
    // C3 9.13 / 9.01 / 9.23, C4 50.84 / 50.57 / 50.58)
    const bool want_wv = k12 == "wv" || (k12.empty() && p.nr <= 32);
    if (p.half || (want_wv && wv_smem <= 200 * 1024)) {
        // warp per view (the half-sample derivative has only this form): views per warp as many as
        // keep >= 4 CTAs per SM, at most 8
        const int nb = (p.nc + 31) / 32;
        int vpw = 8;
        while (vpw > 1 && (int64_t)nb * ((p.n_views + 8 * vpw - 1) / (8 * vpw)) < 4 * device_sms()) vpw /= 2;
        if (const char *e = std::getenv("KATS_K12WV_VPW")) vpw = std::max(1, std::atoi(e));     // A/B
        const dim3 grid(nb, (p.n_views + 8 * vpw - 1) / (8 * vpw));
        if (p.half) {
            smem_opt_in((const void *)k_deriv_fwd_rebin_wv<true>, wv_smem);
            k_deriv_fwd_rebin_wv<true><<<grid, 256, wv_smem, s>>>(p, vpw);
        } else {
            // KATS_K12WV_UR=8|16 (A/B): deeper unroll of the g2 row loop (more raw loads in flight)
            const char *ue = std::getenv("KATS_K12WV_UR");
            const int ur = ue ? std::atoi(ue) : 4;
            auto go = [&](auto kern) {
                smem_opt_in((const void *)kern, wv_smem);
                kern<<<grid, 256, wv_smem, s>>>(p, vpw);
            };
            if (ur == 16) go(k_deriv_fwd_rebin_wv<false, 16>);
            else if (ur == 8) go(k_deriv_fwd_rebin_wv<false, 8>);
            else go(k_deriv_fwd_rebin_wv<false, 4>);
        }
        return;
    }
    if ((k12.empty() || k12 == "rows") && p.nr <= K12R_WARPS * K12R_MAXR) {
        // views per CTA: as many as keep >= 4 CTAs per SM in the launch (the block's rebin entries are
        // staged once per CTA), at most 16
        const int nb = (p.nc + 31) / 32;
        int nvb = 16;
        while (nvb > 1 && (int64_t)nb * ((p.n_views + nvb - 1) / nvb) < 4 * device_sms()) nvb /= 2;
        if (const char *e = std::getenv("KATS_K12R_NVB")) nvb = std::max(1, std::atoi(e));     // A/B
        const size_t smem = sizeof(float) * (2 * (size_t)p.npsi * 32 + 2 * (size_t)p.nr * 32);
        if (smem <= 200 * 1024) {
            // three CTAs per SM (80 registers, no spills): C3 K12 0.402 -> 0.332 ms (0.43 -> 0.52 of
            // HBM), C4 0.665 -> 0.564 ms; four (64 registers, a small spill) is slower: C3 0.482,
            // C4 0.789 ms (scripts/ab/gpu_r02n.sh; KATS_K12R_MINB=2|3|4)
            int minb = 3;
            if (const char *e = std::getenv("KATS_K12R_MINB")) minb = std::atoi(e);
            const dim3 g(nb, (p.n_views + nvb - 1) / nvb);
            auto go = [&](auto kern) {
                smem_opt_in((const void *)kern, smem);
                kern<<<g, 32 * K12R_WARPS, smem, s>>>(p, nvb);
            };
            if (minb == 4) go(k_deriv_fwd_rebin_rows<4>);
            else if (minb == 3) go(k_deriv_fwd_rebin_rows<3>);
            else go(k_deriv_fwd_rebin_rows<2>);
            return;
        }
    }
    if (k12 == "sample") {
        const int bx = std::min(256, (p.nc + 31) / 32 * 32);
        k_deriv_fwd_rebin<<<dim3((p.nc + bx - 1) / bx, (p.npsi + kPsiPer - 1) / kPsiPer, p.n_views), bx, 0, s>>>(p);
        return;
    }
    const size_t plane = (size_t)p.nr * K12_TL * sizeof(float);
    if (k12 == "tile" && plane + (size_t)K12_TL * sizeof(float) <= 48 * 1024) {
        k_deriv_fwd_rebin_tile<<<dim3((p.nc + K12_TL - 1) / K12_TL, p.n_views), K12_THREADS, plane + K12_TL * sizeof(float), s>>>(p);
        return;
    }
    // round-1 default: the column walk over two views per thread (scripts/ab/gpu_k12v.sh: C5 4.29 ->
    // 4.22 ms, C3 9.30 -> 9.27, C2 / C4 unchanged; colv4 no better); "col8" = one view per thread
    if (k12.empty() || k12 == "rows" || k12 == "colv2" || k12 == "colv4") {
        if (k12 != "colv4") k_deriv_fwd_rebin_colv<2><<<dim3((p.nc + 127) / 128, (p.n_views + 1) / 2, (p.npsi + 7) / 8), 128, 0, s>>>(p, 8);
        else k_deriv_fwd_rebin_colv<4><<<dim3((p.nc + 127) / 128, (p.n_views + 3) / 4, (p.npsi + 7) / 8), 128, 0, s>>>(p, 8);
        return;
    }
    const int seg = k12.rfind("col", 0) == 0 && std::atoi(k12.c_str() + 3) > 0 ? std::atoi(k12.c_str() + 3) : 8;
    k_deriv_fwd_rebin_col<<<dim3((p.nc + 127) / 128, p.n_views, (p.npsi + seg - 1) / seg), 128, 0, s>>>(p, seg);
}

size_t hilbert_tc_table_floats(int nc) { return 2 * 2 * (size_t)hilbert_tc_nh(nc) * hilbert_tc_nh(nc); }

// [par][kc][hi, lo][NH x 32 canonical K-major] (see k_hilbert_tc)
void hilbert_tc_table(int nc, const float *kd, std::vector<float> &out)
{
    const int NH = hilbert_tc_nh(nc), NK = NH / TC_KC;
    out.assign(hilbert_tc_table_floats(nc), 0.f);
    for (int par = 0; par < 2; ++par) {
        const int nin = (nc - (1 - par) + 1) / 2, nout = (nc - par + 1) / 2;
        for (int kc = 0; kc < NK; ++kc)
            for (int n = 0; n < NH; ++n)
                for (int kl = 0; kl < TC_KC; ++kl) {
                    const int k = kc * TC_KC + kl;
                    float b = 0.f;
                    if (n < nout && k < nin) b = kd[2 * (n - k) + 2 * par - 1 + nc - 1];
                    uint32_t u;
                    std::memcpy(&u, &b, 4);
                    u &= 0xFFFFE000u;
                    float hi;
                    std::memcpy(&hi, &u, 4);
                    const size_t off = (size_t)((n >> 3) * 1024 + (kl >> 2) * 128 + (n & 7) * 16 + (kl & 3) * 4) / 4;
                    const size_t blk = (((size_t)par * NK + kc) * 2) * NH * TC_KC;
                    out[blk + off] = hi;
                    out[blk + (size_t)NH * TC_KC + off] = b - hi;
                }
    }
}

size_t hilbert_hk_table_floats(int nc) { return 2 * 2 * (size_t)(hilbert_tc_nh(nc) / 2) * 32; }

// [par][hi, lo][NH/2 Hankel cores][8 rows x 4] (see k_hilbert_hk): core s, row r, column c holds
// the tap of n - k = 4 s + r + c - (NH - 1), i.e. K[2 (n - k) + 2 par - 1] (0 outside the kernel)
void hilbert_hk_table(int nc, const float *kd, std::vector<float> &out)
{
    const int NH = hilbert_tc_nh(nc), NS = NH / 2;
    out.assign(hilbert_hk_table_floats(nc), 0.f);
    for (int par = 0; par < 2; ++par)
        for (int sc = 0; sc < NS; ++sc)
            for (int r = 0; r < 8; ++r)
                for (int c = 0; c < 4; ++c) {
                    const int d = 4 * sc + r + c - (NH - 1);
                    const int t = 2 * d + 2 * par - 1;
                    const float b = (t >= -(nc - 1) && t <= nc - 1) ? kd[t + nc - 1] : 0.f;
                    uint32_t u;
                    std::memcpy(&u, &b, 4);
                    u &= 0xFFFFE000u;
                    float hi;
                    std::memcpy(&hi, &u, 4);
                    const size_t o = (size_t)sc * 32 + r * 4 + c;
                    out[((size_t)par * 2 + 0) * NS * 32 + o] = hi;
                    out[((size_t)par * 2 + 1) * NS * 32 + o] = b - hi;
                }
}

bool hilbert_tc_usable(const FilterParams &p)
{
    const char *e = std::getenv("KATS_HILBERT");
    if (e && std::string(e) == "fp32") return false;
    return p.hilbert_tc != nullptr && hilbert_tc_nh(p.nc) <= 512;
}

// The warp-specialized Hankel kernel (wide detectors, or KATS_HILBERT=ws) reads parity-split input
// lines; the filter drivers ask here before the input's writer (K12 / K4^T) runs and set
// k3_in_split, which launch_hilbert then follows.
bool hilbert_split_input(const FilterParams &p)
{
    if (!hilbert_tc_usable(p) || p.hilbert_overlap || !p.hilbert_hk) return false;
    const char *he = std::getenv("KATS_HILBERT");
    const std::string h = he ? he : "";
    if (h == "tc" || h == "hk" || h == "hk1" || h == "tc2") return false;
    // round 2 (scripts/ab/gpu_k3ws.sh, K3 isolated / step): also the narrow detectors — C4 (NH 96)
    // 1.09 -> 0.87 ms / 50.8 -> 50.2 ms, C2 (NH 192) 1.678 -> 1.664 ms; at NH 64 (C1) the Hankel
    // kernel is faster (step 0.129 tc2 / 0.135 ws / 0.122 ms hk)
    return hilbert_tc_nh(p.nc) > 64 || h == "ws";
}

int launch_hilbert(const FilterParams &p, cudaStream_t s)
{
    if (hilbert_tc_usable(p) && p.hilbert_overlap) {
        // next to the TMEM backprojection (3 CTAs x 128 columns, 62K registers per SM) a tensor-core
        // Hilbert CTA waits for TMEM / registers; the fp32 direct convolution fits beside it
        // (C4 host path 59.4 -> 56.5 ms)
        FilterParams q = p;
        q.hilbert_tc = nullptr;
        return launch_hilbert(q, s);
    }
    // KATS_HILBERT=tc: the per-chunk tap-streaming kernels (A/B tests); =hk: Hankel cores for every width
    const char *he = std::getenv("KATS_HILBERT");
    const bool force_tc = he && (std::string(he) == "tc" || std::string(he) == "tc2"),
               force_hk = he && (std::string(he) == "hk" || std::string(he) == "hk1" || std::string(he) == "ws");
    if (p.k3_in_split || (hilbert_tc_usable(p) && p.hilbert_hk && !force_tc && (hilbert_tc_nh(p.nc) > 32 || force_hk))) {
        const int NH = hilbert_tc_nh(p.nc);
        // halves only where 2 CTAs per SM pay for reading A twice (C3 NH 384: 1.20 -> 1.13 ms;
        // C5 NH 320: 1.32 -> 1.59 ms, measured)
        int nsplit = NH > 352 ? 2 : 1;
        if (const char *e = std::getenv("KATS_HILBERT_SPLIT")) nsplit = std::atoi(e) == 1 || NH % 64 ? 1 : 2;
        const size_t taps = (size_t)128 * NH, stage = (size_t)2 * TC_M * TC_KC * 4;
        // as many A stages (2..4) as leave room for two CTAs per SM (the epilogue reuses the ring:
        // 16 warps x 32 x 17 floats <= 2 stages)
        int nstage = 4;
        while (nstage > 2 && taps + nstage * stage > 110 * 1024) --nstage;
        const size_t smem = taps + nstage * stage;
        smem_opt_in((const void *)k_hilbert_hk, 225 * 1024);
        const int64_t n_lines = (int64_t)p.n_views * p.npsi;
        // warp-specialized for wide detectors (hilbert_split_input: its input lines are parity-split);
        // at NH <= 256 the two-CTA persistent kernel is faster (C2 0.18 vs 0.21 ms)
        const bool ws = p.k3_in_split != 0;
        if (ws) {
            int ns = NH > 256 ? 2 : 1;                                // accumulators of <= 256 columns, two of them
            if (const char *e = std::getenv("KATS_HILBERT_WSSPLIT")) {   // A/B: output parts per item
                const int v = std::atoi(e);
                if (v >= 1 && NH % (16 * v) == 0 && NH / v <= 256) ns = v;
            }
            // converted A stages / raw chunks: 2 / 4 (KATS_WS_STAGES=3: three A stages, with four raw chunks where
            // shared memory allows, else three)
            auto wsm_of = [&](int nst, int raw) {
                return taps + (size_t)nst * 2 * WS_ATILE + (size_t)raw * WS_RAWB + (size_t)WS_EPI * 32 * 17 * 4;
            };
            int nst = 2, nraw = 4;
            if (const char *e = std::getenv("KATS_WS_STAGES"))
                if (std::atoi(e) == 3) { nst = 3; nraw = wsm_of(3, 4) <= 225 * 1024 ? 4 : 3; }
            if (wsm_of(nst, nraw) > 225 * 1024) { nst = 2; nraw = 4; }
            // KATS_WS_RAW=6|8 (A/B): more raw TMA chunks in flight with two A stages, where they fit
            if (const char *e = std::getenv("KATS_WS_RAW")) {
                const int r = std::atoi(e);
                if (nst == 2 && (r == 6 || r == 8) && wsm_of(2, r) <= 225 * 1024) nraw = r;
                else if (nst == 2 && r == 8 && wsm_of(2, 6) <= 225 * 1024) nraw = 6;
            }
            const size_t wsm = wsm_of(nst, nraw);
            CUtensorMap amap;                                         // the K3 input: [n_lines][2 hp] fp32
            if (!make_tensor_map_2d_f32(&amap, p.g3, (uint64_t)2 * p.hp, (uint64_t)n_lines, (uint64_t)8 * p.hp, 32, TC_M)) {
                // cannot happen on a driver that has cuTensorMapEncodeTiled (16-B aligned scratch lines);
                // nothing else reads parity-split lines: the caller turns this into KATS_ERR_CUDA
                return -1;
            }
            int nsm2 = 148;
            nsm2 = device_sms();
            const int64_t items = (n_lines + TC_M - 1) / TC_M * ns;
            const int per = (int)std::min<int64_t>(items, std::max(1, nsm2 / 2));   // one CTA per SM, half per parity
            auto go = [&](auto kern) {
                smem_opt_in((const void *)kern, 225 * 1024);
                kern<<<(unsigned)(2 * per), WS_THREADS, wsm, s>>>(amap, p, n_lines, ns);
            };
            if (nst == 3 && nraw == 4) go(k_hilbert_ws<3, 4>);
            else if (nst == 3) go(k_hilbert_ws<3, 3>);
            else if (nraw == 8) go(k_hilbert_ws<2, 8>);
            else if (nraw == 6) go(k_hilbert_ws<2, 6>);
            else go(k_hilbert_ws<2, 4>);
            return 0;
        }
        const int64_t n_items = (n_lines + TC_M - 1) / TC_M * nsplit;
        int nsm = 148;
        nsm = device_sms();
        const int per_par = (int)std::min<int64_t>(n_items, nsm);      // persistent: 2 CTAs per SM, one per parity
        k_hilbert_hk<<<(unsigned)(2 * per_par), HK_THREADS, smem, s>>>(p, n_lines, nstage, nsplit);
        return 0;
    }
    if (hilbert_tc_usable(p) && hilbert_tc_nh(p.nc) <= 256 && !p.hilbert_overlap) {
        const int NH = hilbert_tc_nh(p.nc);
        const size_t smem = (size_t)4 * TC_M * TC_KC * 4 + (size_t)4 * NH * TC_KC * 4;
        smem_opt_in((const void *)k_hilbert_tc2, 220 * 1024);
        const int64_t n_lines = (int64_t)p.n_views * p.npsi;
        k_hilbert_tc2<<<(unsigned)((n_lines + TC_M - 1) / TC_M), TC2_THREADS, smem, s>>>(p, n_lines);
        return 0;
    }
    if (hilbert_tc_usable(p)) {
        const int NH = hilbert_tc_nh(p.nc);
        const size_t stage = (size_t)2 * TC_M * TC_KC * 4 + (size_t)2 * NH * TC_KC * 4;
        // double-buffer when two stages fit, except next to the backprojection (keep its footprint small)
        const int nstage = (!p.hilbert_overlap && 2 * stage <= 220 * 1024) ? 2 : 1;
        const size_t smem = nstage * stage;
        smem_opt_in((const void *)k_hilbert_tc, 225 * 1024);
        const int64_t n_lines = (int64_t)p.n_views * p.npsi;
        dim3 grid((unsigned)((n_lines + TC_M - 1) / TC_M), 2);
        k_hilbert_tc<<<grid, TC_THREADS, smem, s>>>(p, n_lines, nstage);
        return 0;
    }
    const int tpl = 2 * (((p.nc + 1) / 2 + HR - 1) / HR);
    const int lpb = tpl >= 256 ? 1 : 256 / tpl;
    const int64_t n_lines = (int64_t)p.n_views * p.npsi;
    size_t smem = sizeof(float) * (2 * (size_t)p.nc - 1 + 2 * (2 * HR + 4) + (size_t)lpb * p.nc);
    smem_opt_in((const void *)k_hilbert, 200 * 1024);
    const int threads = ((lpb * tpl + 31) / 32) * 32;
    k_hilbert<<<(unsigned)((n_lines + lpb - 1) / lpb), threads, smem, s>>>(p, n_lines, lpb);
    return 0;
}

template <int VPB>
static void launch_k4(const FilterParams &p, cudaStream_t s)
{
    dim3 grid((p.nc + K4_COLS - 1) / K4_COLS, (p.n_views + VPB - 1) / VPB);
    size_t smem = sizeof(float) * VPB * (size_t)(p.nr + 3) * (K4_COLS + 1);
    // KATS_K4=rows: the row form (entries in registers over a run of view groups); measured slower
    // than the tile kernel on every config (scripts/ab/gpu_k12k4rows.sh: C5 K4 0.94 vs 0.68 ms,
    // C2 0.31 vs 0.11 ms), so the tile kernel stays the default
    const char *ke = std::getenv("KATS_K4");
    const int tiles = (p.nr + 3) * (K4_COLS + 1);
    if (ke && std::string(ke) == "rows" && tiles <= 256 * 9) {
        // view groups per CTA: as many as keep >= 4 CTAs per SM (entries held over the run), at most 8
        const int nb = (p.nc + K4_COLS - 1) / K4_COLS, groups = (p.n_views + VPB - 1) / VPB;
        int ng = 8;
        while (ng > 1 && (int64_t)nb * ((groups + ng - 1) / ng) < 4 * device_sms()) ng /= 2;
        const size_t sm2 = 2 * smem;
        const dim3 g2(nb, (groups + ng - 1) / ng);
        if (tiles <= 256 * 4) {
            smem_opt_in((const void *)k_bwd_rebin_cos_rows<VPB, 4>, sm2);
            k_bwd_rebin_cos_rows<VPB, 4><<<g2, 256, sm2, s>>>(p, ng);
        } else {
            smem_opt_in((const void *)k_bwd_rebin_cos_rows<VPB, 9>, sm2);
            k_bwd_rebin_cos_rows<VPB, 9><<<g2, 256, sm2, s>>>(p, ng);
        }
        return;
    }
    smem_opt_in((const void *)k_bwd_rebin_cos<VPB>, 200 * 1024);
    k_bwd_rebin_cos<VPB><<<grid, 256, smem, s>>>(p);
}

void launch_bwd_rebin_cos(const FilterParams &p, cudaStream_t s)
{
    // KATS_K4_VPB (A/B): views per CTA.  Default 4 for detectors of <= 32 rows, else 2
    // (scripts/ab/gpu_k4vpb.sh: 2 vs 1 view C5 4.37 -> 4.29 ms, C3 9.38 -> 9.31 ms, C4 unchanged,
    // 4 views made C4's K4 1.14 -> 1.32 ms; gpu_k4vpb2.sh, 4x chunks: 4 vs 2 views C5 4.14-4.24 ->
    // 4.07 ms, C2 1.703 -> 1.696 ms)
    const char *e = std::getenv("KATS_K4_VPB");
    const int vpb = e ? std::atoi(e) : (p.nr <= 32 ? 4 : 2);
    if (vpb >= 4) launch_k4<4>(p, s);
    else if (vpb == 2) launch_k4<2>(p, s);
    else launch_k4<1>(p, s);
}

// ---------------------------------------------------------------------------
// Adjoint of steps 1-6 (NEXT-1); DESIGN.md §5.  Per view:
//   quad adjoint -> gF^T (transpose of the quad construction of K4, gathered)
//   -> K4^T: g4^T = scatter over ψ of cos α · gF^T           (k_bwd_rebin_cos_T)
//   -> K3^T = -K3 (the kernel is odd: K[-d] = -K[d])          (launch_hilbert, sign -1)
//   -> K2^T with the length weight: g1^T = wlen · scatter over w of g3^T  (k_fwd_rebin_T)
//   -> K1^T: transposed view/α difference stencils (gathered, k_deriv_T).
// A thread owns one detector column of a view in the scatters, so no atomics.
// ---------------------------------------------------------------------------
// k_fwd_rebin_T: the scatter target (one column of g1^T) is private to the thread; it is accumulated
// in shared memory ([entry][thread]: conflict-free) and written out once, coalesced across α.
// (K4^T keeps its global read-modify-write: its npsi-deep column would cost occupancy.)
constexpr int KT_THREADS = 64;

// Two views per thread (KATS_K4T_VPB=2): the same per-view arithmetic, the rebin entry and cos α
// loaded once for both views, their quad loads issued together.
__global__ void __launch_bounds__(128) k_bwd_rebin_cos_T2(FilterParams p, const float4 *__restrict__ qT)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, v0 = blockIdx.y * 2;
    if (l >= p.nc) return;
    const int nv = min(2, p.n_views - v0);
    const int nc = p.nc, nr = p.nr, nq = nr + 2, c = (nr + 2) / 2;
    for (int j = 0; j < nv; ++j)
        for (int i = 0; i < p.npsi; ++i) p.g4[k3in_off(p, (size_t)(v0 + j) * p.npsi + i, l)] = 0.f;
    const float ca = __ldg(p.cos_alpha + l);
    const float4 *qa[2], *qb[2];
    for (int j = 0; j < 2; ++j) {
        const int v = v0 + min(j, nv - 1);
        qa[j] = qT + ((size_t)v * nc + l) * nq;
        qb[j] = l > 0 ? qa[j] - nq : nullptr;
    }
    for (int m = 0; m < nr; ++m) {
        const float rh = (float)(m + 2 - c), rl = (float)(m + 1 - c);
        float gt[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float4 A = qa[j][m + 2], B = qa[j][m + 1];
            gt[j] = 0.5f * A.x - (A.z - rh * A.x) + 0.5f * B.x + (B.z - rl * B.x);
            if (qb[j]) {
                const float4 C = qb[j][m + 2], D = qb[j][m + 1];
                gt[j] += 0.5f * C.y - (C.w - rh * C.y) + 0.5f * D.y + (D.w - rl * D.y);
            }
        }
        const RebinEntry e = p.br[m * nc + l];
        if (e.idx < 0) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (j >= nv) break;
            const size_t line0 = (size_t)(v0 + j) * p.npsi;
            const float val = ca * gt[j];
            p.g4[k3in_off(p, line0 + e.idx, l)] += (1.f - e.frac) * val;
            p.g4[k3in_off(p, line0 + e.idx + 1, l)] += e.frac * val;
        }
    }
}

__global__ void __launch_bounds__(128) k_bwd_rebin_cos_T(FilterParams p, const float4 *__restrict__ qT)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
    if (l >= p.nc) return;
    const int nc = p.nc, nr = p.nr, nq = nr + 2, c = (nr + 2) / 2;
    const size_t line0 = (size_t)v * p.npsi;                    // output: K3^T's input lines
    for (int i = 0; i < p.npsi; ++i) p.g4[k3in_off(p, line0 + i, l)] = 0.f;
    const float4 *qa = qT + ((size_t)v * nc + l) * nq;           // column l: its taps are quad x, z
    const float4 *qb = l > 0 ? qa - nq : nullptr;                // column l-1: this column is its y, w
    const float ca = __ldg(p.cos_alpha + l);
    for (int m = 0; m < nr; ++m) {
        // quad r = m + 2 has row m as its lower tap, quad r = m + 1 as its upper tap
        const float rh = (float)(m + 2 - c), rl = (float)(m + 1 - c);
        const float4 A = qa[m + 2], B = qa[m + 1];
        float gt = 0.5f * A.x - (A.z - rh * A.x) + 0.5f * B.x + (B.z - rl * B.x);
        if (qb) {
            const float4 C = qb[m + 2], D = qb[m + 1];
            gt += 0.5f * C.y - (C.w - rh * C.y) + 0.5f * D.y + (D.w - rl * D.y);
        }
        const RebinEntry e = p.br[m * nc + l];
        if (e.idx < 0) continue;
        const float val = ca * gt;
        p.g4[k3in_off(p, line0 + e.idx, l)] += (1.f - e.frac) * val;
        p.g4[k3in_off(p, line0 + e.idx + 1, l)] += e.frac * val;
    }
}

__global__ void __launch_bounds__(KT_THREADS) k_fwd_rebin_T(FilterParams p, float *__restrict__ g1T)
{
    extern __shared__ float acc_s[];                               // [nr][KT_THREADS]
    const int l = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
    const int nc = p.nc;
    float *acc = acc_s + threadIdx.x;
    for (int m = 0; m < p.nr; ++m) acc[m * KT_THREADS] = 0.f;
    if (l < nc) {
        const float *g3T = p.g3 + (size_t)v * p.npsi * nc + l;
        for (int i = 0; i < p.npsi; ++i) {
            const RebinEntry e = p.fr[i * nc + l];
            if (e.idx < 0) continue;
            const float t = g3T[(size_t)i * nc];
            acc[e.idx * KT_THREADS] += (1.f - e.frac) * t;
            acc[(e.idx + 1) * KT_THREADS] += e.frac * t;
        }
        float *o = g1T + (size_t)v * p.nr * nc + l;
        if (p.flat) {                                              // D/sqrt(D²+u²+w²) (A27)
            const float a = __ldg(p.flat_a + l);
            for (int m = 0; m < p.nr; ++m) {
                const float wd = ((float)m - 0.5f * (float)(p.nr - 1)) * p.dw_over_D;
                o[(size_t)m * nc] = acc[m * KT_THREADS] * rsqrtf(1.f + fmaf(a, a, wd * wd));
            }
        } else {
            for (int m = 0; m < p.nr; ++m) o[(size_t)m * nc] = acc[m * KT_THREADS] * __ldg(p.wlen + m);
        }
    }
}

// raw view v (absolute u0 - 1 .. u0 + nu) <- g1^T of filtered views v-1, v, v+1 (those in [u0, u0+nu))
__global__ void __launch_bounds__(128) k_deriv_T(FilterParams p, const float *__restrict__ g1T, int64_t nu,
                                                 int items, float *__restrict__ out)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
    if (l >= p.nc) return;
    const int64_t per = nu + 2;                                   // raw views of an item (slab of a batch)
    const int nc = p.nc;
    const size_t rs = (size_t)p.nr * nc;
    // grid.z (<= 65535) strides over the items' raw views
    for (int64_t z = blockIdx.z; z < per * items; z += gridDim.z) {
        const int64_t item = z / per, vr = z - item * per;       // raw view - (u0 - 1)
        const float *gi = g1T + (size_t)item * nu * rs;           // the stencils stay inside the item
        auto g = [&](int64_t f, int ll) -> float {                // g1^T of filtered view f (relative to u0)
            return (f >= 0 && f < nu) ? gi[(size_t)f * rs + (size_t)m * nc + ll] : 0.f;
        };
        const int64_t f = vr - 1;                                 // this raw view as a filtered view
        float acc = (g(f - 1, l) - g(f + 1, l)) * p.inv_2dlam;    // view stencil (g(v+1) - g(v-1)) / 2Δλ
        // α stencil of the same view: centred inside, one-sided at both edges (flat, A27: the u stencil,
        // each source column's term weighted by (u²+D²)/D)
        auto gu = [&](int ll) -> float {
            if (!p.flat) return g(f, ll);
            const float a = __ldg(p.flat_a + ll);
            return g(f, ll) * p.D * fmaf(a, a, 1.f);
        };
        if (l == 0) acc -= gu(0) * p.inv_dalpha;
        if (l == nc - 1) acc += gu(nc - 1) * p.inv_dalpha;
        if (l >= 1) acc += gu(l - 1) * (l - 1 == 0 ? p.inv_dalpha : p.inv_2dalpha);
        if (l + 1 <= nc - 1) acc -= gu(l + 1) * (l + 1 == nc - 1 ? p.inv_dalpha : p.inv_2dalpha);
        if (p.flat) {
            // the w stencil's transpose (weights u w / D of the source row), one-sided at both row edges
            const int nr = p.nr;
            const float a = __ldg(p.flat_a + l);
            auto gw = [&](int mm) -> float {
                const float wd = ((float)mm - 0.5f * (float)(nr - 1)) * p.dw_over_D;
                return (f >= 0 && f < nu) ? gi[(size_t)f * rs + (size_t)mm * nc + l] * a * wd * p.D : 0.f;
            };
            if (m == 0) acc -= gw(0) * p.inv_dw;
            if (m == 1) acc += gw(0) * p.inv_dw;
            if (m == nr - 1) acc += gw(nr - 1) * p.inv_dw;
            if (m == nr - 2) acc -= gw(nr - 1) * p.inv_dw;
            if (m - 1 >= 1 && m - 1 <= nr - 2) acc += gw(m - 1) * p.inv_2dw;
            if (m + 1 >= 1 && m + 1 <= nr - 2) acc -= gw(m + 1) * p.inv_2dw;
        }
        out[((size_t)item * per + vr) * rs + (size_t)m * nc + l] = acc;
    }
}

// K4^T, streaming form (T_br monotone down each column): a CTA takes one view and 128 columns; the
// quad-adjoint columns (rows contiguous) are staged through shared memory in chunks of rows with
// coalesced loads, and each thread walks its column's rows in order keeping the two κ-lines the
// current row feeds in registers: a line is written once, when the rows have moved past it (lines no
// row reaches are written 0), so there is no read-modify-write and no separate zeroing pass.
constexpr int K4T_COLS = 128, K4T_RC = 16, K4T_QP = K4T_RC + 3;     // rows per chunk; staged pitch (odd)
__global__ void __launch_bounds__(K4T_COLS) k_bwd_rebin_cos_T_stream(FilterParams p, const float4 *__restrict__ qT)
{
    __shared__ float4 sq[(K4T_COLS + 1) * K4T_QP];                    // [column l0-1+c][quad row m0+1+r]
    const int tid = threadIdx.x, l0 = blockIdx.x * K4T_COLS, l = l0 + tid, v = blockIdx.y;
    const int nc = p.nc, nr = p.nr, nq = nr + 2, c = (nr + 2) / 2;
    const size_t line0 = (size_t)v * p.npsi;
    const float4 *qv = qT + (size_t)v * nc * nq;
    const float ca = l < nc ? __ldg(p.cos_alpha + l) : 0.f;
    int L = -1;                                                         // first line of the pair held
    float a0 = 0.f, a1 = 0.f;
    auto put = [&](int line, float val) { p.g4[k3in_off(p, line0 + line, l)] = val; };
    for (int m0 = 0; m0 < nr; m0 += K4T_RC) {
        const int rc = min(K4T_RC, nr - m0);
        __syncthreads();
        // quad rows m0+1 .. m0+rc+1 of columns l0-1 .. l0+127 (coalesced along each column's rows)
        const int nrow = rc + 1;
        for (int i = tid; i < (K4T_COLS + 1) * nrow; i += K4T_COLS) {
            const int cc = i / nrow, r = i - cc * nrow, lc = l0 - 1 + cc;
            sq[cc * K4T_QP + r] = (lc >= 0 && lc < nc) ? __ldg(qv + (size_t)lc * nq + m0 + 1 + r)
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        if (l >= nc) continue;
        const float4 *qa = sq + (tid + 1) * K4T_QP, *qb = sq + tid * K4T_QP;   // column l, column l-1
        for (int j = 0; j < rc; ++j) {
            const int m = m0 + j;
            const float rh = (float)(m + 2 - c), rl = (float)(m + 1 - c);
            const float4 A = qa[j + 1], B = qa[j];
            float gt = 0.5f * A.x - (A.z - rh * A.x) + 0.5f * B.x + (B.z - rl * B.x);
            if (l > 0) {
                const float4 C = qb[j + 1], D = qb[j];
                gt += 0.5f * C.y - (C.w - rh * C.y) + 0.5f * D.y + (D.w - rl * D.y);
            }
            const RebinEntry e = p.br[m * nc + l];
            if (e.idx < 0) continue;
            const float val = ca * gt, c0 = (1.f - e.frac) * val, c1 = e.frac * val;
            if (L < 0) {
                for (int i = 0; i < e.idx; ++i) put(i, 0.f);
                L = e.idx; a0 = c0; a1 = c1;
            } else if (e.idx == L) {
                a0 += c0; a1 += c1;
            } else if (e.idx == L + 1) {
                put(L, a0);
                L = e.idx; a0 = a1 + c0; a1 = c1;
            } else {
                put(L, a0); put(L + 1, a1);
                for (int i = L + 2; i < e.idx; ++i) put(i, 0.f);
                L = e.idx; a0 = c0; a1 = c1;
            }
        }
    }
    if (l >= nc) return;
    int next = 0;
    if (L >= 0) { put(L, a0); put(L + 1, a1); next = L + 2; }
    for (int i = next; i < p.npsi; ++i) put(i, 0.f);
}

void launch_bwd_rebin_cos_T(const FilterParams &p, const float4 *qT, cudaStream_t s)
{
    // streaming form when T_br is monotone down every column (all configurations here; KATS_K4T=rmw: the
    // read-modify-write kernel below)
    const char *k4t = std::getenv("KATS_K4T");
    if (p.br_monotone && !(k4t && std::string(k4t) == "rmw")) {
        k_bwd_rebin_cos_T_stream<<<dim3((p.nc + K4T_COLS - 1) / K4T_COLS, p.n_views), K4T_COLS, 0, s>>>(p, qT);
        return;
    }
    const char *e = std::getenv("KATS_K4T_VPB");            // A/B: two views per thread
    if (e && std::atoi(e) == 2) {
        k_bwd_rebin_cos_T2<<<dim3((p.nc + 127) / 128, (p.n_views + 1) / 2), 128, 0, s>>>(p, qT);
        return;
    }
    k_bwd_rebin_cos_T<<<dim3((p.nc + 127) / 128, p.n_views), 128, 0, s>>>(p, qT);
}

void launch_fwd_rebin_T(const FilterParams &p, float *g1T, cudaStream_t s)
{
    smem_opt_in((const void *)k_fwd_rebin_T, sizeof(float) * p.nr * KT_THREADS);
    k_fwd_rebin_T<<<dim3((p.nc + KT_THREADS - 1) / KT_THREADS, p.n_views), KT_THREADS,
                    sizeof(float) * p.nr * KT_THREADS, s>>>(p, g1T);
}

// K1^T of the half-sample derivative (NEXT-4): raw view r (relative to the first filtered view) of an
// item receives from filtered views r-1 (as its upper view) and r (as its lower view), raw row mr from
// rows mr-1, mr and raw column lr from columns lr-1, lr of the half-shifted grid, with the forward's
// coefficients: 1/(4Δλ) (+ upper view, - lower) and 1/(4Δα) (+ right column, - left).
__global__ void __launch_bounds__(128) k_deriv_half_T(FilterParams p, const float *__restrict__ g1T, int64_t nu,
                                                      int items, float *__restrict__ out)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x, mr = blockIdx.y;
    const int nc = p.nc, nr = p.nr, rnc = nc + 1;
    if (lr >= rnc) return;
    const int64_t per = nu + 1;                                   // raw views of an item
    const size_t rs = (size_t)nr * nc, rrs = (size_t)(nr + 1) * rnc;
    const float sq = 0.25f * p.inv_2dlam * 2.f, sa = 0.25f * p.inv_dalpha;
    for (int64_t z = blockIdx.z; z < per * items; z += gridDim.z) {
        const int64_t item = z / per, r = z - item * per;
        const float *gi = g1T + (size_t)item * nu * rs;
        float acc = 0.f;
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) {
            const int64_t k = r - 1 + dk;                         // dk 0: this raw view is k's upper view
            if (k < 0 || k >= nu) continue;
            const float cq = dk == 0 ? sq : -sq;
#pragma unroll
            for (int dm = 0; dm < 2; ++dm) {
                const int m = mr - 1 + dm;
                if (m < 0 || m >= nr) continue;
#pragma unroll
                for (int dl = 0; dl < 2; ++dl) {
                    const int l = lr - 1 + dl;                    // dl 0: this raw column is l's right column
                    if (l < 0 || l >= nc) continue;
                    acc = fmaf(gi[(size_t)k * rs + (size_t)m * nc + l], cq + (dl == 0 ? sa : -sa), acc);
                }
            }
        }
        out[((size_t)item * per + r) * rrs + (size_t)mr * rnc + lr] = acc;
    }
}

void launch_deriv_T(const FilterParams &p, const float *g1T, int64_t nu, float *out, cudaStream_t s, int items)
{
    if (p.half) {
        const int64_t nz = std::min<int64_t>((nu + 1) * items, 65535);
        k_deriv_half_T<<<dim3((p.nc + 1 + 127) / 128, p.nr + 1, (unsigned)nz), 128, 0, s>>>(p, g1T, nu, items, out);
        return;
    }
    const int64_t nz = std::min<int64_t>((nu + 2) * items, 65535);
    k_deriv_T<<<dim3((p.nc + 127) / 128, p.nr, (unsigned)nz), 128, 0, s>>>(p, g1T, nu, items, out);
}

}  // namespace kats
