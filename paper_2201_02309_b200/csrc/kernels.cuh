// kernels.cuh — launch interfaces of the sm_100a kernels (internal).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "plan.hpp"

namespace kats {

// Runtime helpers (api.cu).  Both act on the current device (the plan's: every entry point calls
// cudaSetDevice first) and are thread-safe.
cudaError_t smem_opt_in(const void *kernel, size_t bytes);   // dynamic shared-memory opt-in, once per device
int device_sms();                                            // multiprocessor count of the current device

// Filter steps 1-6 over `n_views` consecutive views.
struct FilterParams {
    const float *sino;        // raw data of filtered view g = view0 + v at sino + raw(g) * rows*cols, raw(g) = g (+ 2 per
                              // preceding slab), halo at raw(g) -+ 1
    int n_views;
    int nr, nc, npsi;
    float inv_2dlam, inv_dalpha, inv_2dalpha;
    const float *wlen;        // D/sqrt(D²+w_m²)
    const RebinEntry *fr;     // [npsi][nc]
    const RebinEntry *br;     // [nr][nc]
    const float *cos_alpha;   // [nc]
    const float *hilbert;     // [2nc-1]
    const float *hilbert_tc;  // tensor-core tap table (hilbert_tc_table), or null
    const float *hilbert_hk;  // tensor-core Hankel-core tap table (hilbert_hk_table), or null
    float *g3, *g4;           // κ-line intermediates [n_views][npsi][nc]
    float4 *gq;               // filtered views as column-major 2x2 sum/difference tap quads [n_views][nc][nr+2] (BP input)
    float *gF;                // optional plain filtered views [n_views][nr][nc] (debug), may be null
    float sign;               // K3 output sign: +1 forward, -1 for the adjoint (odd kernel)
    int hilbert_overlap;      // K3 runs next to the TMEM backprojection: keep its TMEM allocation <= 128 columns
    int64_t view0;            // K12: first filtered view of this launch in the run_filter sequence
    int64_t slab_views;       // K12: filtered views per slab of a batch (each slab carries its own +-1 halo); 0 = one scan
    int k3_in_split;          // K3's input lines are parity-split (even columns, then odd, each hp floats): written
                              // by K12 (forward) / K4^T (adjoint) when the warp-specialized K3 reads them
    int hp;                   // half pitch of a parity-split line (floats, multiple of 4)
    int half;                 // NEXT-4: Noo's half-sample derivative (raw views have nr+1 rows, nc+1 columns)
    int apod;                 // NEXT-4: Hann-apodised Hilbert (K3's input lines smoothed [1/4, 1/2, 1/4])
    int flat;                 // NEXT-4: flat detector (K12 flat: derivative at constant ray direction, 2-D length weight)
    const float *flat_a;      // flat: u_l / D per column
    float D, dw_over_D, inv_dw, inv_2dw;   // flat K12
    int br_monotone;          // T_br's κ-line index nondecreasing down every column (K4^T streams its lines)
};

void launch_deriv_fwd_rebin(const FilterParams &p, cudaStream_t s);   // K12: Eqs. 8, 9, 10-11
int launch_hilbert(const FilterParams &p, cudaStream_t s);            // K3:  Eq. 12 (-1: input tensor map failed)
bool hilbert_split_input(const FilterParams &p);                      // the K3 launch_hilbert picks reads split lines
void launch_hann_smooth(const FilterParams &p, float *lines, int64_t n_lines, int split, cudaStream_t s);  // A26, in place
inline int g3_half_pitch(int nc) { return ((nc + 1) / 2 + 3) & ~3; }
inline int g3_line_pitch(int nc) { return 2 * g3_half_pitch(nc); }   // >= nc; scratch line pitch
size_t hilbert_tc_table_floats(int nc);
void hilbert_tc_table(int nc, const float *kd, std::vector<float> &out);
size_t hilbert_hk_table_floats(int nc);
void hilbert_hk_table(int nc, const float *kd, std::vector<float> &out);
void launch_bwd_rebin_cos(const FilterParams &p, cudaStream_t s);     // K4:  Eqs. 13-15
// adjoint (NEXT-1)
void launch_bwd_rebin_cos_T(const FilterParams &p, const float4 *qT, cudaStream_t s);   // quad^T + K4^T
void launch_fwd_rebin_T(const FilterParams &p, float *g1T, cudaStream_t s);            // K2^T + length weight
void launch_deriv_T(const FilterParams &p, const float *g1T, int64_t nu, float *out, cudaStream_t s,
                    int items = 1);  // K1^T (items: slabs of a batch, nu filtered views each)

// Step 7 backprojection over `n_items`
// independent pitches/slabs sharing the periodic tables.
struct BPParams {
    const float4 *gq;         // filtered views as column-major sum/difference tap quads [views][nc][nr+2]
    int64_t off0, item_views; // view index of pitch-relative view k for item b: k + off0 + b*item_views
    int n_items;
    int nr, nc, nx, ny, nz;
    unsigned colbytes;        // (nr + 2) * 16: one quad column (rows contiguous)
    int64_t viewbytes;        // nc * (nr + 2) * 16: one quad view
    const int2 *pi_k;         // [nz][ny][nx] (k_first, k_last)
    const float2 *pi_w;       // [nz][ny][nx] (ω_first, ω_last)
    const ViewGeom *view;     // [k - view_lo]
    int view_lo;
    float R, D_over_dw, inv_dalpha, col_c, row_c15, colmax, rowmax;
    float row_cc, qmagic;     // centred quad-row origin row_c15 - c and kMagic + c, c = (nr + 2) / 2
    float pm_lo, pm_hi;       // centred quad-row range of an in-detector sample (checked taps)
    float at[7];              // α*/Δα polynomial in t = u/v*: t·Σ at[i] t^(2i)
    float uu;                 // 1: curved (w* = D(z-z_src)/sqrt(u²+v*²)); 0: flat detector (D(z-z_src)/v*; at = {D/Δu, 0..})
    float x0, dx, y0, dy, dz;
    float scale;              // Δλ / 2π
    bool poly;                // use the polynomial arctangent (|α| <= 36.8°)
    bool checked;             // per-sample detector test on interior views (margin check failed)
    bool staged;              // use the shared-memory staged kernel
    int fp_cols, fp_rows;     // per-view quad box of one CTA (staged kernel)
    int nbatch;               // slots in the staged kernel's ring (set by the launcher)
    int64_t gq_views;         // views in the gq array (TMA tensor extent)
    int max_cta_views;        // upper bound of a CTA's interior view range (box table size)
    int fp_cols_column;       // quad columns of a tile's full-column box (sliding-window kernel)
    int max_active;           // max slices of a column sharing an interior view
    bool windows_monotone;    // host check: per-column interior windows non-empty and monotone in z
    int tail_quads;           // shared-memory pad after the ring for reads of not-yet-open window entries
    unsigned zero;            // runtime 0 (opaque to ptxas)
    int warp_span;            // max live slices of a warp (host, TMEM-window kernel)
    int warp_span2;           // the same over two consecutive views (TMEM kernel, view pairs)
    int pad_quads;            // head/tail pad (quads) for the TMEM-window kernel: span + 8 slices of row travel
    int pad_quads2;           // the same for view pairs (span2)
    int nq_s;                 // staged-kernel column pitch in quads: staged rows rounded up to 3 or 5 mod 8
    int q_lo;                 // first staged quad row (interior samples reach quad rows q_lo ..)
    int box_w[3];             // staged box widths (columns): full, and two narrower classes (set by the launcher)
    int box_h[4];             // window kernel: staged box heights (quad rows), full and narrower classes (launcher)
    int crop;                 // window kernel: crop each view's box to the rows of the tile's open slices
    int ring_bytes;           // window kernel with cropped boxes: byte ring of variable-size view regions
    int ring_prefetch;        // byte ring: L2 prefetch of the boxes this many views ahead (0: none)
    int qmap44;               // TMEM kernel: lanes in 4x2 quarter-warps / 4x4 half-warps (else 8x1 / 8x2)
    int adj_nqp;              // adjoint: quad-row pitch of a box column in shared memory (set by the launcher)
    bool adj_fixed_ok;        // adjoint: the int32 fixed-point box cannot overflow (<= 2^10 contributions per cell)
    int ends_pre;             // staged kernels: end views written ahead into vol by k_bp_ends (launcher)
    const int *tile_order;    // staged kernels: 16x16 column tiles heaviest first (ty * ntx + tx), or null
    int bp_items;             // window kernel: batch items per CTA (1 or 2; set by the launcher)
    int win_variant;          // window kernel variant V (0 plain, 1 uniform sample tail, 2 + two items per CTA)
    int tmem_cols, tmem_alloc;   // TMEM columns per warp / allocated per CTA (set by the launcher)
    int lg_nbatch;            // log2(nbatch) (TMEM kernel: slot parity from the view counter)
    unsigned slot_bytes, col_bytes;   // TMEM kernel: bytes per ring slot / per quad column in a slot
    float *vol;               // [n_items][nz][ny][nx] (adjoint: the input)
    float4 *gqT;              // adjoint: quad-adjoint output, layout of gq (accumulated)
};

int launch_backproject(const BPParams &p, cudaStream_t s);            // K5; returns the KATS_BP_* variant
int launch_backproject_adjoint(const BPParams &p, cudaStream_t s);    // K5^T into p.gqT (-1: plan unsupported)
void launch_make_quads(const float *gF, float4 *q, int64_t n, int nr, int nc, cudaStream_t s);

// ---- data generation (NEXT-3, datagen.cu) ----
struct DataGenParams {
    double R, D, h, lambda0, z0, dlam, d_w, d_alpha, alpha_offset, dx, dy;
    int nr, nc, nx, ny;
    int flat;                 // KATS_FLAG_FLAT: column coordinate u [mm] on the plane at distance D
};
void launch_project_ellipsoids(const DataGenParams &p, const double *ell, int n, int64_t v0, int64_t nv, float *out,
                               cudaStream_t s);
void launch_project_volume(const DataGenParams &p, const float *vol, int nzv, float zv0, float dzv, int64_t v0,
                           int64_t nv, float *out, unsigned long long *n_trunc, cudaStream_t s);
void launch_degrade(const DataGenParams &p, const float *in, int64_t v0, int64_t nv, int stride, double I0, double var,
                    uint64_t seed, int mode, float *up, unsigned *maxbits, float *out, long long *counts, float *M_out,
                    cudaStream_t s);

}  // namespace kats
