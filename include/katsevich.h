/*
 * katsevich.h — C ABI of the B200-native pitch-periodic Katsevich
 * reconstruction (arXiv 2201.02309 §II).
 *
 * Problem statement:
 *   helix       a(λ) = (R cos(λ+λ0), R sin(λ+λ0), z0 + P λ / 2π)          Eq. (1), l.88
 *   FOV         U = {x² + y² ≤ r²}, 0 < r < R                                l.96
 *   detector    curved, centred on the source at distance D; coordinates (α, w)   l.117
 *               α_l = (l - (n_cols-1)/2 + alpha_offset)·d_alpha   (P:l.328, quarter offset)
 *               w_m = (m - (n_rows-1)/2)·d_w                       (P:l.340)
 *   views       view index v <-> λ = v·Δλ,  Δλ = 2π / views_per_turn
 *   volume      x_i = (i - nx/2)·dx, y likewise (P:l.316); per pitch k slices
 *               z = j·P/nz + k·P, j = 0..nz-1 (the slice at z = P belongs to
 *               the next pitch, P:l.357-368, l.740)
 *
 * Data layouts (all C order, fp32, little endian):
 *   sinogram  g[v][m][l]       views × rows × cols (α contiguous)
 *   volume    f[j][iy][ix]     nz·n_pitches × ny × nx (x contiguous)
 *
 * Ownership: the caller owns every data pointer it passes (sinograms,
 * volumes, workspace).  Device pointers may come from any allocator (e.g.
 * torch tensors' data_ptr()); `cuda_stream` is a cudaStream_t (0 = legacy
 * default stream), e.g. torch.cuda.current_stream().cuda_stream.  The plan
 * owns its host and device tables (freed by katsevich_destroy) and is
 * immutable after katsevich_precompute; concurrent reconstruct calls on
 * different streams with distinct workspaces are safe.  All launches are
 * asynchronous on the given stream; only katsevich_precompute (table upload),
 * katsevich_reconstruct_host and katsevich_profile_read synchronise.
 *
 * Errors: every int-returning call returns KATS_OK (0), a positive warning or
 * a negative error code; no call aborts or exits.  katsevich_error_string()
 * names a code, katsevich_last_error_detail() gives the plan's last detail
 * message (e.g. the first and last reconstructible pitch on KATS_ERR_COVERAGE,
 * or cudaGetErrorString on KATS_ERR_CUDA).
 */
#ifndef KATSEVICH_H
#define KATSEVICH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    KATS_OK = 0,
    KATS_WARN_TD_NOT_COVERED = 1,     /* detector rows do not cover the Tam–Danielsson window (w_L > (n_rows-1)d_w/2) */
    KATS_ERR_NULL = -1,               /* a required pointer argument is NULL */
    KATS_ERR_INVALID_GEOMETRY = -2,   /* R, D, P <= 0; r_fov >= R; views_per_turn < 3; n_cols < 2; n_rows < 2; spacings <= 0; ... */
    KATS_ERR_NOT_PRECOMPUTED = -3,    /* katsevich_precompute has not run on this plan */
    KATS_ERR_COVERAGE = -4,           /* the sinogram view range does not contain a requested pitch's slab */
    KATS_ERR_PI_NONCONVERGENCE = -5,  /* a PI-line or κ-line root did not converge */
    KATS_ERR_WORKSPACE = -6,          /* workspace smaller than katsevich_workspace_bytes() */
    KATS_ERR_CUDA = -7,               /* a CUDA runtime call or launch failed (detail: cudaGetErrorString) */
    KATS_ERR_NO_DEVICE = -8,          /* device operation on a host-only plan (cuda_device < 0) */
    KATS_ERR_ARGUMENT = -9            /* other invalid argument (counts, ranges) */
};

/* Geometry of PAPER.md l.87-98/l.117/l.189/l.311-349.  Lengths in mm, angles in rad. */
typedef struct {
    double  R;               /* helix radius R (P:l.88) */
    double  D;               /* source-to-detector distance D, curved detector centred on the source (P:l.125) */
    double  pitch;           /* table feed per turn P (P:l.90) */
    double  lambda0, z0;     /* start angle λ0 and height z0 of the helix (P:l.92) */
    double  r_fov;           /* FOV cylinder radius r, 0 < r < R (P:l.96); 0 => half-diagonal of the xy grid (P:l.322) */
    int32_t n_rows;          /* detector rows (w) */
    double  d_w;             /* row pitch at distance D */
    int32_t n_cols;          /* detector columns (α) */
    double  d_alpha;         /* column pitch in fan angle (KATS_FLAG_FLAT: in mm on the detector plane) */
    double  alpha_offset;    /* fractional column offset in samples (quarter offset 0.25, P:l.328) */
    int32_t views_per_turn;  /* Δλ = 2π/views_per_turn (integer, so pitches are whole view strides) */
    int32_t nx, ny;          /* voxel grid */
    double  dx, dy;
    int32_t nz_per_pitch;    /* slices per pitch; dz = pitch / nz_per_pitch */
    int32_t n_psi;           /* κ-lines ψ_i on [-π/2-α_m, π/2+α_m] (P:l.132); 0 => 2·n_rows+1 */
    int32_t flags;           /* 0 or an OR of KATS_FLAG_HALF_SAMPLE, KATS_FLAG_HANN, KATS_FLAG_FLAT */
} katsevich_geometry;

/* Method variant flags (katsevich_geometry.flags):
 * KATS_FLAG_HALF_SAMPLE — step 1 (Eq. 8) by Noo's 2x2x2 half-sample derivative
 *   ([Noo2003a], cited at P:l.115; reading A25): g1 on the grid shifted by half a sample in
 *   λ, α and w, where steps 2-7 then run — every table (T_pi, T_fr, T_br) and the filtered data
 *   (katsevich_filter's g3/g4/gF, katsevich_export_tables) live on that grid: n_rows-1 rows,
 *   n_cols-1 columns, views at λ_{k+½}.  Filtered view k needs raw views k and k+1 (no lower halo):
 *   katsevich_pitch_views / _scan_views report the raw views.  Needs 3 <= n_rows <= 65, n_cols >= 3. */
#define KATS_FLAG_HALF_SAMPLE 1
/* KATS_FLAG_HANN — step 4 (Eq. 12) with the Hann-apodised Hilbert filter (reading A26): the
 *   kernel's frequency response -i sgn(σ) times cos²(πσΔα), i.e. the band-limited kernel of reading
 *   A10 applied to each κ-line smoothed by [1/4, 1/2, 1/4] along α (zeros beyond the detector).  A
 *   noise/resolution trade-off for noisy sparse-view data (P:l.396-404); the adjoint is exact. */
#define KATS_FLAG_HANN 2
/* KATS_FLAG_FLAT — a flat detector (reading A27): the plane at distance D from the source,
 *   perpendicular to the central ray, columns u_l = (l-(n_cols-1)/2+alpha_offset)·d_alpha [mm], rows
 *   w_m as for the curved detector.  Steps 1-7 in those coordinates after [Noo2003a] (the
 *   implementation PAPER.md l.115 cites): the derivative at constant ray direction
 *   (∂_λ + (u²+D²)/D ∂_u + uw/D ∂_w), the length weight D/√(D²+u²+w²), κ-lines
 *   w_κ(u,ψ) = DP/(2πR)(ψ + (ψ/tanψ) u/D) (Eq. 11 over cos α at u = D tan α), the Hilbert kernel
 *   1/(π(u−u')) along u, no post-cosine, and step 7 at u* = D x·e_t/v*, w* = D(z−z_src)/v*; the
 *   adjoint transposes those steps.  Not with KATS_FLAG_HALF_SAMPLE (the plan is rejected). */
#define KATS_FLAG_FLAT 4

typedef struct katsevich_plan katsevich_plan;

/* Validate `geom` and create a plan bound to CUDA device `cuda_device`
 * (cuda_device < 0: host-only plan — precompute and table export work,
 * device entry points return KATS_ERR_NO_DEVICE).  *out receives the plan
 * (NULL on error). */
int katsevich_plan_create(const katsevich_geometry *geom, int cuda_device, katsevich_plan **out);

/* Pre-calculating step ("implemented by the CPU" l.265):
 * in double precision on the host, computes once for pitch 0 and reuses for
 * every pitch by periodicity (l.174-185, l.222-231):
 *   T_pi  PI-line backprojection limits per voxel (k_first, k_last, end weights),
 *   T_fr  forward rebin row index/fraction of w_κ(α_l, ψ_i) (Eq. 11),
 *   T_br  backward rebin ψ index/fraction of ψ̂(α_l, w_m) (Eq. 14),
 *   T_view per-view cos/sin(λ+λ0) over the pitch's slab;
 * then uploads them to the device on `cuda_stream` and synchronises.
 * Returns KATS_WARN_TD_NOT_COVERED when the rows do not cover the TD window
 * (the result is still computed), KATS_ERR_PI_NONCONVERGENCE on solver failure. */
int katsevich_precompute(katsevich_plan *plan, void *cuda_stream);

/* Views pitch `pitch` needs: [first_view, first_view + n_views) including the
 * ±1-view derivative halo (P:l.246, l.373-377). */
int katsevich_pitch_views(const katsevich_plan *plan, int32_t pitch, int64_t *first_view, int32_t *n_views);

/* Union of the views needed by pitches [first_pitch, first_pitch + n_pitches). */
int katsevich_scan_views(const katsevich_plan *plan, int32_t first_pitch, int32_t n_pitches,
                         int64_t *first_view, int64_t *n_views);

/* Device workspace bytes for katsevich_reconstruct over n_pitches pitches
 * (and for katsevich_reconstruct_batch with B = n_pitches slabs). */
int katsevich_workspace_bytes(const katsevich_plan *plan, int32_t n_pitches, size_t *bytes);

/* Workspace bytes for katsevich_reconstruct_host (adds device sinogram + volume). */
int katsevich_workspace_bytes_host(const katsevich_plan *plan, int32_t n_pitches, size_t *bytes);

/* Reconstruction step for pitches [first_pitch,
 * first_pitch + n_pitches) of a helical scan.  `sino` (device) holds views
 * [sino_first_view, sino_first_view + sino_n_views) as g[v][m][l]; `vol`
 * (device) receives f[(k-first_pitch)·nz + j][iy][ix].  Steps 1-6 run once per
 * needed view (the filtered view is pitch-independent), then the PI-limited
 * backprojection runs pitch by pitch with the periodic tables.
 * KATS_ERR_COVERAGE if the sinogram misses a needed view. */
int katsevich_reconstruct(katsevich_plan *plan, const float *sino, int64_t sino_first_view, int64_t sino_n_views,
                          int32_t first_pitch, int32_t n_pitches, float *vol,
                          void *workspace, size_t workspace_bytes, void *cuda_stream);

/* katsevich_reconstruct whose backprojection runs in n_groups launches over consecutive pitch
 * groups (group i = pitches first_pitch + [n_pitches*i/n_groups, n_pitches*(i+1)/n_groups)), after
 * one filter pass over the union of the views.  If group_done is not NULL, group_done[i] (a
 * caller-created cudaEvent_t, or NULL to skip) is recorded on cuda_stream once group i's volume
 * slices are written, so a consumer on another stream — e.g. the NCCL send of finished pitch slabs
 * in a pitch-sharded run (SURVEY §8(e), P:l.246, l.265) — overlaps the remaining groups.
 * Results equal katsevich_reconstruct's bit for bit.  1 <= n_groups <= n_pitches
 * (KATS_ERR_ARGUMENT otherwise). */
int katsevich_reconstruct_grouped(katsevich_plan *plan, const float *sino, int64_t sino_first_view,
                                  int64_t sino_n_views, int32_t first_pitch, int32_t n_pitches, float *vol,
                                  void *workspace, size_t workspace_bytes, void *cuda_stream,
                                  int32_t n_groups, void **group_done);

/* B independent one-pitch slabs (the network's embedded layer, P:l.284-286):
 * slabs [B][n_views][rows][cols] (device), each holding pitch 0's views
 * katsevich_pitch_views(plan, 0, ...); vols [B][nz][ny][nx] (device). */
int katsevich_reconstruct_batch(katsevich_plan *plan, const float *slabs, int32_t B, float *vols,
                                void *workspace, size_t workspace_bytes, void *cuda_stream);

/* Workspace bytes for katsevich_reconstruct_batch_host (adds the device slabs and volumes). */
int katsevich_workspace_bytes_batch_host(const katsevich_plan *plan, int32_t B, size_t *bytes);

/* katsevich_reconstruct_batch with HOST slabs [B][n_views][rows][cols] and volumes [B][nz][ny][nx]:
 * the batch runs in groups of slabs whose host->device copies, filtering, backprojection and
 * device->host copies overlap on separate streams (the paper's training layer fed from host
 * memory, P:l.284-304).  Synchronises `cuda_stream` before returning; pinned host memory gives
 * asynchronous copies.  Same results as katsevich_reconstruct_batch. */
int katsevich_reconstruct_batch_host(katsevich_plan *plan, const float *host_slabs, int32_t B, float *host_vols,
                                     void *workspace, size_t workspace_bytes, void *cuda_stream);

/* katsevich_reconstruct with HOST sinogram and volume: copies the needed
 * views host->device, reconstructs and copies the volume device->host inside
 * the call (synchronises `cuda_stream` before returning).  Pinned host
 * memory gives asynchronous, overlapped copies; pageable memory works. */
int katsevich_reconstruct_host(katsevich_plan *plan, const float *host_sino, int64_t sino_first_view, int64_t sino_n_views,
                               int32_t first_pitch, int32_t n_pitches, float *host_vol,
                               void *workspace, size_t workspace_bytes, void *cuda_stream);

/* ---- adjoint (NEXT-1: training through the layer) ---- */

/* Workspace for katsevich_adjoint: katsevich_workspace_bytes plus one fp32
 * detector image per filtered view of the union. */
int katsevich_adjoint_workspace_bytes(const katsevich_plan *plan, int32_t n_pitches, size_t *bytes);

/* Adjoint (transpose) of katsevich_reconstruct's linear map sinogram -> volume
 * (the layer the paper trains through, P:l.303).
 *   vol       [n_pitches*nz][ny][nx] fp32, device (input)
 *   sino_out  [sn][rows][cols] fp32, device, first view s0 (output, overwritten;
 *             0 outside the pitches' slabs); must cover views
 *             k*views_per_turn + bp_lo - 1 .. k*views_per_turn + bp_hi + 1 for
 *             every requested pitch k (KATS_ERR_COVERAGE otherwise)
 * Steps in reverse: step 7^T (quad adjoints, per-CTA shared-memory
 * accumulation + red.global.add), then per view the transposes of steps 6..1.
 * fp32, summation order not fixed (atomics): results are reproducible to
 * rounding, not bitwise.  Asynchronous on cuda_stream. */
int katsevich_adjoint(katsevich_plan *plan, const float *vol, int32_t first_pitch, int32_t n_pitches,
                      float *sino_out, int64_t s0, int64_t sn, void *workspace, size_t workspace_bytes,
                      void *cuda_stream);

/* Workspace for katsevich_adjoint_batch. */
int katsevich_adjoint_batch_workspace_bytes(const katsevich_plan *plan, int32_t B, size_t *bytes);

/* Adjoint of katsevich_reconstruct_batch (the training-shaped workload: B
 * independent one-pitch slabs, the layer the paper trains through):
 *   vols       [B][nz][ny][nx] fp32, device (input)
 *   slabs_out  [B][n_slab][rows][cols] fp32, device (output, overwritten), n_slab
 *              as katsevich_pitch_views reports for pitch 0 (each slab with its
 *              own +-1 halo).  Asynchronous; reproducible to rounding. */
int katsevich_adjoint_batch(katsevich_plan *plan, const float *vols, int32_t B, float *slabs_out, void *workspace,
                            size_t workspace_bytes, void *cuda_stream);

/* ---- data generation (NEXT-3: training-shaped inputs) ---- */

/* Exact line integrals of an ellipsoid phantom along the plan's helical scan
 * rays (helix P:l.87-94, curved detector P:l.117, l.311-349) for views
 * first_view .. first_view+n_views-1.
 *   ell   [n_ell][8] double, HOST: {cx, cy, cz, a, b, c, phi, rho} (mm, rad,
 *         density; c <= 0: infinite elliptic cylinder along z; densities add)
 *   sino  [n_views][rows][cols] fp32, device (output)
 * fp64 chords (closed-form quadratic); asynchronous on cuda_stream. */
int katsevich_project_ellipsoids(katsevich_plan *plan, const double *ell, int32_t n_ell, int64_t first_view,
                                 int64_t n_views, float *sino, void *cuda_stream);

/* Sampled line integrals of a voxel volume (P:l.354, "simulate scanning the CT
 * image labels"): vol [nz_vol][ny][nx] fp32, device, on the plan's x/y grid
 * (x_i = (i - nx/2) dx) with slices z_j = z_first + j dz_vol; trilinear
 * interpolation (0 outside the grid), N = ceil(length / (0.5 min voxel)) equal
 * steps sampled at their midpoints.  n_truncated (host, optional: synchronises)
 * receives the number of rays whose x/y segment leaves the volume's z extent. */
int katsevich_project_volume(katsevich_plan *plan, const float *vol, int32_t nz_vol, double z_first, double dz_vol,
                             int64_t first_view, int64_t n_views, float *sino, int64_t *n_truncated,
                             void *cuda_stream);

/* Sparse-view degradation of P:l.394-404 on a sinogram of views first_view ..
 * (device fp32 in / out [n_views][rows][cols]): keep the α columns 0,
 * alpha_stride, ... and interpolate linearly back (last kept value held
 * beyond it); then the 'Gaussian+Poisson' noise with M = max of the upsampled
 * data (computed on the device): t = I0 exp(-g/M), s = Poisson(t) +
 * Normal(0, gauss_var), s = max(s, 1), out = log(I0/s) M.  Random numbers:
 * Philox4x32-10 keyed by (seed, absolute sample index) — deterministic and
 * independent of chunking.  mode 1: noiseless check (Poisson -> its mean,
 * var 0).  counts (device int64, optional) receives the Poisson draws; M_out
 * (device fp32, optional) the M used.  Input must be >= 0 (KATS_ERR_ARGUMENT
 * for bad parameters). */
int katsevich_degrade(katsevich_plan *plan, const float *sino, int64_t first_view, int64_t n_views,
                      int32_t alpha_stride, double I0, double gauss_var, uint64_t seed, int32_t mode, float *out,
                      int64_t *counts, float *M_out, void *cuda_stream);

/* ---- debug / parity entry points ---- */

/* Steps 1-6 (Eqs. 8-15) for views [out_first_view, out_first_view + n_out):
 * gF [n_out][rows][cols] (device, required); g3 and g4 [n_out][n_psi][cols]
 * (device, optional: NULL to skip).  The sinogram must hold views
 * out_first_view-1 .. out_first_view+n_out. */
int katsevich_filter(katsevich_plan *plan, const float *sino, int64_t sino_first_view, int64_t sino_n_views,
                     int64_t out_first_view, int32_t n_out, float *g3, float *g4, float *gF, void *cuda_stream);

/* Step 7 for pitch `pitch` from filtered views gF [gF_n_views][rows][cols]
 * (device) whose first view is gF_first_view; vol [nz][ny][nx] (device). */
int katsevich_backproject(katsevich_plan *plan, const float *gF, int64_t gF_first_view, int64_t gF_n_views,
                          int32_t pitch, float *vol, void *cuda_stream);

/* Sizes of the periodic tables: n_psi; T_pi view range of pitch 0 [bp_lo, bp_hi]. */
int katsevich_table_info(const katsevich_plan *plan, int32_t *n_psi, int64_t *bp_view_lo, int64_t *bp_view_hi);

/* Copy the host tables (any pointer may be NULL):
 *   pi_first, pi_last  [nz][ny][nx] int32, pitch-0 view indices (empty voxel: first=0, last=-1)
 *   w_first, w_last    [nz][ny][nx] double, fractional end weights
 *   fr_idx, fr_frac    [n_psi][n_cols] int32/double  (-1: outside the rows)
 *   br_idx, br_frac    [n_rows][n_cols] int32/double (-1: no root / outside the ψ grid) */
int katsevich_export_tables(const katsevich_plan *plan, int32_t *pi_first, int32_t *pi_last,
                            double *w_first, double *w_last, int32_t *fr_idx, double *fr_frac,
                            int32_t *br_idx, double *br_frac);

/* Tensor-core Hilbert taps (Eq. 12 on the tcgen05 tensor cores, DESIGN.md §5 "Hankel tap cores"):
 * fill out[] (host memory, out_floats >= 64 * NH with NH = 32 * ceil(ceil(n_cols / 2) / 32)) with
 * the layout k_hilbert_hk / k_hilbert_ws load into shared memory: [parity 2][hi, lo][NH/2 cores]
 * [8 rows][4], core s row r column c = the TF32 hi part / fp32 remainder of the tap
 * taps[2 (n - k) + 2 parity - 1 + n_cols - 1] with n + k' = 4 s + r + c, k = NH - 1 - k' (0 where
 * that offset is outside the 2 n_cols - 1 taps).  taps: host, [2 n_cols - 1], K[d] at d + n_cols - 1.
 * Pure host function (no plan, no device).  KATS_ERR_ARGUMENT if out_floats is too small. */
int katsevich_hilbert_hk_table(int32_t n_cols, const float *taps, float *out, size_t out_floats);

/* ---- in-run kernel timing (CUDA events on the launching stream) ---- */

/* Per-stage statistics accumulated while profiling is enabled. */
typedef struct {
    int64_t launches[6];     /* 0: K12 deriv+length weight+forward rebin, 1: K3 Hilbert,
                                2: K4 backward rebin+cos, 3: K5 backprojection, 4: end-weight fix-up, 5: other */
    double  ms[6];           /* summed CUDA-event durations per stage */
    double  busy_ms[6];      /* union of the stage's launch intervals (launches overlapping on
                                different streams count once), per profile_read batch */
    int64_t total_launches;  /* all kernel launches issued by the plan since the last reset (always counted) */
} katsevich_stats;

int katsevich_profile_enable(katsevich_plan *plan, int enable);   /* 1: record events around each launch */
int katsevich_profile_read(katsevich_plan *plan, katsevich_stats *out, int reset); /* synchronises recorded events */

/* ---- which backprojection kernel ran ---- */

/* Variant of the most recent step-7 (K5) launch of this plan: 0 none yet,
 * KATS_BP_L1 (chunked kernel, global-memory reads; used for plans whose
 * footprints leave the detector), KATS_BP_WINDOW (register sliding window),
 * KATS_BP_TMEM (tensor-memory sliding window, the default), KATS_BP_ITEMS (batches whose windows
 * hold <= 8 slices, e.g. the paper's 16-slab training batch: the CTA's slabs share each view's
 * geometry).  The environment variables KATS_BP_KERNEL=window|l1 and KATS_BP_ITEMS=0|N force variants
 * for A/B tests. */
#define KATS_BP_L1 1
#define KATS_BP_WINDOW 2
#define KATS_BP_TMEM 3
#define KATS_BP_ITEMS 4   /* batches of narrow-window slabs (C5): per-view geometry shared by the CTA's slabs */
int katsevich_bp_kernel(const katsevich_plan *plan);

void katsevich_destroy(katsevich_plan *plan);
const char *katsevich_error_string(int code);
const char *katsevich_last_error_detail(const katsevich_plan *plan);

#ifdef __cplusplus
}
#endif
#endif /* KATSEVICH_H */
