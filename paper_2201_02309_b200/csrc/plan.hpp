// plan.hpp — internal plan of the B200 Katsevich library (not part of the ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

#include "../../include/katsevich.h"

namespace kats {

constexpr double kPi = 3.14159265358979323846;

// Backprojection work decomposition (backproject.cu): a CTA owns a TILE_X x TILE_Y
// tile of (x, y) columns and a chunk of CHUNK_Z slices.
constexpr int kTileX = 16, kTileY = 16, kChunkZ = 16;

// Host-side periodic tables (double precision, pitch 0).
struct HostTables {
    int32_t n_psi = 0;
    double dlam = 0, h = 0, r_fov = 0, alpha_m = 0, psi_max = 0, dpsi = 0, kappa = 0;
    // T_pi per voxel [nz][ny][nx], pitch-relative view indices
    std::vector<int32_t> pi_first, pi_last;
    std::vector<double> w_first, w_last;
    int64_t bp_lo = 0, bp_hi = -1;          // min k_first / max k_last over the pitch
    // T_fr [n_psi][n_cols], T_br [n_rows][n_cols]
    std::vector<int32_t> fr_idx, br_idx;
    std::vector<double> fr_frac, br_frac;
    bool td_covered = true;
    double w_L = 0;                         // max |w*| over grid views inside PI windows (P:l.336)
    bool interior_in_detector = false;      // interior BP samples provably inside rows and columns (fp32 margin)
    int32_t fp_cols = 0, fp_rows = 0;       // quad box (columns x quad rows) covering any CTA's interior samples of one view
    int32_t max_active = 0;                 // max slices of one column whose interior windows share a view
    bool windows_monotone = false;          // per column: k_first, k_last nondecreasing in z, interior windows non-empty
    bool br_monotone = false;               // per column: T_br's κ-line index nondecreasing in the row (K4^T streams)
    int32_t fp_cols_column = 0;             // quad columns covering a tile's full-column samples of one view
    int32_t warp_span = 0;                  // max live slices of one warp (8x4 columns): newest open .. oldest unflushed
    int32_t warp_span2 = 0;                 // same for two consecutive views done together: open at k+1 .. unflushed at k
};

// Per-view geometry for the backprojection (pitch-relative view k in [bp_lo, bp_hi]).
struct ViewGeom { float c, s, zc, pad; };    // cos(λ'+λ0), sin(λ'+λ0), z0 + hλ'

struct RebinEntry { int32_t idx; float frac; };

struct DeviceTables {
    int2 *pi_k = nullptr;          // (k_first, k_last) per voxel [nz][ny][nx]
    float2 *pi_w = nullptr;        // (ω_first, ω_last)
    ViewGeom *view = nullptr;      // [bp_hi - bp_lo + 1]
    RebinEntry *fr = nullptr;      // [n_psi][n_cols]
    RebinEntry *br = nullptr;      // [n_rows][n_cols]
    float *cos_alpha = nullptr;    // [n_cols]
    float *wlen = nullptr;         // [n_rows]  D / sqrt(D² + w²)
    float *hilbert = nullptr;      // [2 n_cols - 1]  K[d], d = -(nc-1)..nc-1
    float *hilbert_tc = nullptr;   // K3 tensor-core tap matrices (hi/lo TF32 split, UMMA layout)
    float *hilbert_hk = nullptr;   // K3 tensor-core Hankel tap cores (hi/lo TF32 split)
    int *tile_order = nullptr;     // step-7 column tiles (16x16), heaviest first (ty * ntx + tx)
    float *flat_a = nullptr;       // KATS_FLAG_FLAT: u_l / D per column
};

struct ProfRecord { int stage; void *ev0; void *ev1; };

}  // namespace kats

struct katsevich_plan {
    katsevich_geometry g{};                 // effective geometry of the filtered grid (tables, kernels)
    katsevich_geometry graw{};              // the caller's geometry (raw sinogram, data generation)
    bool half = false;                      // NEXT-4: Noo's half-sample derivative (g = half-shifted grid)
    int device = -1;
    bool precomputed = false;
    kats::HostTables t;
    kats::DeviceTables d;
    std::string detail;
    // profiling
    bool profiling = false;
    std::vector<kats::ProfRecord> prof;
    std::vector<void *> event_pool;
    int64_t total_launches = 0;
    int last_bp_kernel = 0;                 // KATS_BP_* variant of the last K5 launch
    int64_t stage_launches[6] = {0, 0, 0, 0, 0, 0};
    double stage_ms[6] = {0, 0, 0, 0, 0, 0};
    double stage_busy_ms[6] = {0, 0, 0, 0, 0, 0};
    // host entry point: copy stream + sync events (created on first use)
    void *copy_stream = nullptr;            // host->device
    void *copy_stream2 = nullptr;           // device->host
    void *bp_streams[2] = {nullptr, nullptr};  // alternating per-pitch backprojection streams (low priority)
    void *filter_stream = nullptr;          // filter chunks (highest priority)
    void *filter_xs[2] = {nullptr, nullptr};     // device entry points: extra filter-chunk streams
    void *fork_events[3] = {nullptr, nullptr, nullptr};  // fork / joins of filter_xs
    void *dg_scratch = nullptr;             // data generation: phantom / counter / upsampled scratch
    size_t dg_scratch_bytes = 0;
    std::vector<void *> sync_events;
};

namespace kats {
// precompute.cpp
int validate(const katsevich_geometry &g, std::string &detail);
int compute_host_tables(const katsevich_geometry &g, HostTables &t, std::string &detail);
katsevich_geometry half_sample_geometry(const katsevich_geometry &g);   // DESIGN.md reading A25
}  // namespace kats
