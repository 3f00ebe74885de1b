// api.cu — the C ABI declared in include/katsevich.h.
//
// Host plumbing only: argument checking, device table upload, workspace
// carving, launch sequencing and optional CUDA-event timing.  Every step of
// the method runs in the kernels of filter.cu / backproject.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "kernels.cuh"

using namespace kats;

namespace kats {

// cudaFuncAttributeMaxDynamicSharedMemorySize is per device context: remember, per (kernel, device),
// the largest opt-in made (a second plan on another device in the same process must opt in again)
cudaError_t smem_opt_in(const void *kernel, size_t bytes)
{
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t &have = done[{kernel, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

int device_sms()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    static std::mutex mu;
    static std::map<int, int> sms;
    std::lock_guard<std::mutex> lk(mu);
    auto it = sms.find(dev);
    if (it != sms.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    sms[dev] = n;
    return n;
}

}  // namespace kats

namespace {

// Base views per filter chunk: 256 keeps a wide-κ chunk's g3/g4 L2-resident (C4: 2 x 24 MB); with few
// κ-lines a chunk grows so the tensor-core Hilbert launch has enough CTAs to hide its per-CTA latency.
// The device entry points (katsevich_reconstruct, _batch, the adjoints) take chunks
// device_chunk_mul() times larger; the host-staged path keeps the base chunk (its H2D copy is
// pipelined per chunk).
static int filter_chunk_views(const katsevich_plan *p, int mul = 1)
{
    return mul * 256 * std::max(1, 128 / std::max(1, p->t.n_psi));
}
// KATS_FILTER_CHUNK_MUL (A/B tests; read once per process so workspace sizing and use agree).
// Default 4 (scripts/ab/gpu_fchunk.sh, two runs each: C5 4.21 -> 4.14 ms, C3 9.25 -> 9.12 ms,
// C2 1.73 -> 1.71 ms, C4 50.85 -> 50.78 ms; fewer, fuller K3 launches outweigh L2 residency)
static int device_chunk_mul()
{
    static const int mul = [] {
        const char *e = std::getenv("KATS_FILTER_CHUNK_MUL");
        return e ? std::max(1, std::min(64, std::atoi(e))) : 4;
    }();
    return mul;
}
// Filter chunks in flight at once on the device entry points (one chunk scratch each; run_filter)
constexpr int kFilterStreamsMax = 2;   // 3 measured no faster (C4 51.0 vs 50.8 ms, C5 equal)

enum Stage { ST_K12 = 0, ST_K3 = 1, ST_K4 = 2, ST_K5 = 3, ST_FIX = 4, ST_OTHER = 5 };

int cuda_fail(katsevich_plan *p, cudaError_t e, const char *where)
{
    if (p) {
        p->detail = std::string(where) + ": " + cudaGetErrorString(e);
    }
    return KATS_ERR_CUDA;
}

int hilbert_fail(katsevich_plan *p)
{
    p->detail = "K3: cuTensorMapEncodeTiled failed for the Hilbert input lines (Hilbert not run)";
    return KATS_ERR_CUDA;
}

#define KCHECK(p, call)                                          \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) return cuda_fail((p), _e, #call); \
    } while (0)

// Records CUDA events around one launch when profiling is on; counts launches.
struct LaunchScope {
    katsevich_plan *p;
    int stage;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    LaunchScope(katsevich_plan *p_, int st, cudaStream_t s_) : p(p_), stage(st), s(s_)
    {
        p->total_launches++;
        p->stage_launches[stage]++;
        if (p->profiling) {
            e0 = take(); e1 = take();
            cudaEventRecord(e0, s);
        }
    }
    cudaEvent_t take()
    {
        if (!p->event_pool.empty()) {
            cudaEvent_t e = (cudaEvent_t)p->event_pool.back();
            p->event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    ~LaunchScope()
    {
        if (e0) {
            cudaEventRecord(e1, s);
            p->prof.push_back({stage, (void *)e0, (void *)e1});
        }
    }
};

// table upload on the caller's stream; the sources are pageable vectors, whose H2D copies return once
// the data is staged, so a vector may go out of scope before the stream reaches the copy
// (katsevich_precompute synchronises the stream at the end)
template <typename T>
int upload(katsevich_plan *p, T **dst, const std::vector<T> &src, cudaStream_t s)
{
    if (src.empty()) { *dst = nullptr; return KATS_OK; }
    KCHECK(p, cudaMalloc((void **)dst, sizeof(T) * src.size()));
    KCHECK(p, cudaMemcpyAsync(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
    return KATS_OK;
}

void free_device(katsevich_plan *p)
{
    if (p->device < 0) return;
    cudaSetDevice(p->device);
    void *ptrs[] = {p->d.pi_k, p->d.pi_w, p->d.view, p->d.fr, p->d.br, p->d.cos_alpha, p->d.wlen, p->d.hilbert,
                    p->d.hilbert_tc, p->d.hilbert_hk, p->d.tile_order, p->d.flat_a};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    p->d = DeviceTables{};
    for (auto &r : p->prof) { cudaEventDestroy((cudaEvent_t)r.ev0); cudaEventDestroy((cudaEvent_t)r.ev1); }
    p->prof.clear();
    for (void *e : p->event_pool) cudaEventDestroy((cudaEvent_t)e);
    p->event_pool.clear();
    for (void *e : p->sync_events) cudaEventDestroy((cudaEvent_t)e);
    p->sync_events.clear();
    if (p->dg_scratch) { cudaFree(p->dg_scratch); p->dg_scratch = nullptr; p->dg_scratch_bytes = 0; }
    if (p->copy_stream) { cudaStreamDestroy((cudaStream_t)p->copy_stream); p->copy_stream = nullptr; }
    if (p->copy_stream2) { cudaStreamDestroy((cudaStream_t)p->copy_stream2); p->copy_stream2 = nullptr; }
    for (void *&b : p->bp_streams)
        if (b) { cudaStreamDestroy((cudaStream_t)b); b = nullptr; }
    if (p->filter_stream) { cudaStreamDestroy((cudaStream_t)p->filter_stream); p->filter_stream = nullptr; }
    for (void *&x : p->filter_xs)
        if (x) { cudaStreamDestroy((cudaStream_t)x); x = nullptr; }
    for (void *&e : p->fork_events)
        if (e) { cudaEventDestroy((cudaEvent_t)e); e = nullptr; }
}

int64_t n_union_views(const katsevich_plan *p, int32_t n_pitches)
{
    const HostTables &t = p->t;
    return (int64_t)(n_pitches - 1) * p->g.views_per_turn + (t.bp_hi - t.bp_lo + 1);
}

// raw sinogram views: the caller's detector; filtered view u needs raw views u - halo_lo(p) .. u + 1
// (centred λ difference; the half-sample derivative reads u and u + 1)
size_t raw_view_elems(const katsevich_plan *p) { return (size_t)p->graw.n_rows * p->graw.n_cols; }
int halo_lo(const katsevich_plan *p) { return p->half ? 0 : 1; }

size_t chunk_bytes_views(const katsevich_plan *p, int64_t views)
{
    return 2 * sizeof(float) * (size_t)views * p->t.n_psi * g3_line_pitch(p->g.n_cols);
}
size_t filter_chunk_bytes(const katsevich_plan *p, int mul = 1) { return chunk_bytes_views(p, filter_chunk_views(p, mul)); }

// Filter chunk of the batch entry point: the batch's filtered views in an even number of equal chunks
// of at most 8 base chunks, alternating over the two filter streams (C5: two chunks of 4640 views, step
// 3.675 -> 3.59 ms against 3072-view chunks; scripts/ab/gpu_fchunk_c5.sh); KATS_BATCH_CHUNK=0 keeps
// the device chunk
static int64_t batch_chunk_views(const katsevich_plan *p, int32_t B)
{
    static const bool off = [] { const char *e = std::getenv("KATS_BATCH_CHUNK"); return e && e[0] == '0'; }();
    const int64_t dev = filter_chunk_views(p, device_chunk_mul());
    if (off) return dev;
    const int64_t nb = (p->t.bp_hi - p->t.bp_lo + 1) * (int64_t)B, cap = 8 * (int64_t)filter_chunk_views(p, 1);
    const int64_t k = (nb + 2 * cap - 1) / (2 * cap);
    return std::max<int64_t>(1, (nb + 2 * k - 1) / (2 * k));
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// filtered view as tap quads: (n_rows + 2) x n_cols float4 (two zero rows below)
size_t quad_view_elems(const katsevich_plan *p) { return (size_t)(p->g.n_rows + 2) * p->g.n_cols; }

FilterParams filter_params(const katsevich_plan *p)
{
    FilterParams f{};
    f.nr = p->g.n_rows; f.nc = p->g.n_cols; f.npsi = p->t.n_psi;
    f.inv_2dlam = (float)(1.0 / (2.0 * p->t.dlam));
    f.inv_dalpha = (float)(1.0 / p->g.d_alpha);
    f.inv_2dalpha = (float)(1.0 / (2.0 * p->g.d_alpha));
    f.wlen = p->d.wlen; f.fr = p->d.fr; f.br = p->d.br;
    f.cos_alpha = p->d.cos_alpha; f.hilbert = p->d.hilbert; f.hilbert_tc = p->d.hilbert_tc;
    f.hilbert_hk = p->d.hilbert_hk;
    f.sign = 1.f;
    f.half = p->half ? 1 : 0;
    f.apod = (p->g.flags & KATS_FLAG_HANN) ? 1 : 0;
    f.flat = (p->g.flags & KATS_FLAG_FLAT) ? 1 : 0;
    f.flat_a = p->d.flat_a;
    f.D = (float)p->g.D;
    f.dw_over_D = (float)(p->g.d_w / p->g.D);
    f.inv_dw = (float)(1.0 / p->g.d_w);
    f.inv_2dw = (float)(0.5 / p->g.d_w);
    f.br_monotone = p->t.br_monotone ? 1 : 0;
    return f;
}

// Filter-chunk streams of the device entry points: chunk c runs on stream c mod n into scratch
// c mod n (n = KATS_FILTER_STREAMS, default 2, at most kFilterStreamsMax; the extra streams are
// created on first use).  Returns n (1 if a stream cannot be created).
static int filter_streams(katsevich_plan *p)
{
    const char *e = std::getenv("KATS_FILTER_STREAMS");
    const int n = std::max(1, std::min(kFilterStreamsMax, e ? std::atoi(e) : 2));
    for (int i = 0; i + 1 < n; ++i)
        if (!p->filter_xs[i]) {
            cudaStream_t c;
            if (cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking) != cudaSuccess) return 1;
            p->filter_xs[i] = c;
        }
    for (void *&ev : p->fork_events)
        if (!ev) {
            cudaEvent_t x;
            if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) return 1;
            ev = x;
        }
    return n;
}

// Filter n_out views whose raw data (with ±1 halo) is at sino_v0 - rows*cols
// .. ; writes gF (and optionally full g3/g4 when dbg3/dbg4 are given).
// With multi (kFilterStreamsMax chunk scratches, each filter_chunk_bytes apart from scratch) and
// no debug outputs, chunks alternate over filter_streams() streams and scratches, so one chunk's
// latency-bound K12 overlaps another's K3 / K4 (chunks write disjoint views of gq; the caller's
// stream waits for all of them at the end).  C5 4.75 -> 4.31 ms per step with two streams.
int run_filter(katsevich_plan *p, const float *raw_first_out, int64_t n_out, float4 *gq,
               float *scratch, float *dbg3, float *dbg4, float *dbgF, cudaStream_t s, bool overlapped = false,
               int64_t slab_views = 0, bool multi = false, int chunk_mul = 1, int64_t chunk_views = 0)
{
    FilterParams f = filter_params(p);
    // running concurrently with the TMEM backprojection: K3 uses the fp32 direct convolution
    // (launch_hilbert); results then agree with the device path to fp32 rounding, not bitwise
    // the host path's filter beside the pitch-pair backprojection (2 CTAs per SM) keeps the tensor-core
    // K3: C4 e2e 51.91 -> 51.23 ms, C2 3.07 -> 2.75 ms (scripts/ab/gpu_r02p.sh); KATS_HOST_TC=0: the fp32
    // direct K3 there (the round-1 choice next to three one-pitch TMEM CTAs per SM)
    static const bool host_tc = [] { const char *e = std::getenv("KATS_HOST_TC"); return !(e && e[0] == '0'); }();
    f.hilbert_overlap = overlapped && !host_tc ? 1 : 0;
    f.hp = g3_half_pitch(p->g.n_cols);
    f.k3_in_split = hilbert_split_input(f) ? 1 : 0;         // K12 writes the lines the chosen K3 reads
    const size_t rs = (size_t)p->g.n_rows * p->g.n_cols;
    const size_t qs = quad_view_elems(p);
    const size_t ps_dbg = (size_t)p->t.n_psi * p->g.n_cols;              // debug stage arrays: plain lines
    const size_t ps = (size_t)p->t.n_psi * g3_line_pitch(p->g.n_cols);  // scratch lines
    const int64_t kFilterChunk = chunk_views > 0 ? chunk_views : filter_chunk_views(p, chunk_mul);
    const int64_t nchunks = (n_out + kFilterChunk - 1) / kFilterChunk;
    const int ns = multi && !dbg3 && !dbg4 && !dbgF ? (int)std::min<int64_t>(filter_streams(p), nchunks) : 1;
    cudaStream_t st[kFilterStreamsMax] = {s};
    for (int i = 1; i < ns; ++i) st[i] = (cudaStream_t)p->filter_xs[i - 1];
    if (ns > 1) {
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->fork_events[0], s));
        for (int i = 1; i < ns; ++i) KCHECK(p, cudaStreamWaitEvent(st[i], (cudaEvent_t)p->fork_events[0], 0));
    }
    const size_t chunk_floats = align_up(chunk_bytes_views(p, kFilterChunk)) / sizeof(float);
    for (int64_t v0 = 0; v0 < n_out; v0 += kFilterChunk) {
        const int nv = (int)std::min<int64_t>(kFilterChunk, n_out - v0);
        const int c = (int)((v0 / kFilterChunk) % ns);
        s = st[c];
        f.sino = raw_first_out;                                    // K12 maps view0 + v to its raw view
        f.view0 = v0;
        f.slab_views = slab_views;
        f.n_views = nv;
        f.g3 = scratch + c * chunk_floats;
        f.g4 = dbg4 ? dbg4 + v0 * ps_dbg : f.g3 + (size_t)kFilterChunk * ps;
        f.gq = gq + v0 * qs;
        f.gF = dbgF ? dbgF + v0 * rs : nullptr;
        if (dbg3) {                                                // debug: g3 as plain lines too
            FilterParams d = f;
            d.k3_in_split = 0;
            d.g3 = dbg3 + v0 * ps_dbg;
            { LaunchScope ls(p, ST_K12, s); launch_deriv_fwd_rebin(d, s); }
            KCHECK(p, cudaGetLastError());
            if (!f.k3_in_split && !f.apod) f.g3 = d.g3;            // (apodised: K3's input is smoothed in place)
        }
        if (!dbg3 || f.k3_in_split || f.apod) {
            LaunchScope ls(p, ST_K12, s);
            launch_deriv_fwd_rebin(f, s);
        }
        KCHECK(p, cudaGetLastError());
        if (f.apod) {                                              // reading A26: K3's input lines smoothed
            { LaunchScope ls(p, ST_K3, s); launch_hann_smooth(f, f.g3, (int64_t)nv * f.npsi, f.k3_in_split, s); }
            KCHECK(p, cudaGetLastError());
        }
        { LaunchScope ls(p, ST_K3, s); if (launch_hilbert(f, s)) return hilbert_fail(p); }
        KCHECK(p, cudaGetLastError());
        { LaunchScope ls(p, ST_K4, s); launch_bwd_rebin_cos(f, s); }
        KCHECK(p, cudaGetLastError());
    }
    for (int i = 1; i < ns; ++i) {
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->fork_events[i], st[i]));
        KCHECK(p, cudaStreamWaitEvent(st[0], (cudaEvent_t)p->fork_events[i], 0));
    }
    return KATS_OK;
}

BPParams bp_params(const katsevich_plan *p)
{
    BPParams b{};
    const katsevich_geometry &g = p->g;
    b.nr = g.n_rows; b.nc = g.n_cols; b.nx = g.nx; b.ny = g.ny; b.nz = g.nz_per_pitch;
    b.colbytes = 16u * (unsigned)(g.n_rows + 2);
    b.viewbytes = 16 * (int64_t)quad_view_elems(p);
    b.pi_k = p->d.pi_k; b.pi_w = p->d.pi_w; b.view = p->d.view;
    {   // KATS_BP_ORDER=grid: plain 2-D tile grid (A/B tests)
        const char *e = std::getenv("KATS_BP_ORDER");
        b.tile_order = e && std::string(e) == "grid" ? nullptr : p->d.tile_order;
    }
    b.view_lo = (int)p->t.bp_lo;
    b.R = (float)g.R;
    b.D_over_dw = (float)(g.D / g.d_w);
    b.inv_dalpha = (float)(1.0 / g.d_alpha);
    b.col_c = (float)(0.5 * (g.n_cols - 1) - g.alpha_offset);
    b.row_c15 = (float)(0.5 * (g.n_rows - 1) + 1.5);   // quad row = row + 2, minus ½ for round-to-nearest
    b.colmax = (float)(g.n_cols - 1);
    b.rowmax = (float)(g.n_rows - 1);
    {
        const int c = (g.n_rows + 2) / 2;                      // quad centring row (must match K4)
        b.row_cc = b.row_c15 - (float)c;
        b.qmagic = 12582912.0f + (float)c;
        b.pm_lo = 1.5f - (float)c;
        b.pm_hi = b.rowmax + 1.5f - (float)c;
    }
    // minimax fit of atan(t) = t·Σ c_i t^(2i) on |t| <= 0.75 (max error 9.4e-9 rad), scaled by 1/Δα
    static const double c[7] = {0.99999980689595702, -0.33331974824996929, 0.19972144187876958,
                                -0.14029432575638814, 0.098575642092481805, -0.055588999310759703,
                                0.016795583727292406};
    for (int i = 0; i < 7; ++i) b.at[i] = (float)(c[i] / g.d_alpha);
    b.poly = std::tan(p->t.alpha_m) <= 0.75;
    b.uu = 1.f;
    if (g.flags & KATS_FLAG_FLAT) {          // flat (reading A27): u* / Δu = (D/Δu) (u/v*), w* = D (z - z_src)/v*
        for (int i = 0; i < 7; ++i) b.at[i] = 0.f;
        b.at[0] = (float)(g.D / g.d_alpha);
        b.poly = true;
        b.uu = 0.f;
    }
    b.checked = !p->t.interior_in_detector;
    b.fp_cols = p->t.fp_cols;
    b.max_cta_views = (int)(p->t.bp_hi - p->t.bp_lo + 1);
    b.fp_cols_column = p->t.fp_cols_column;
    b.max_active = p->t.max_active;
    b.windows_monotone = p->t.windows_monotone;
    {   // rows an inactive window entry (up to 3 slices above the top open one) can overshoot
        const double r_near = g.R - p->t.r_fov;
        const double step_max = g.D / (r_near * g.d_w) * (g.pitch / g.nz_per_pitch);
        b.tail_quads = 8 + (int)std::ceil(3.0 * step_max) + 2;
        // TMEM kernel: warp-union groups of one view / of two views
        b.pad_quads = 12 + (int)std::ceil((p->t.warp_span + 8) * step_max);
        b.pad_quads2 = 12 + (int)std::ceil((std::max(p->t.warp_span, p->t.warp_span2) + 8) * step_max);
    }
    {   // staged quad rows: interior samples have |w| <= w_L (the plan's margin check), i.e. quad rows
        // round(w/dw + (nr-1)/2 + 1.5); one row of slack either side for fp32 rounding (C3: 51 of 66)
        int q0 = 0, q1 = g.n_rows + 1;
        if (p->t.interior_in_detector) {
            const double cr = 0.5 * (g.n_rows - 1) + 1.5, hw = p->t.w_L / g.d_w;
            q0 = std::max(0, (int)std::floor(cr - hw) - 1);
            q1 = std::min(g.n_rows + 1, (int)std::ceil(cr + hw) + 1);
        }
        // staged column pitch: 3 or 5 (mod 8) quads, so lanes on neighbouring detector columns
        // (C3: ~1 column per voxel) read different 16-B bank groups; rows past the detector are TMA zero fill
        int nq = q1 - q0 + 1;
        while ((nq & 7) != 3 && (nq & 7) != 5) ++nq;
        if (2 * nq > 256) { q0 = 0; nq = g.n_rows + 2; }
        b.q_lo = q0;
        b.nq_s = nq;
        b.bp_items = 1;
    }
    {   // K5^T's int32 fixed-point box (backproject.cu k_bp_adjoint) holds <= 2^10 full-scale contributions
        // per (box column, quad row) cell of one view and lane-parity copy: bound the count by the tile
        // columns a detector column's ray strip can cover (a copy holds 128 of the 256) times the slices one
        // quad row can hold (the smallest row step per slice is at the far side of the FOV)
        const double vmax = g.R + p->t.r_fov;
        const double colw = vmax * g.d_alpha / ((g.flags & KATS_FLAG_FLAT) ? g.D : 1.0);   // a column's width at v*
        const double strip = std::ceil(colw / std::min(g.dx, g.dy) + 1.0) * std::ceil(16.0 * std::sqrt(2.0) + 1.0);
        const double step_min = g.D / (vmax * g.d_w) * (g.pitch / g.nz_per_pitch);
        b.adj_fixed_ok = std::min(128.0, strip) * (std::ceil(1.0 / step_min) + 1.0) <= 1024.0;
    }
    b.zero = 0u;
    b.warp_span = p->t.warp_span;
    b.warp_span2 = p->t.warp_span2;
    b.fp_rows = p->t.fp_rows;
    const char *ev = std::getenv("KATS_BP_KERNEL");          // "l1" forces the L1-path kernel (A/B tests)
    b.staged = !(ev && std::string(ev) == "l1");
    b.x0 = (float)(-0.5 * g.nx * g.dx); b.dx = (float)g.dx;
    b.y0 = (float)(-0.5 * g.ny * g.dy); b.dy = (float)g.dy;
    b.dz = (float)(g.pitch / g.nz_per_pitch);
    b.scale = (float)(p->t.dlam / (2.0 * kPi));      // +1/2π (P:l.157; A3)
    return b;
}

int check_device_plan(katsevich_plan *p)
{
    if (!p) return KATS_ERR_NULL;
    if (p->device < 0) { p->detail = "host-only plan"; return KATS_ERR_NO_DEVICE; }
    if (!p->precomputed) { p->detail = "katsevich_precompute has not run"; return KATS_ERR_NOT_PRECOMPUTED; }
    if (cudaSetDevice(p->device) != cudaSuccess) return cuda_fail(p, cudaGetLastError(), "cudaSetDevice");
    return KATS_OK;
}

}  // namespace

extern "C" {

int katsevich_plan_create(const katsevich_geometry *geom, int cuda_device, katsevich_plan **out)
{
    if (!out) return KATS_ERR_NULL;
    *out = nullptr;
    if (!geom) return KATS_ERR_NULL;
    std::string detail;
    int rc = validate(*geom, detail);
    if (rc != KATS_OK) return rc;
    if (cuda_device >= 0) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device >= n) return KATS_ERR_NO_DEVICE;
    }
    katsevich_plan *p = new (std::nothrow) katsevich_plan;
    if (!p) return KATS_ERR_ARGUMENT;
    p->graw = *geom;
    p->half = (geom->flags & KATS_FLAG_HALF_SAMPLE) != 0;
    p->g = p->half ? half_sample_geometry(*geom) : *geom;
    p->device = cuda_device;
    *out = p;
    return KATS_OK;
}

int katsevich_precompute(katsevich_plan *p, void *cuda_stream)
{
    if (!p) return KATS_ERR_NULL;
    cudaStream_t us = (cudaStream_t)cuda_stream;
    p->precomputed = false;
    int rc = compute_host_tables(p->g, p->t, p->detail);
    if (rc < 0) return rc;
    if (!p->t.td_covered && p->detail.empty())
        p->detail = "detector rows do not cover the Tam-Danielsson window";
    if (p->device >= 0) {
        KCHECK(p, cudaSetDevice(p->device));
        free_device(p);
        const katsevich_geometry &g = p->g;
        const HostTables &t = p->t;
        const size_t nvox = t.pi_first.size();
        std::vector<int2> pik(nvox);
        std::vector<float2> piw(nvox);
        for (size_t i = 0; i < nvox; ++i) {
            pik[i] = make_int2(t.pi_first[i], t.pi_last[i]);
            piw[i] = make_float2((float)t.w_first[i], (float)t.w_last[i]);
        }
        std::vector<ViewGeom> vg;
        for (int64_t k = t.bp_lo; k <= t.bp_hi; ++k) {
            double lam = (double)k * t.dlam;    // pitch-relative λ'
            vg.push_back({(float)std::cos(lam + g.lambda0), (float)std::sin(lam + g.lambda0),
                          (float)(g.z0 + t.h * lam), 0.f});
        }
        std::vector<RebinEntry> fr(t.fr_idx.size()), br(t.br_idx.size());
        for (size_t i = 0; i < fr.size(); ++i) fr[i] = {t.fr_idx[i], (float)t.fr_frac[i]};
        for (size_t i = 0; i < br.size(); ++i) br[i] = {t.br_idx[i], (float)t.br_frac[i]};
        const bool flat = (g.flags & KATS_FLAG_FLAT) != 0;
        std::vector<float> cosa(g.n_cols), wlen(g.n_rows), hk(2 * (size_t)g.n_cols - 1), fa(g.n_cols);
        for (int l = 0; l < g.n_cols; ++l) {
            const double a = ((double)l - 0.5 * (g.n_cols - 1) + g.alpha_offset) * g.d_alpha;
            cosa[l] = flat ? 1.f : (float)std::cos(a);                       // Eq. (15); flat: none (A27)
            fa[l] = flat ? (float)(a / g.D) : 0.f;
        }
        for (int m = 0; m < g.n_rows; ++m) {
            double w = ((double)m - 0.5 * (g.n_rows - 1)) * g.d_w;
            wlen[m] = (float)(g.D / std::sqrt(g.D * g.D + w * w));          // Eq. (9)
        }
        for (int d = -(g.n_cols - 1); d <= g.n_cols - 1; ++d) {            // reading A10 (flat: 1/(π(u-u')), A27)
            double kd = (d & 1) ? (flat ? 2.0 / (kPi * d) : 2.0 * g.d_alpha / (kPi * std::sin(d * g.d_alpha))) : 0.0;
            hk[(size_t)(d + g.n_cols - 1)] = (float)kd;
        }
        if (flat && (rc = upload(p, &p->d.flat_a, fa, us))) return rc;
        if ((rc = upload(p, &p->d.pi_k, pik, us)) || (rc = upload(p, &p->d.pi_w, piw, us)) ||
            (rc = upload(p, &p->d.view, vg, us)) || (rc = upload(p, &p->d.fr, fr, us)) ||
            (rc = upload(p, &p->d.br, br, us)) || (rc = upload(p, &p->d.cos_alpha, cosa, us)) ||
            (rc = upload(p, &p->d.wlen, wlen, us)) || (rc = upload(p, &p->d.hilbert, hk, us)))
            return rc;
        {   // step-7 tiles heaviest first (work ~ the tile's summed view span over its columns), so the
            // last wave of CTAs holds the lightest tiles (FOV edge)
            const int ntx = (g.nx + 15) / 16, nty = (g.ny + 15) / 16;
            const size_t plane = (size_t)g.nx * g.ny;
            std::vector<double> work((size_t)ntx * nty, 0.0);
            for (int iy = 0; iy < g.ny; ++iy)
                for (int ix = 0; ix < g.nx; ++ix) {
                    const size_t c = (size_t)iy * g.nx + ix;
                    if (t.pi_last[c] < t.pi_first[c]) continue;
                    work[(size_t)(iy / 16) * ntx + ix / 16] +=
                        (double)(t.pi_last[c + (size_t)(g.nz_per_pitch - 1) * plane] - t.pi_first[c]);
                }
            std::vector<int> order(work.size());
            for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
            if ((rc = upload(p, &p->d.tile_order, order, us))) return rc;
        }
        std::vector<float> htc;
        hilbert_tc_table(g.n_cols, hk.data(), htc);
        if ((rc = upload(p, &p->d.hilbert_tc, htc, us))) return rc;
        std::vector<float> hhk;
        hilbert_hk_table(g.n_cols, hk.data(), hhk);
        if ((rc = upload(p, &p->d.hilbert_hk, hhk, us))) return rc;
        KCHECK(p, cudaStreamSynchronize(us));
    }
    p->precomputed = true;
    if (const char *v = std::getenv("KATS_VERBOSE"); v && *v == '1')
        std::fprintf(stderr, "[katsevich] n_psi %d, bp views [%lld, %lld], w_L %.6f, interior_in_detector %d, "
                             "footprint box %d cols x %d quad rows, column box %d cols, max active slices %d, monotone %d, warp span %d (pairs %d)\n",
                     p->t.n_psi, (long long)p->t.bp_lo, (long long)p->t.bp_hi, p->t.w_L,
                     (int)p->t.interior_in_detector, p->t.fp_cols, p->t.fp_rows, p->t.fp_cols_column,
                     p->t.max_active, (int)p->t.windows_monotone, p->t.warp_span, p->t.warp_span2);
    return p->t.td_covered ? KATS_OK : KATS_WARN_TD_NOT_COVERED;
}

int katsevich_pitch_views(const katsevich_plan *p, int32_t pitch, int64_t *first_view, int32_t *n_views)
{
    if (!p || !first_view || !n_views) return KATS_ERR_NULL;
    if (!p->precomputed) return KATS_ERR_NOT_PRECOMPUTED;
    *first_view = (int64_t)pitch * p->g.views_per_turn + p->t.bp_lo - halo_lo(p);
    *n_views = (int32_t)(p->t.bp_hi - p->t.bp_lo + 2 + halo_lo(p));
    return KATS_OK;
}

int katsevich_scan_views(const katsevich_plan *p, int32_t first_pitch, int32_t n_pitches,
                         int64_t *first_view, int64_t *n_views)
{
    if (!p || !first_view || !n_views) return KATS_ERR_NULL;
    if (!p->precomputed) return KATS_ERR_NOT_PRECOMPUTED;
    if (n_pitches < 1) return KATS_ERR_ARGUMENT;
    *first_view = (int64_t)first_pitch * p->g.views_per_turn + p->t.bp_lo - halo_lo(p);
    *n_views = n_union_views(p, n_pitches) + 1 + halo_lo(p);
    return KATS_OK;
}

int katsevich_workspace_bytes(const katsevich_plan *p, int32_t n_pitches, size_t *bytes)
{
    if (!p || !bytes) return KATS_ERR_NULL;
    if (!p->precomputed) return KATS_ERR_NOT_PRECOMPUTED;
    if (n_pitches < 1) return KATS_ERR_ARGUMENT;
    const size_t qs = quad_view_elems(p);
    const int64_t nslab = p->t.bp_hi - p->t.bp_lo + 1;
    // reconstruct: filtered quads over the union of views; batch: per slab
    size_t gf = sizeof(float4) * qs * (size_t)std::max<int64_t>(n_union_views(p, n_pitches), nslab * n_pitches);
    // chunk scratches (run_filter): the device chunk, or the batch chunk of B = n_pitches slabs
    const size_t chunk = std::max(filter_chunk_bytes(p, device_chunk_mul()), chunk_bytes_views(p, batch_chunk_views(p, n_pitches)));
    *bytes = align_up(gf) + kFilterStreamsMax * align_up(chunk);
    return KATS_OK;
}

int katsevich_workspace_bytes_host(const katsevich_plan *p, int32_t n_pitches, size_t *bytes)
{
    int rc = katsevich_workspace_bytes(p, n_pitches, bytes);
    if (rc) return rc;
    const size_t rs = raw_view_elems(p);
    const size_t vol = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch * n_pitches;
    *bytes += align_up(sizeof(float) * rs * (size_t)(n_union_views(p, n_pitches) + 1 + halo_lo(p))) + align_up(sizeof(float) * vol);
    return KATS_OK;
}

int katsevich_adjoint_workspace_bytes(const katsevich_plan *p, int32_t n_pitches, size_t *bytes)
{
    int rc = katsevich_workspace_bytes(p, n_pitches, bytes);
    if (rc) return rc;
    const size_t rs = (size_t)p->g.n_rows * p->g.n_cols;
    *bytes += align_up(sizeof(float) * rs * (size_t)n_union_views(p, n_pitches));      // g1^T of every view
    return KATS_OK;
}

int katsevich_adjoint_batch_workspace_bytes(const katsevich_plan *p, int32_t B, size_t *bytes)
{
    int rc = katsevich_workspace_bytes(p, B, bytes);
    if (rc) return rc;
    const size_t rs = (size_t)p->g.n_rows * p->g.n_cols;
    *bytes += align_up(sizeof(float) * rs * (size_t)(p->t.bp_hi - p->t.bp_lo + 1) * B);   // g1^T of every view
    return KATS_OK;
}

// two low-priority streams for per-pitch backprojections and one highest-priority stream for
// the filter chunks that must finish before the next pitch's backprojection can start
static int ensure_bp_streams(katsevich_plan *p)
{
    int lo = 0, hi = 0;
    KCHECK(p, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (void *&b : p->bp_streams)
        if (!b) {
            cudaStream_t c;
            KCHECK(p, cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, lo));
            b = c;
        }
    if (!p->filter_stream) {
        cudaStream_t c;
        KCHECK(p, cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, hi));
        p->filter_stream = c;
    }
    return KATS_OK;
}

static int ensure_events(katsevich_plan *p, size_t n)
{
    while (p->sync_events.size() < n) {
        cudaEvent_t e;
        KCHECK(p, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->sync_events.push_back(e);
    }
    return KATS_OK;
}

int katsevich_reconstruct(katsevich_plan *p, const float *sino, int64_t s0, int64_t sn,
                          int32_t first_pitch, int32_t n_pitches, float *vol,
                          void *workspace, size_t workspace_bytes, void *cuda_stream)
{
    return katsevich_reconstruct_grouped(p, sino, s0, sn, first_pitch, n_pitches, vol, workspace, workspace_bytes,
                                         cuda_stream, 1, nullptr);
}

int katsevich_reconstruct_grouped(katsevich_plan *p, const float *sino, int64_t s0, int64_t sn,
                                  int32_t first_pitch, int32_t n_pitches, float *vol,
                                  void *workspace, size_t workspace_bytes, void *cuda_stream,
                                  int32_t n_groups, void **group_done)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    const int dm = device_chunk_mul();
    const int kFilterChunk = filter_chunk_views(p, dm);
    if (!sino || !vol || !workspace) return KATS_ERR_NULL;
    if (n_pitches < 1 || sn < 3 || n_groups < 1 || n_groups > n_pitches) return KATS_ERR_ARGUMENT;
    size_t need;
    katsevich_workspace_bytes(p, n_pitches, &need);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    const int vt = p->g.views_per_turn;
    const HostTables &t = p->t;
    const int64_t u0 = (int64_t)first_pitch * vt + t.bp_lo;                  // first filtered view
    const int64_t nu = n_union_views(p, n_pitches);
    if (u0 - halo_lo(p) < s0 || u0 + nu + 1 > s0 + sn) {
        // reconstructible pitches k need [k vt + bp_lo - halo, k vt + bp_hi + 1] inside the scan
        double ka = std::ceil((double)(s0 - (t.bp_lo - halo_lo(p))) / vt);
        double kb = std::floor((double)(s0 + sn - 1 - (t.bp_hi + 1)) / vt);
        char buf[200];
        std::snprintf(buf, sizeof buf, "sinogram views [%lld, %lld) do not cover pitches [%d, %d); reconstructible pitches: %.0f..%.0f",
                      (long long)s0, (long long)(s0 + sn), first_pitch, first_pitch + n_pitches, ka, kb);
        p->detail = buf;
        return KATS_ERR_COVERAGE;
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const size_t rs = raw_view_elems(p);
    float4 *gq = (float4 *)workspace;
    float *scratch = (float *)((char *)workspace + align_up(sizeof(float4) * quad_view_elems(p) * (size_t)std::max<int64_t>(nu, (t.bp_hi - t.bp_lo + 1) * n_pitches)));
    const char *pe = std::getenv("KATS_PIPELINE");
    if (n_pitches == 1 || n_groups > 1 || group_done || !(pe && (pe[0] == '1' || pe[0] == '2'))) {
        // filter every needed view once, then one backprojection launch per pitch group (default: one
        // group); group_done[i] marks the end of group i's launch on the caller's stream
        rc = run_filter(p, sino + (u0 - s0) * rs, nu, gq, scratch, nullptr, nullptr, nullptr, s, false, 0, true, dm);
        if (rc) return rc;
        const size_t vpitch = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch;
        for (int gi = 0; gi < n_groups; ++gi) {
            const int a = (int)((int64_t)n_pitches * gi / n_groups), e = (int)((int64_t)n_pitches * (gi + 1) / n_groups);
            BPParams b = bp_params(p);
            b.gq = gq;
            b.gq_views = nu;
            b.off0 = (int64_t)(first_pitch + a) * vt - u0;
            b.item_views = vt;
            b.n_items = e - a;
            b.vol = vol + (size_t)a * vpitch;
            { LaunchScope ls(p, ST_K5, s); p->last_bp_kernel = launch_backproject(b, s); }
            KCHECK(p, cudaGetLastError());
            if (group_done && group_done[gi]) KCHECK(p, cudaEventRecord((cudaEvent_t)group_done[gi], s));
        }
        return KATS_OK;
    }
    // Pipelined (KATS_PIPELINE=1; worthwhile when filtering is a large share of the step): pitch k
    // is backprojected as soon as its views are filtered, on one of two
    // streams forked from the caller's, so a launch's last wave overlaps the filtering and the
    // backprojection of the next pitch; joined back into the caller's stream (still asynchronous).
    rc = ensure_bp_streams(p);
    if (rc) return rc;
    const size_t qs = quad_view_elems(p);
    const size_t vpitch = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch;
    const int64_t nchunks = (nu + kFilterChunk - 1) / kFilterChunk;
    rc = ensure_events(p, 2 * (size_t)n_pitches + 1);
    if (rc) return rc;
    cudaStream_t fs = (cudaStream_t)p->filter_stream;
    KCHECK(p, cudaEventRecord((cudaEvent_t)p->sync_events[2 * n_pitches], s));     // fork
    KCHECK(p, cudaStreamWaitEvent(fs, (cudaEvent_t)p->sync_events[2 * n_pitches], 0));
    int64_t c_next = 0;
    // KATS_PIPELINE=2: pitch pairs (the pitch-pair kernel) while two or more pitches remain
    const int G = pe[0] == '2' ? 2 : 1;
    for (int k = 0, grp = 1; k < n_pitches; k += grp) {
        grp = std::min(G, n_pitches - k);
        const int64_t filt_end = (int64_t)(first_pitch + k + grp - 1) * vt + t.bp_hi + 1;   // exclusive
        if (c_next < nchunks && u0 + c_next * kFilterChunk < filt_end) {
            int64_t c_end = c_next;
            while (c_end < nchunks && u0 + c_end * kFilterChunk < filt_end) ++c_end;
            const int64_t a = u0 + c_next * kFilterChunk, n = std::min<int64_t>(c_end * kFilterChunk, nu) - c_next * kFilterChunk;
            rc = run_filter(p, sino + (a - s0) * rs, n, gq + (a - u0) * qs, scratch, nullptr, nullptr, nullptr, fs, false, 0, false, dm);
            if (rc) return rc;
            c_next = c_end;
        }
        cudaEvent_t e_filt = (cudaEvent_t)p->sync_events[n_pitches + k];
        KCHECK(p, cudaEventRecord(e_filt, fs));
        cudaStream_t bs = (cudaStream_t)p->bp_streams[(k / G) & 1];
        KCHECK(p, cudaStreamWaitEvent(bs, e_filt, 0));
        BPParams b = bp_params(p);
        b.gq = gq;
        b.gq_views = nu;
        b.off0 = (int64_t)(first_pitch + k) * vt - u0;
        b.item_views = vt;
        b.n_items = grp;
        b.vol = vol + (size_t)k * vpitch;
        { LaunchScope ls(p, ST_K5, bs); p->last_bp_kernel = launch_backproject(b, bs); }
        KCHECK(p, cudaGetLastError());
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->sync_events[k], bs));
    }
    for (int k = 0; k < n_pitches; ++k)                                 // join (each bp stream is in order)
        if (k % G == 0 && k + 2 * G >= n_pitches) KCHECK(p, cudaStreamWaitEvent(s, (cudaEvent_t)p->sync_events[k], 0));
    return KATS_OK;
}

// Steps 6..1 transposed (K4^T, K3^T = -K3, K12's rebin^T) over nu views in device_chunk_mul()-sized
// chunks that alternate over the filter streams and chunk scratches like run_filter (chunks write
// disjoint views of g1T; the caller's stream waits for all of them).
static int run_filter_T(katsevich_plan *p, FilterParams f, const float4 *qT, float *scratch, float *g1T,
                        int64_t nu, cudaStream_t s0)
{
    const int dm = device_chunk_mul();
    const int kFilterChunk = filter_chunk_views(p, dm);
    const size_t rs = (size_t)p->g.n_rows * p->g.n_cols;
    const size_t qs = quad_view_elems(p);
    const size_t ps = (size_t)p->t.n_psi * g3_line_pitch(p->g.n_cols);
    const size_t chunk_floats = align_up(filter_chunk_bytes(p, dm)) / sizeof(float);
    const int64_t nchunks = (nu + kFilterChunk - 1) / kFilterChunk;
    const int ns = (int)std::min<int64_t>(filter_streams(p), nchunks);
    cudaStream_t st[kFilterStreamsMax] = {s0};
    for (int i = 1; i < ns; ++i) st[i] = (cudaStream_t)p->filter_xs[i - 1];
    if (ns > 1) {
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->fork_events[0], s0));
        for (int i = 1; i < ns; ++i) KCHECK(p, cudaStreamWaitEvent(st[i], (cudaEvent_t)p->fork_events[0], 0));
    }
    for (int64_t v0 = 0; v0 < nu; v0 += kFilterChunk) {
        const int c = (int)((v0 / kFilterChunk) % std::max(ns, 1));
        cudaStream_t s = st[c];
        f.n_views = (int)std::min<int64_t>(kFilterChunk, nu - v0);
        f.g3 = scratch + c * chunk_floats;                         // g3^T
        f.g4 = f.g3 + (size_t)kFilterChunk * ps;                   // g4^T
        { LaunchScope ls(p, ST_K4, s); launch_bwd_rebin_cos_T(f, qT + v0 * qs, s); }
        KCHECK(p, cudaGetLastError());
        FilterParams h = f;                                        // K3^T = -K3: reads g4^T, writes g3^T
        h.g3 = f.g4;
        h.g4 = f.g3;
        h.sign = -1.f;
        { LaunchScope ls(p, ST_K3, s); if (launch_hilbert(h, s)) return hilbert_fail(p); }
        KCHECK(p, cudaGetLastError());
        if (f.apod) {                                              // A26: the smoothing is symmetric
            { LaunchScope ls(p, ST_K3, s); launch_hann_smooth(f, h.g4, (int64_t)f.n_views * f.npsi, 0, s); }
            KCHECK(p, cudaGetLastError());
        }
        { LaunchScope ls(p, ST_K12, s); launch_fwd_rebin_T(f, g1T + v0 * rs, s); }
        KCHECK(p, cudaGetLastError());
    }
    for (int i = 1; i < ns; ++i) {
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->fork_events[i], st[i]));
        KCHECK(p, cudaStreamWaitEvent(s0, (cudaEvent_t)p->fork_events[i], 0));
    }
    return KATS_OK;
}

// Adjoint of katsevich_reconstruct (NEXT-1): vol [n_pitches*nz][ny][nx] -> sino_out [sn][rows][cols]
// (overwritten; views outside the pitches' slabs are 0).  Step 7^T into quad adjoints over the
// union of filtered views, then steps 6..1 transposed per 256-view chunk, then the view/α
// difference stencils transposed onto the raw views.
int katsevich_adjoint(katsevich_plan *p, const float *vol, int32_t first_pitch, int32_t n_pitches,
                      float *sino_out, int64_t s0, int64_t sn, void *workspace, size_t workspace_bytes,
                      void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!vol || !sino_out || !workspace) return KATS_ERR_NULL;
    if (n_pitches < 1 || sn < 3) return KATS_ERR_ARGUMENT;
    size_t need;
    katsevich_adjoint_workspace_bytes(p, n_pitches, &need);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    const int vt = p->g.views_per_turn;
    const HostTables &t = p->t;
    const int64_t u0 = (int64_t)first_pitch * vt + t.bp_lo;
    const int64_t nu = n_union_views(p, n_pitches);
    if (u0 - halo_lo(p) < s0 || u0 + nu + 1 > s0 + sn) {
        p->detail = "output sinogram views do not cover the pitches' slabs";
        return KATS_ERR_COVERAGE;
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const size_t rs = raw_view_elems(p);
    const size_t qs = quad_view_elems(p);
    float4 *qT = (float4 *)workspace;
    const size_t qbytes = align_up(sizeof(float4) * qs * (size_t)std::max<int64_t>(nu, (t.bp_hi - t.bp_lo + 1) * n_pitches));
    float *scratch = (float *)((char *)workspace + qbytes);
    float *g1T = (float *)((char *)workspace + qbytes + kFilterStreamsMax * align_up(filter_chunk_bytes(p, device_chunk_mul())));
    KCHECK(p, cudaMemsetAsync(qT, 0, sizeof(float4) * qs * (size_t)nu, s));
    KCHECK(p, cudaMemsetAsync(sino_out, 0, sizeof(float) * rs * (size_t)sn, s));
    BPParams b = bp_params(p);
    b.gqT = qT;
    b.gq_views = nu;
    b.off0 = (int64_t)first_pitch * vt - u0;
    b.item_views = vt;
    b.n_items = n_pitches;
    b.vol = const_cast<float *>(vol);
    {
        LaunchScope ls(p, ST_K5, s);
        if (launch_backproject_adjoint(b, s) != 0) {
            p->detail = "adjoint backprojection: plan not supported (non-monotone PI windows)";
            return KATS_ERR_ARGUMENT;
        }
    }
    KCHECK(p, cudaGetLastError());
    FilterParams f = filter_params(p);
    f.hp = g3_half_pitch(p->g.n_cols);
    f.k3_in_split = hilbert_split_input(f) ? 1 : 0;         // K4^T writes the lines K3^T reads
    rc = run_filter_T(p, f, qT, scratch, g1T, nu, s);
    if (rc) return rc;
    { LaunchScope ls(p, ST_K12, s); launch_deriv_T(f, g1T, nu, sino_out + (u0 - halo_lo(p) - s0) * rs, s); }
    KCHECK(p, cudaGetLastError());
    return KATS_OK;
}

// Adjoint of katsevich_reconstruct_batch: vols [B][nz][ny][nx] -> slabs_out [B][n_slab][rows][cols]
// (overwritten).  Step 7^T over the B slabs as items, the filter transposes over all slabs' views
// in one chunked pass, the difference stencils transposed inside each slab.
int katsevich_adjoint_batch(katsevich_plan *p, const float *vols, int32_t B, float *slabs_out, void *workspace,
                            size_t workspace_bytes, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!vols || !slabs_out || !workspace) return KATS_ERR_NULL;
    if (B < 1) return KATS_ERR_ARGUMENT;
    size_t need;
    katsevich_adjoint_batch_workspace_bytes(p, B, &need);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const HostTables &t = p->t;
    const size_t rs = raw_view_elems(p);
    const size_t qs = quad_view_elems(p);
    const int64_t nbp = t.bp_hi - t.bp_lo + 1, nu = nbp * B;
    float4 *qT = (float4 *)workspace;
    const size_t qbytes = align_up(sizeof(float4) * qs * (size_t)std::max<int64_t>(n_union_views(p, B), nu));
    float *scratch = (float *)((char *)workspace + qbytes);
    float *g1T = (float *)((char *)workspace + qbytes + kFilterStreamsMax * align_up(filter_chunk_bytes(p, device_chunk_mul())));
    KCHECK(p, cudaMemsetAsync(qT, 0, sizeof(float4) * qs * (size_t)nu, s));
    KCHECK(p, cudaMemsetAsync(slabs_out, 0, sizeof(float) * rs * (size_t)(nbp + 1 + halo_lo(p)) * B, s));
    BPParams b = bp_params(p);
    b.gqT = qT;
    b.gq_views = nu;
    b.off0 = -t.bp_lo;
    b.item_views = nbp;
    b.n_items = B;
    b.vol = const_cast<float *>(vols);
    {
        LaunchScope ls(p, ST_K5, s);
        if (launch_backproject_adjoint(b, s) != 0) {
            p->detail = "adjoint backprojection: plan not supported (non-monotone PI windows)";
            return KATS_ERR_ARGUMENT;
        }
    }
    KCHECK(p, cudaGetLastError());
    FilterParams f = filter_params(p);
    f.hp = g3_half_pitch(p->g.n_cols);
    f.k3_in_split = hilbert_split_input(f) ? 1 : 0;         // K4^T writes the lines K3^T reads
    rc = run_filter_T(p, f, qT, scratch, g1T, nu, s);
    if (rc) return rc;
    { LaunchScope ls(p, ST_K12, s); launch_deriv_T(f, g1T, nbp, slabs_out, s, B); }
    KCHECK(p, cudaGetLastError());
    return KATS_OK;
}

int katsevich_reconstruct_batch(katsevich_plan *p, const float *slabs, int32_t B, float *vols,
                                void *workspace, size_t workspace_bytes, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!slabs || !vols || !workspace) return KATS_ERR_NULL;
    if (B < 1) return KATS_ERR_ARGUMENT;
    size_t need;
    katsevich_workspace_bytes(p, B, &need);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const HostTables &t = p->t;
    const size_t rs = raw_view_elems(p);
    const int64_t nbp = t.bp_hi - t.bp_lo + 1;        // filtered views per slab
    const int64_t nslab = nbp + 1 + halo_lo(p);        // raw views per slab
    float4 *gq = (float4 *)workspace;
    const size_t qs = quad_view_elems(p);
    float *scratch = (float *)((char *)workspace + align_up(sizeof(float4) * qs * (size_t)std::max<int64_t>(n_union_views(p, B), nbp * B)));
    (void)nslab;
    // groups of slabs (KATS_BATCH_GROUPS, default 1): group g+1 is filtered on the highest-priority
    // stream while group g backprojects on a low-priority one, so the filter fills the SMs the
    // backprojection leaves idle (group sizes stay even for the window kernel's slab pairs)
    // (default: two groups for batches of >= 16 slabs in groups of a multiple of 4, the window
    // kernel's four slabs per CTA — C5 3.58 -> 3.49 ms, scripts/ab/gpu_r02h.sh; four groups: 3.94 ms)
    std::vector<int> gsz;                                       // slabs per group
    {
        // (not with the half-sample derivative or the Hann filter: C5 6.49 -> 6.87 ms and 3.86 -> 3.95 ms
        // in groups, measured in the bench's variants; the caller's flags: the half-sample plan's
        // effective grid p->g has that flag cleared)
        int ng = B >= 16 && B % 8 == 0 && !(p->graw.flags & (KATS_FLAG_HALF_SAMPLE | KATS_FLAG_HANN)) ? 2 : 1;
        if (const char *e = std::getenv("KATS_BATCH_GROUPS")) ng = std::max(1, std::atoi(e));
        while (ng > 1 && (B % ng != 0 || ((B / ng) % 2 != 0 && B % 2 == 0))) --ng;
        gsz.assign(ng, B / ng);
        // KATS_BATCH_SPLIT=a,b,...: explicit group sizes (A/B; used when they sum to B)
        if (const char *e = std::getenv("KATS_BATCH_SPLIT")) {
            std::vector<int> v;
            for (const char *c = e; *c;) {
                char *end;
                const long n = std::strtol(c, &end, 10);
                if (end == c || n < 1) { v.clear(); break; }
                v.push_back((int)n);
                c = *end == ',' ? end + 1 : end;
                if (*end && *end != ',') { v.clear(); break; }
            }
            int sum = 0;
            for (int n : v) sum += n;
            if (sum == B && !v.empty()) gsz = v;
        }
    }
    const int ng = (int)gsz.size();
    if (ng == 1) {
        // every slab's filtered views in one chunked pass (chunks run across slab ends; each slab
        // keeps its own +-1 halo)
        rc = run_filter(p, slabs + halo_lo(p) * rs, nbp * B, gq, scratch, nullptr, nullptr, nullptr, s, false, nbp, true,
                        device_chunk_mul(), batch_chunk_views(p, B));
        if (rc) return rc;
        BPParams bp = bp_params(p);
        bp.gq = gq;
        bp.gq_views = nbp * B;
        bp.off0 = -t.bp_lo;
        bp.item_views = nbp;
        bp.n_items = B;
        bp.vol = vols;
        { LaunchScope ls(p, ST_K5, s); p->last_bp_kernel = launch_backproject(bp, s); }
        KCHECK(p, cudaGetLastError());
        return KATS_OK;
    }
    rc = ensure_bp_streams(p);
    if (rc) return rc;
    rc = ensure_events(p, 2 * (size_t)ng + 1);
    if (rc) return rc;
    cudaStream_t fs = (cudaStream_t)p->filter_stream;
    cudaEvent_t e_fork = (cudaEvent_t)p->sync_events[2 * ng];
    KCHECK(p, cudaEventRecord(e_fork, s));
    KCHECK(p, cudaStreamWaitEvent(fs, e_fork, 0));
    for (int g = 0, b0 = 0; g < ng; b0 += gsz[g], ++g) {
        const int gs = gsz[g];
        // each group's views in device chunks (KATS_BATCH_GCHUNK=1: in the batch chunking, two equal
        // chunks on the two filter streams, no larger than the chunk the workspace was sized for —
        // measured slower, C5 3.574 vs 3.497 ms, scripts/ab/gpu_r02i.sh)
        int64_t gchunk = 0;
        if (const char *e = std::getenv("KATS_BATCH_GCHUNK"))
            if (e[0] == '1')
                gchunk = std::min(batch_chunk_views(p, gs), std::max<int64_t>(filter_chunk_views(p, device_chunk_mul()),
                                                                              batch_chunk_views(p, B)));
        rc = run_filter(p, slabs + ((size_t)b0 * nslab + halo_lo(p)) * rs, nbp * gs, gq + (size_t)b0 * nbp * qs,
                        scratch, nullptr, nullptr, nullptr, fs, false, nbp, true, device_chunk_mul(), gchunk);
        if (rc) return rc;
        cudaEvent_t e_filt = (cudaEvent_t)p->sync_events[ng + g];
        KCHECK(p, cudaEventRecord(e_filt, fs));
        cudaStream_t bs = (cudaStream_t)p->bp_streams[g & 1];
        KCHECK(p, cudaStreamWaitEvent(bs, e_filt, 0));
        BPParams bp = bp_params(p);
        bp.gq = gq;
        bp.gq_views = nbp * B;
        bp.off0 = -t.bp_lo + (int64_t)b0 * nbp;
        bp.item_views = nbp;
        bp.n_items = gs;
        bp.vol = vols + (size_t)b0 * p->g.nx * p->g.ny * p->g.nz_per_pitch;
        { LaunchScope ls(p, ST_K5, bs); p->last_bp_kernel = launch_backproject(bp, bs); }
        KCHECK(p, cudaGetLastError());
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->sync_events[g], bs));
    }
    for (int g = std::max(0, ng - 2); g < ng; ++g)                 // join (each bp stream is in order)
        KCHECK(p, cudaStreamWaitEvent(s, (cudaEvent_t)p->sync_events[g], 0));
    return KATS_OK;
}

int katsevich_workspace_bytes_batch_host(const katsevich_plan *p, int32_t B, size_t *bytes)
{
    int rc = katsevich_workspace_bytes(p, B, bytes);
    if (rc) return rc;
    const int64_t nslab = p->t.bp_hi - p->t.bp_lo + 2 + halo_lo(p);
    const size_t vol = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch;
    *bytes += align_up(sizeof(float) * raw_view_elems(p) * (size_t)nslab * B) + align_up(sizeof(float) * vol * B);
    return KATS_OK;
}

// katsevich_reconstruct_batch with host slabs and volumes: the batch runs in groups of slabs; group
// i's slabs are copied in on one stream, filtered on the highest-priority stream as soon as they
// land, backprojected on a third, and their volumes copied out on a fourth while the next group
// runs, so the PCIe transfers overlap the kernels.  Synchronises before returning.
int katsevich_reconstruct_batch_host(katsevich_plan *p, const float *host_slabs, int32_t B, float *host_vols,
                                     void *workspace, size_t workspace_bytes, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!host_slabs || !host_vols || !workspace) return KATS_ERR_NULL;
    if (B < 1) return KATS_ERR_ARGUMENT;
    size_t need, base;
    katsevich_workspace_bytes_batch_host(p, B, &need);
    katsevich_workspace_bytes(p, B, &base);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (!p->copy_stream) {
        cudaStream_t a, b;
        KCHECK(p, cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
        KCHECK(p, cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        p->copy_stream = a;
        p->copy_stream2 = b;
    }
    rc = ensure_bp_streams(p);
    if (rc) return rc;
    const HostTables &t = p->t;
    const size_t rs = raw_view_elems(p), qs = quad_view_elems(p);
    const int64_t nbp = t.bp_hi - t.bp_lo + 1, nslab = nbp + 1 + halo_lo(p);
    const size_t vpitch = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch;
    // groups of 4 slabs (even groups keep the window kernel's slab pairs)
    const int gs = B % 4 == 0 ? 4 : B % 2 == 0 ? 2 : 1, ng = B / gs;
    rc = ensure_events(p, 3 * (size_t)ng + 1);
    if (rc) return rc;
    float4 *gq = (float4 *)workspace;
    float *scratch = (float *)((char *)workspace + align_up(sizeof(float4) * qs * (size_t)std::max<int64_t>(n_union_views(p, B), nbp * B)));
    float *dslabs = (float *)((char *)workspace + base);
    float *dvols = (float *)((char *)dslabs + align_up(sizeof(float) * rs * (size_t)nslab * B));
    cudaStream_t cs = (cudaStream_t)p->copy_stream, ds = (cudaStream_t)p->copy_stream2;
    cudaStream_t fs = (cudaStream_t)p->filter_stream, bs = (cudaStream_t)p->bp_streams[0];
    cudaEvent_t e_start = (cudaEvent_t)p->sync_events[3 * ng];
    KCHECK(p, cudaEventRecord(e_start, s));                   // the caller's pending work comes first
    KCHECK(p, cudaStreamWaitEvent(cs, e_start, 0));
    KCHECK(p, cudaStreamWaitEvent(fs, e_start, 0));
    KCHECK(p, cudaStreamWaitEvent(bs, e_start, 0));
    const size_t gslab = rs * (size_t)nslab * gs;             // floats of one group's slabs
    for (int g = 0; g < ng; ++g) {
        KCHECK(p, cudaMemcpyAsync(dslabs + g * gslab, host_slabs + g * gslab, sizeof(float) * gslab,
                                  cudaMemcpyHostToDevice, cs));
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->sync_events[g], cs));
    }
    for (int g = 0; g < ng; ++g) {
        KCHECK(p, cudaStreamWaitEvent(fs, (cudaEvent_t)p->sync_events[g], 0));
        rc = run_filter(p, dslabs + g * gslab + halo_lo(p) * rs, nbp * gs, gq + (size_t)g * gs * nbp * qs, scratch,
                        nullptr, nullptr, nullptr, fs, false, nbp);
        if (rc) return rc;
        cudaEvent_t e_filt = (cudaEvent_t)p->sync_events[ng + g];
        KCHECK(p, cudaEventRecord(e_filt, fs));
        KCHECK(p, cudaStreamWaitEvent(bs, e_filt, 0));
        BPParams bp = bp_params(p);
        bp.gq = gq;
        bp.gq_views = nbp * B;
        bp.off0 = -t.bp_lo + (int64_t)g * gs * nbp;
        bp.item_views = nbp;
        bp.n_items = gs;
        bp.vol = dvols + (size_t)g * gs * vpitch;
        { LaunchScope ls(p, ST_K5, bs); p->last_bp_kernel = launch_backproject(bp, bs); }
        KCHECK(p, cudaGetLastError());
        cudaEvent_t e_bp = (cudaEvent_t)p->sync_events[2 * ng + g];
        KCHECK(p, cudaEventRecord(e_bp, bs));
        KCHECK(p, cudaStreamWaitEvent(ds, e_bp, 0));
        KCHECK(p, cudaMemcpyAsync(host_vols + (size_t)g * gs * vpitch, bp.vol, sizeof(float) * vpitch * gs,
                                  cudaMemcpyDeviceToHost, ds));
    }
    KCHECK(p, cudaStreamSynchronize(ds));
    KCHECK(p, cudaStreamSynchronize(cs));
    KCHECK(p, cudaStreamSynchronize(bs));
    KCHECK(p, cudaStreamSynchronize(fs));
    KCHECK(p, cudaStreamSynchronize(s));
    return KATS_OK;
}

int katsevich_reconstruct_host(katsevich_plan *p, const float *host_sino, int64_t s0, int64_t sn,
                               int32_t first_pitch, int32_t n_pitches, float *host_vol,
                               void *workspace, size_t workspace_bytes, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    const int kFilterChunk = filter_chunk_views(p);
    if (!host_sino || !host_vol || !workspace) return KATS_ERR_NULL;
    if (n_pitches < 1) return KATS_ERR_ARGUMENT;
    size_t need, base;
    katsevich_workspace_bytes_host(p, n_pitches, &need);
    katsevich_workspace_bytes(p, n_pitches, &base);
    if (workspace_bytes < need) { p->detail = "workspace too small"; return KATS_ERR_WORKSPACE; }
    int64_t fv, nv;
    katsevich_scan_views(p, first_pitch, n_pitches, &fv, &nv);
    if (fv < s0 || fv + nv > s0 + sn) return katsevich_reconstruct(p, host_sino, s0, sn, first_pitch, n_pitches,
                                                                   host_vol, workspace, workspace_bytes, cuda_stream);
    // Pipelined on three streams: every host->device copy is enqueued up front on the copy stream,
    // one piece per 256-view filter chunk with an event each, so filtering trails the copy chunk by
    // chunk; each pitch is backprojected as soon as its views are filtered and its volume goes back
    // on a second copy stream while the next pitch runs (caller's stream: filter + BP).
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (!p->copy_stream) {
        cudaStream_t a, b;
        KCHECK(p, cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
        KCHECK(p, cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        p->copy_stream = a;
        p->copy_stream2 = b;
    }
    rc = ensure_bp_streams(p);
    if (rc) return rc;
    cudaStream_t cs = (cudaStream_t)p->copy_stream, ds = (cudaStream_t)p->copy_stream2;
    const HostTables &t = p->t;
    const int vt = p->g.views_per_turn;
    const size_t rs = raw_view_elems(p);
    const size_t qs = quad_view_elems(p);
    const size_t vpitch = (size_t)p->g.nx * p->g.ny * p->g.nz_per_pitch;
    const int64_t u0 = (int64_t)first_pitch * vt + t.bp_lo;   // first filtered view (= fv + halo)
    const int64_t nu = n_union_views(p, n_pitches);
    const int64_t nchunks = (nu + kFilterChunk - 1) / kFilterChunk;
    while ((int64_t)p->sync_events.size() < nchunks + 2 * n_pitches + 1) {
        cudaEvent_t e;
        KCHECK(p, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->sync_events.push_back(e);
    }
    float4 *gq = (float4 *)workspace;
    float *scratch = (float *)((char *)workspace + align_up(sizeof(float4) * qs * (size_t)std::max<int64_t>(nu, (t.bp_hi - t.bp_lo + 1) * n_pitches)));
    float *dsino = (float *)((char *)workspace + base);
    float *dvol = (float *)((char *)dsino + align_up(sizeof(float) * rs * (size_t)nv));
    // the caller's pending work on s (e.g. earlier writes to the workspace) precedes our copies
    cudaEvent_t e_start = (cudaEvent_t)p->sync_events[nchunks + 2 * n_pitches];
    KCHECK(p, cudaEventRecord(e_start, s));
    KCHECK(p, cudaStreamWaitEvent(cs, e_start, 0));
    cudaStream_t fs = (cudaStream_t)p->filter_stream;
    KCHECK(p, cudaStreamWaitEvent(fs, e_start, 0));
    // chunk c filters views [u0 + 256 c, u0 + 256 c + n) and needs raw views up to one past its end
    int64_t copied_to = fv;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t raw_end = u0 + std::min<int64_t>((c + 1) * kFilterChunk, nu) + 1;   // exclusive
        KCHECK(p, cudaMemcpyAsync(dsino + (copied_to - fv) * rs, host_sino + (copied_to - s0) * rs,
                                  sizeof(float) * rs * (size_t)(raw_end - copied_to), cudaMemcpyHostToDevice, cs));
        KCHECK(p, cudaEventRecord((cudaEvent_t)p->sync_events[c], cs));
        copied_to = raw_end;
    }
    int64_t c_next = 0;                                       // next chunk to filter
    // pitches go to step 7 in pairs while at least three remain (a pair shares its windows and
    // geometry in the TMEM kernel: pitch pairs), the last ones alone (shorter device->host tail);
    // KATS_HOST_PAIRS=0: one pitch per launch
    const char *hp = std::getenv("KATS_HOST_PAIRS");
    const bool pairs = !(hp && hp[0] == '0');
    int grp = 0, gi = 0;
    for (int k = 0; k < n_pitches; k += grp, ++gi) {
        grp = pairs && n_pitches - k >= 3 ? 2 : 1;
        const int kl = k + grp - 1;                            // last pitch of the group
        const int64_t filt_end = (int64_t)(first_pitch + kl) * vt + t.bp_hi + 1;   // exclusive
        while (c_next < nchunks && u0 + c_next * kFilterChunk < filt_end) {
            const int64_t a = u0 + c_next * kFilterChunk, n = std::min<int64_t>(kFilterChunk, nu - c_next * kFilterChunk);
            KCHECK(p, cudaStreamWaitEvent(fs, (cudaEvent_t)p->sync_events[c_next], 0));
            // before the first pitch's BP nothing runs beside the filter: tensor-core Hilbert; after
            // it the filter shares SMs with TMEM backprojection CTAs: fp32 Hilbert (launch_hilbert)
            rc = run_filter(p, dsino + (a - fv) * rs, n, gq + (a - u0) * qs, scratch, nullptr, nullptr, nullptr, fs,
                            k > 0);
            if (rc) return rc;
            ++c_next;
        }
        // pitch k's BP on alternating streams: its tail overlaps the next pitch's filter and BP
        cudaEvent_t e_filt = (cudaEvent_t)p->sync_events[nchunks + n_pitches + k];
        KCHECK(p, cudaEventRecord(e_filt, fs));
        cudaStream_t bs = (cudaStream_t)p->bp_streams[gi & 1];
        KCHECK(p, cudaStreamWaitEvent(bs, e_filt, 0));
        BPParams b = bp_params(p);
        b.gq = gq;
        b.gq_views = nu;
        b.off0 = (int64_t)(first_pitch + k) * vt - u0;
        b.item_views = vt;
        b.n_items = grp;
        b.vol = dvol + (size_t)k * vpitch;
        { LaunchScope ls(p, ST_K5, bs); p->last_bp_kernel = launch_backproject(b, bs); }
        KCHECK(p, cudaGetLastError());
        cudaEvent_t e_bp = (cudaEvent_t)p->sync_events[nchunks + k];
        KCHECK(p, cudaEventRecord(e_bp, bs));
        KCHECK(p, cudaStreamWaitEvent(ds, e_bp, 0));
        KCHECK(p, cudaMemcpyAsync(host_vol + (size_t)k * vpitch, b.vol, sizeof(float) * vpitch * grp,
                                  cudaMemcpyDeviceToHost, ds));
    }
    KCHECK(p, cudaStreamSynchronize(ds));
    KCHECK(p, cudaStreamSynchronize(cs));
    KCHECK(p, cudaStreamSynchronize((cudaStream_t)p->bp_streams[0]));
    KCHECK(p, cudaStreamSynchronize((cudaStream_t)p->bp_streams[1]));
    KCHECK(p, cudaStreamSynchronize(fs));
    KCHECK(p, cudaStreamSynchronize(s));
    return KATS_OK;
}

// ---- data generation (NEXT-3) ----
static DataGenParams datagen_params(const katsevich_plan *p)
{
    const katsevich_geometry &g = p->graw;                  // the physical scan (not the half-shifted grid)
    DataGenParams d{};
    d.R = g.R; d.D = g.D; d.h = g.pitch / (2.0 * kPi); d.lambda0 = g.lambda0; d.z0 = g.z0;
    d.dlam = 2.0 * kPi / g.views_per_turn; d.d_w = g.d_w; d.d_alpha = g.d_alpha; d.alpha_offset = g.alpha_offset;
    d.dx = g.dx; d.dy = g.dy; d.nr = g.n_rows; d.nc = g.n_cols; d.nx = g.nx; d.ny = g.ny;
    d.flat = (g.flags & KATS_FLAG_FLAT) ? 1 : 0;
    return d;
}

static int plan_scratch(katsevich_plan *p, size_t bytes)
{
    if (p->dg_scratch_bytes >= bytes) return KATS_OK;
    if (p->dg_scratch) cudaFree(p->dg_scratch);
    p->dg_scratch = nullptr;
    p->dg_scratch_bytes = 0;
    KCHECK(p, cudaMalloc(&p->dg_scratch, bytes));
    p->dg_scratch_bytes = bytes;
    return KATS_OK;
}

int katsevich_project_ellipsoids(katsevich_plan *p, const double *ell, int32_t n_ell, int64_t first_view,
                                 int64_t n_views, float *sino, void *cuda_stream)
{
    if (!p) return KATS_ERR_NULL;
    if (p->device < 0) return KATS_ERR_NO_DEVICE;
    if (!sino || (n_ell > 0 && !ell)) return KATS_ERR_NULL;
    if (n_views < 1 || n_ell < 0 || n_ell > 2048) return KATS_ERR_ARGUMENT;
    cudaSetDevice(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    int rc = plan_scratch(p, sizeof(double) * 8 * (size_t)std::max(n_ell, 1));
    if (rc) return rc;
    if (n_ell > 0)
        KCHECK(p, cudaMemcpyAsync(p->dg_scratch, ell, sizeof(double) * 8 * (size_t)n_ell, cudaMemcpyHostToDevice, s));
    { LaunchScope ls(p, ST_OTHER, s);
      launch_project_ellipsoids(datagen_params(p), (const double *)p->dg_scratch, n_ell, first_view, n_views, sino, s); }
    KCHECK(p, cudaGetLastError());
    return KATS_OK;
}

int katsevich_project_volume(katsevich_plan *p, const float *vol, int32_t nz_vol, double z_first, double dz_vol,
                             int64_t first_view, int64_t n_views, float *sino, int64_t *n_truncated, void *cuda_stream)
{
    if (!p) return KATS_ERR_NULL;
    if (p->device < 0) return KATS_ERR_NO_DEVICE;
    if (!vol || !sino) return KATS_ERR_NULL;
    if (n_views < 1 || nz_vol < 1 || !(dz_vol > 0.0)) return KATS_ERR_ARGUMENT;
    cudaSetDevice(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    int rc = plan_scratch(p, 64);
    if (rc) return rc;
    unsigned long long *cnt = (unsigned long long *)p->dg_scratch;
    KCHECK(p, cudaMemsetAsync(cnt, 0, sizeof(*cnt), s));
    { LaunchScope ls(p, ST_OTHER, s);
      launch_project_volume(datagen_params(p), vol, nz_vol, (float)z_first, (float)dz_vol, first_view, n_views, sino,
                            cnt, s); }
    KCHECK(p, cudaGetLastError());
    if (n_truncated) {
        unsigned long long h = 0;
        KCHECK(p, cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
        KCHECK(p, cudaStreamSynchronize(s));
        *n_truncated = (int64_t)h;
    }
    return KATS_OK;
}

int katsevich_degrade(katsevich_plan *p, const float *sino, int64_t first_view, int64_t n_views, int32_t alpha_stride,
                      double I0, double gauss_var, uint64_t seed, int32_t mode, float *out, int64_t *counts,
                      float *M_out, void *cuda_stream)
{
    if (!p) return KATS_ERR_NULL;
    if (p->device < 0) return KATS_ERR_NO_DEVICE;
    if (!sino || !out) return KATS_ERR_NULL;
    if (n_views < 1 || alpha_stride < 1 || !(I0 > 0.0) || gauss_var < 0.0 || (mode != 0 && mode != 1))
        return KATS_ERR_ARGUMENT;
    cudaSetDevice(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const size_t n = (size_t)n_views * raw_view_elems(p);
    int rc = plan_scratch(p, 256 + sizeof(float) * n);
    if (rc) return rc;
    unsigned *maxbits = (unsigned *)p->dg_scratch;
    float *up = (float *)((char *)p->dg_scratch + 256);
    { LaunchScope ls(p, ST_OTHER, s);
      launch_degrade(datagen_params(p), sino, first_view, n_views, alpha_stride, I0, gauss_var, seed, mode, up, maxbits,
                     out, (long long *)counts, M_out, s); }
    KCHECK(p, cudaGetLastError());
    return KATS_OK;
}

int katsevich_filter(katsevich_plan *p, const float *sino, int64_t s0, int64_t sn,
                     int64_t out_first_view, int32_t n_out, float *g3, float *g4, float *gF, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!sino || !gF) return KATS_ERR_NULL;
    if (n_out < 1) return KATS_ERR_ARGUMENT;
    if (out_first_view - halo_lo(p) < s0 || out_first_view + n_out + 1 > s0 + sn) {
        p->detail = "sinogram does not hold the derivative halo of the requested views";
        return KATS_ERR_COVERAGE;
    }
    const size_t rs = raw_view_elems(p);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    float *scratch = nullptr;
    float4 *gq = nullptr;
    KCHECK(p, cudaMallocAsync((void **)&scratch, filter_chunk_bytes(p), s));   // (split K3 input lines)
    KCHECK(p, cudaMallocAsync((void **)&gq, sizeof(float4) * quad_view_elems(p) * (size_t)n_out, s));
    rc = run_filter(p, sino + (out_first_view - s0) * rs, n_out, gq, scratch, g3, g4, gF, s);
    cudaFreeAsync(scratch, s);
    cudaFreeAsync(gq, s);
    return rc;
}

int katsevich_backproject(katsevich_plan *p, const float *gF, int64_t gF0, int64_t gFn,
                          int32_t pitch, float *vol, void *cuda_stream)
{
    int rc = check_device_plan(p);
    if (rc) return rc;
    if (!gF || !vol) return KATS_ERR_NULL;
    const int vt = p->g.views_per_turn;
    const int64_t a = (int64_t)pitch * vt + p->t.bp_lo, b = (int64_t)pitch * vt + p->t.bp_hi;
    if (a < gF0 || b >= gF0 + gFn) { p->detail = "filtered views do not cover the pitch"; return KATS_ERR_COVERAGE; }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    float4 *gq = nullptr;
    const int nr = p->g.n_rows, nc = p->g.n_cols;
    KCHECK(p, cudaMallocAsync((void **)&gq, sizeof(float4) * quad_view_elems(p) * gFn, s));
    { LaunchScope ls(p, ST_OTHER, s); launch_make_quads(gF, gq, gFn, nr, nc, s); }
    KCHECK(p, cudaGetLastError());
    BPParams bp = bp_params(p);
    bp.gq = gq;
    bp.gq_views = gFn;
    bp.off0 = (int64_t)pitch * vt - gF0;
    bp.item_views = 0;
    bp.n_items = 1;
    bp.vol = vol;
    { LaunchScope ls(p, ST_K5, s); p->last_bp_kernel = launch_backproject(bp, s); }
    KCHECK(p, cudaGetLastError());
    cudaFreeAsync(gq, s);
    return KATS_OK;
}

int katsevich_hilbert_hk_table(int32_t n_cols, const float *taps, float *out, size_t out_floats)
{
    if (n_cols < 1 || !taps || !out) return KATS_ERR_ARGUMENT;
    if (out_floats < hilbert_hk_table_floats(n_cols)) return KATS_ERR_ARGUMENT;
    std::vector<float> t;
    hilbert_hk_table(n_cols, taps, t);
    std::copy(t.begin(), t.end(), out);
    return KATS_OK;
}

int katsevich_table_info(const katsevich_plan *p, int32_t *n_psi, int64_t *lo, int64_t *hi)
{
    if (!p) return KATS_ERR_NULL;
    if (!p->precomputed) return KATS_ERR_NOT_PRECOMPUTED;
    if (n_psi) *n_psi = p->t.n_psi;
    if (lo) *lo = p->t.bp_lo;
    if (hi) *hi = p->t.bp_hi;
    return KATS_OK;
}

int katsevich_export_tables(const katsevich_plan *p, int32_t *pi_first, int32_t *pi_last,
                            double *w_first, double *w_last, int32_t *fr_idx, double *fr_frac,
                            int32_t *br_idx, double *br_frac)
{
    if (!p) return KATS_ERR_NULL;
    if (!p->precomputed) return KATS_ERR_NOT_PRECOMPUTED;
    const HostTables &t = p->t;
    auto cp = [](auto *dst, const auto &v) {
        if (dst) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(pi_first, t.pi_first); cp(pi_last, t.pi_last); cp(w_first, t.w_first); cp(w_last, t.w_last);
    cp(fr_idx, t.fr_idx); cp(fr_frac, t.fr_frac); cp(br_idx, t.br_idx); cp(br_frac, t.br_frac);
    return KATS_OK;
}

int katsevich_bp_kernel(const katsevich_plan *plan)
{
    if (!plan) return KATS_ERR_NULL;
    return plan->last_bp_kernel;
}

int katsevich_profile_enable(katsevich_plan *p, int enable)
{
    if (!p) return KATS_ERR_NULL;
    if (p->device < 0) return KATS_ERR_NO_DEVICE;
    p->profiling = enable != 0;
    return KATS_OK;
}

int katsevich_profile_read(katsevich_plan *p, katsevich_stats *out, int reset)
{
    if (!p || !out) return KATS_ERR_NULL;
    if (p->device >= 0) {
        cudaSetDevice(p->device);
        // per launch: duration, and its interval against the first recorded event so that
        // launches overlapping on different streams count once in the stage's busy time
        std::vector<std::pair<float, float>> iv[6];
        for (auto &r : p->prof) {
            float ms = 0.f, a = 0.f, b = 0.f;
            KCHECK(p, cudaEventSynchronize((cudaEvent_t)r.ev1));
            KCHECK(p, cudaEventElapsedTime(&ms, (cudaEvent_t)r.ev0, (cudaEvent_t)r.ev1));
            KCHECK(p, cudaEventElapsedTime(&a, (cudaEvent_t)p->prof[0].ev0, (cudaEvent_t)r.ev0));
            KCHECK(p, cudaEventElapsedTime(&b, (cudaEvent_t)p->prof[0].ev0, (cudaEvent_t)r.ev1));
            p->stage_ms[r.stage] += ms;
            iv[r.stage].push_back({a, b});
        }
        for (int st = 0; st < 6; ++st) {
            std::sort(iv[st].begin(), iv[st].end());
            double busy = 0.0, lo = 0.0, hi = -1e300;
            for (auto &x : iv[st]) {
                if (x.first > hi) { if (hi > lo) busy += hi - lo; lo = x.first; hi = x.second; }
                else hi = std::max<double>(hi, x.second);
            }
            if (hi > lo) busy += hi - lo;
            p->stage_busy_ms[st] += busy;
        }
        for (auto &r : p->prof) {
            p->event_pool.push_back(r.ev0);
            p->event_pool.push_back(r.ev1);
        }
        p->prof.clear();
    }
    for (int i = 0; i < 6; ++i) {
        out->launches[i] = p->stage_launches[i];
        out->ms[i] = p->stage_ms[i];
        out->busy_ms[i] = p->stage_busy_ms[i];
    }
    out->total_launches = p->total_launches;
    if (reset) {
        for (int i = 0; i < 6; ++i) { p->stage_launches[i] = 0; p->stage_ms[i] = 0; p->stage_busy_ms[i] = 0; }
        p->total_launches = 0;
    }
    return KATS_OK;
}

void katsevich_destroy(katsevich_plan *p)
{
    if (!p) return;
    free_device(p);
    delete p;
}

const char *katsevich_error_string(int code)
{
    switch (code) {
    case KATS_OK: return "ok";
    case KATS_WARN_TD_NOT_COVERED: return "warning: detector does not cover the Tam-Danielsson window";
    case KATS_ERR_NULL: return "null pointer argument";
    case KATS_ERR_INVALID_GEOMETRY: return "invalid geometry";
    case KATS_ERR_NOT_PRECOMPUTED: return "plan not precomputed";
    case KATS_ERR_COVERAGE: return "sinogram does not cover the requested pitches";
    case KATS_ERR_PI_NONCONVERGENCE: return "PI-line / kappa-line solver did not converge";
    case KATS_ERR_WORKSPACE: return "workspace too small";
    case KATS_ERR_CUDA: return "CUDA error";
    case KATS_ERR_NO_DEVICE: return "no CUDA device for this plan";
    case KATS_ERR_ARGUMENT: return "invalid argument";
    default: return "unknown error code";
    }
}

const char *katsevich_last_error_detail(const katsevich_plan *p)
{
    return p ? p->detail.c_str() : "";
}

}  // extern "C"
