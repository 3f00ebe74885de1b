// filter.cu — filtering steps 1-6 of the Katsevich implementation of
// PAPER.md §II (l.117-154) as sm_100a kernels.  Each filtered view depends
// only on raw views v-1, v, v+1, so the same kernels serve the per-pitch slab
// (P:l.250) and the filter-once long-scan path.
#include "kernels.cuh"

namespace kats {

// ---------------------------------------------------------------------------
// K12: g3[v][i][l] = lerp_w(g2[v][·][l], w_κ(α_l, ψ_i)),  g2 = D/sqrt(D²+w²)·g1,
//      g1 = (∂_q + ∂_α) g   (Eqs. 8-11).  g2 is never materialised: the two
//      rows the κ-line sample needs are differentiated on the fly (centred
//      differences, one-sided at the α edges; reading A5).
// Grid: x over α (coalesced), y over ψ, z over views.
// ---------------------------------------------------------------------------
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

__global__ void __launch_bounds__(128) k_deriv_fwd_rebin(FilterParams p)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    const int v = blockIdx.z;
    if (l >= p.nc) return;
    const RebinEntry e = p.fr[i * p.nc + l];
    float out = 0.f;
    if (e.idx >= 0) {
        const float *gv = p.sino + (size_t)v * p.nr * p.nc;
        float a = g2_at(p, gv, e.idx, l);
        float b = g2_at(p, gv, e.idx + 1, l);
        out = fmaf(e.frac, b - a, a);
    }
    p.g3[((size_t)v * p.npsi + i) * p.nc + l] = out;
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
        if (l0 + 2 * j < nc) dst[l0 + 2 * j] = acc[j];
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

__global__ void __launch_bounds__(256) k_bwd_rebin_cos(FilterParams p)
{
    extern __shared__ float tile[];            // [nr + 3][K4_COLS + 1], rows m = -2 .. nr
    const int nc = p.nc, nr = p.nr, nq = nr + 2;
    const int l0 = blockIdx.x * K4_COLS;
    const int v = blockIdx.y;
    const int cols = min(K4_COLS, nc - l0);
    const int ld = K4_COLS + 1;
    for (int e = threadIdx.x; e < (nr + 3) * ld; e += blockDim.x) {
        const int mm = e / ld, ll = e - mm * ld, m = mm - 2, l = l0 + ll;
        float out = 0.f;
        if (m >= 0 && m < nr && l < nc && ll <= cols) {
            const RebinEntry r = p.br[m * nc + l];
            if (r.idx >= 0) {
                const float *g = p.g4 + ((size_t)v * p.npsi + r.idx) * nc + l;
                const float a = g[0], b = g[nc];
                out = __ldg(p.cos_alpha + l) * fmaf(r.frac, b - a, a);
            }
            if (p.gF && ll < cols) p.gF[((size_t)v * nr + m) * nc + l] = out;
        }
        tile[e] = out;
    }
    __syncthreads();
    float4 *q = p.gq + ((size_t)v * nc + l0) * nq;
    for (int e = threadIdx.x; e < cols * nq; e += blockDim.x) {
        const int ll = e / nq, r = e - ll * nq;        // r = quad row; taps rows r-2, r-1
        const float *t0 = tile + r * ld + ll;
        const float a0 = t0[0], a1 = t0[1], c0 = t0[ld], c1 = t0[ld + 1];
        const float rc = (float)(r - (nr + 2) / 2);      // centred quad row
        q[e] = make_float4(fmaf(-rc, c0 - a0, 0.5f * (a0 + c0)), fmaf(-rc, c1 - a1, 0.5f * (a1 + c1)), c0 - a0, c1 - a1);
    }
}

void launch_deriv_fwd_rebin(const FilterParams &p, cudaStream_t s)
{
    dim3 grid((p.nc + 127) / 128, p.npsi, p.n_views);
    k_deriv_fwd_rebin<<<grid, 128, 0, s>>>(p);
}

void launch_hilbert(const FilterParams &p, cudaStream_t s)
{
    const int tpl = 2 * (((p.nc + 1) / 2 + HR - 1) / HR);
    const int lpb = tpl >= 256 ? 1 : 256 / tpl;
    const int64_t n_lines = (int64_t)p.n_views * p.npsi;
    size_t smem = sizeof(float) * (2 * (size_t)p.nc - 1 + 2 * (2 * HR + 4) + (size_t)lpb * p.nc);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_hilbert, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int threads = ((lpb * tpl + 31) / 32) * 32;
    k_hilbert<<<(unsigned)((n_lines + lpb - 1) / lpb), threads, smem, s>>>(p, n_lines, lpb);
}

void launch_bwd_rebin_cos(const FilterParams &p, cudaStream_t s)
{
    dim3 grid((p.nc + K4_COLS - 1) / K4_COLS, p.n_views);
    size_t smem = sizeof(float) * (size_t)(p.nr + 3) * (K4_COLS + 1);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_bwd_rebin_cos, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    k_bwd_rebin_cos<<<grid, 256, smem, s>>>(p);
}

}  // namespace kats
