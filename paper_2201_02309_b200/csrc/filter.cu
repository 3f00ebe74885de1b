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
//     distances contribute).  One CTA per line; line and kernel staged in
//     shared memory; direct convolution (n_cols/2 MACs per output).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hilbert_direct(FilterParams p)
{
    extern __shared__ float smem[];
    const int nc = p.nc;
    float *gl = smem;             // [nc]
    float *ks = smem + nc;        // [2nc-1]
    const size_t line = blockIdx.x;
    const float *src = p.g3 + line * nc;
    for (int t = threadIdx.x; t < nc; t += blockDim.x) gl[t] = src[t];
    for (int t = threadIdx.x; t < 2 * nc - 1; t += blockDim.x) ks[t] = __ldg(p.hilbert + t);
    __syncthreads();
    for (int l = threadIdx.x; l < nc; l += blockDim.x) {
        float acc0 = 0.f, acc1 = 0.f;
        const float *kk = ks + l + nc - 1;
        int lp = (l & 1) ^ 1;
        for (; lp + 2 < nc; lp += 4) {
            acc0 = fmaf(kk[-lp], gl[lp], acc0);
            acc1 = fmaf(kk[-lp - 2], gl[lp + 2], acc1);
        }
        for (; lp < nc; lp += 2) acc0 = fmaf(kk[-lp], gl[lp], acc0);
        p.g4[line * nc + l] = acc0 + acc1;
    }
}

// ---------------------------------------------------------------------------
// K4: gF[v][m][l] = cos α_l · lerp_ψ(g4[v][·][l], ψ̂(α_l, w_m))   (Eqs. 13-15)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_bwd_rebin_cos(FilterParams p)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;
    const int v = blockIdx.z;
    if (l >= p.nc) return;
    const RebinEntry e = p.br[m * p.nc + l];
    float out = 0.f;
    if (e.idx >= 0) {
        const float *g = p.g4 + ((size_t)v * p.npsi + e.idx) * p.nc + l;
        float a = g[0], b = g[p.nc];
        out = __ldg(p.cos_alpha + l) * fmaf(e.frac, b - a, a);
    }
    p.gF[((size_t)v * p.nr + m) * p.nc + l] = out;
}

void launch_deriv_fwd_rebin(const FilterParams &p, cudaStream_t s)
{
    dim3 grid((p.nc + 127) / 128, p.npsi, p.n_views);
    k_deriv_fwd_rebin<<<grid, 128, 0, s>>>(p);
}

void launch_hilbert(const FilterParams &p, cudaStream_t s)
{
    size_t smem = sizeof(float) * (3 * (size_t)p.nc - 1);
    int threads = p.nc >= 256 ? 256 : ((p.nc + 31) / 32) * 32;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_hilbert_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    k_hilbert_direct<<<(unsigned)((size_t)p.n_views * p.npsi), threads, smem, s>>>(p);
}

void launch_bwd_rebin_cos(const FilterParams &p, cudaStream_t s)
{
    dim3 grid((p.nc + 127) / 128, p.nr, p.n_views);
    k_bwd_rebin_cos<<<grid, 128, 0, s>>>(p);
}

}  // namespace kats
