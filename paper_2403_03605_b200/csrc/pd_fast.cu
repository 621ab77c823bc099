// Fast-mode bond kernels on ELL families (sm_100a, FMA allowed).
//
// Fast mode: eta = ubar_p - ubar_e from per-element centroid
// displacements (sum of N u over the element's nodes, perifem.hpp:149-157
// regrouped), squared break test |xi + eta|^2 >= ((1 + s_crit) |xi|)^2 (no
// fp64 sqrt/div per bond), force -w c (xi . eta) xi summed in partner order.
// Both directed entries of a bond evaluate the same expression on exactly
// negated operands, so the two sides always agree on a break.
#include <stdexcept>
#include <string>

#include "pd_common.cuh"

namespace pmts {

#define PMTS_CUDA_F(x)                                                                   \
    do {                                                                                 \
        cudaError_t err_ = (x);                                                          \
        if (err_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(err_)); \
    } while (0)

constexpr int kFastThreads = 256;

template <int DIM>
__global__ void __launch_bounds__(kFastThreads) k_fast_ubar(DevPD d) {
    constexpr int NN = DIM == 2 ? 4 : 8;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    double s[DIM];
    for (int c = 0; c < DIM; ++c) s[c] = 0.0;
    for (int a = 0; a < NN; ++a) {
        const int node = __ldg(d.conn + (size_t)a * d.E + e);
        for (int c = 0; c < DIM; ++c) s[c] += d.rd[(size_t)node * DIM + c];
    }
    for (int c = 0; c < DIM; ++c) d.ubar[(size_t)e * DIM + c] = d.Nsh * s[c];
}

void launch_fast_ubar(const DevPD& d, cudaStream_t s) {
    const int blocks = (d.E + kFastThreads - 1) / kFastThreads;
    if (d.dim == 2) k_fast_ubar<2><<<blocks, kFastThreads, 0, s>>>(d);
    else k_fast_ubar<3><<<blocks, kFastThreads, 0, s>>>(d);
    PMTS_CUDA_F(cudaGetLastError());
}

template <int DIM>
__global__ void __launch_bounds__(kFastThreads) k_fast_bond(DevPD d, int step, int do_break) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    if (e < d.E) {
        const int E = d.E;
        double ue[DIM], ce[DIM], G[DIM];
        for (int c = 0; c < DIM; ++c) {
            ue[c] = d.ubar[(size_t)e * DIM + c];
            ce[c] = __ldg(d.cen + (size_t)c * E + e);
            G[c] = 0.0;
        }
        const double s1 = 1.0 + d.s_crit;
        int wcur = -1;
        uint32_t word = 0, word0 = 0;
        for (int k = 0; k < d.K; ++k) {
            const int p = __ldg(d.col + (size_t)k * E + e);
            if (p < 0) break;
            const int w = k >> 5;
            if (w != wcur) {
                if (wcur >= 0 && word != word0) d.mask[(size_t)wcur * E + e] = word;
                word = word0 = d.mask[(size_t)w * E + e];
                wcur = w;
            }
            const uint32_t bit = 1u << (k & 31);
            if (!(word & bit)) continue;
            double xi[DIM], eta[DIM];
            for (int c = 0; c < DIM; ++c) {
                xi[c] = __ldg(d.cen + (size_t)c * E + p) - ce[c];
                eta[c] = d.ubar[(size_t)p * DIM + c] - ue[c];
            }
            double dot = 0.0, x2 = 0.0, l2 = 0.0;
            for (int c = 0; c < DIM; ++c) {
                dot += xi[c] * eta[c];
                x2 += xi[c] * xi[c];
                const double y = xi[c] + eta[c];
                l2 += y * y;
            }
            const double t = __ldg(d.coef + (size_t)k * E + e) * dot;
            for (int c = 0; c < DIM; ++c) G[c] -= t * xi[c];
            if (do_break) {
                double sc = s1;
                if (d.spread != 0.0) {
                    const int lo = e < p ? e : p, hi = e < p ? p : e;
                    sc = 1.0 + bond_s_crit(d.s_crit, d.spread, d.seed, global_elem(d, lo), global_elem(d, hi));
                }
                if (l2 >= sc * sc * x2) {
                    word &= ~bit;
                    if (e < p && owns_elem(d, e)) ++nb;
                }
            }
        }
        if (wcur >= 0 && word != word0) d.mask[(size_t)wcur * E + e] = word;
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
    }
    if (do_break) {
        __shared__ unsigned long long part[kFastThreads / 32];
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = nb;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kFastThreads / 32; ++w) t += part[w];
            if (t) atomicAdd(d.broken_count + step, t);
        }
    }
}

void launch_fast_bond(const DevPD& d, int step, int do_break, cudaStream_t s) {
    const int blocks = (d.E + kFastThreads - 1) / kFastThreads;
    if (d.dim == 2) k_fast_bond<2><<<blocks, kFastThreads, 0, s>>>(d, step, do_break);
    else k_fast_bond<3><<<blocks, kFastThreads, 0, s>>>(d, step, do_break);
    PMTS_CUDA_F(cudaGetLastError());
}

}  // namespace pmts
