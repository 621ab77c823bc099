// Shared device-side declarations for the PD fine-step kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pmts {

// Device view of one PD handle.  SoA / ELL layouts:
//   conn[a*E + e]     node a of element e          (int32, 2^dim x E)
//   cen[k*E + e]      centroid component k          (fp64, 3 x E)
//   col[k*E + e]      k-th family partner of e, ascending, -1 padding (int32, K x E)
//   coef[k*E + e]     w c(|xi|) of that bond        (fp64, K x E; host-computed)
//   mask[w*E + e]     intact bits of e's entries    (uint32, W x E)
//   ne[a*N + n]       a-th incident element of node n, ascending, -1 padding
//   u,v,a,rd,rv,M,P   per dof n*dim + c (the reference's DofMap order)
struct DevPD {
    int dim, nn, E, N, K, W, NE;
    const int32_t* conn;
    const double* cen;
    const double* vol;
    const int32_t* col;
    const double* coef;
    uint32_t* mask;
    const int32_t* ne;
    double* u;
    double* v;
    double* a;
    double* rd;
    double* rv;
    const double* M;
    const double* P;
    const uint8_t* bcflag;  // per dof: 1 constrained
    const double* bcvel;    // per dof: prescribed velocity (constrained only)
    double* G;              // per element force (E x dim, AoS)
    double* ubar;           // per element centroid displacement (fast mode)
    double Nsh;             // shape value at the centre: 1/4 or 1/8
    double s_crit, spread;
    uint64_t seed;
    int fracture;
    long long goff;      // global id of local element 0 (slab decomposition)
    int own_lo, own_hi;  // owned local element range (broken counts, break log); with
                         // id_pl the in-layer range of l mod id_pl
    int id_pl;           // 3D slabs cut along y: local elements per z layer (0: contiguous)
    const double* extra;  // per dof: constraint load added to P * scale (coupled hooks; null: none)
    long long id_pg;     // ... and global elements per z layer
    // Newmark coefficients, each rounded exactly as the reference's expression
    double c_pred_v;  // dt*(1-gamma)              newmark.hpp:65
    double c_pred_d;  // (dt*dt)*(0.5-beta)        newmark.hpp:66
    double dt;        //                           newmark.hpp:66
    double c_corr_v;  // gamma*dt                  newmark.hpp:153
    double c_corr_d;  // (beta*dt)*dt              newmark.hpp:154
    unsigned long long* broken_count;  // per step slot
    int32_t* log;                      // (step, i, j) rows
    unsigned long long* log_n;
    int64_t log_cap;
};

// global element id of local element l (per-bond hash keys, break log): a contiguous
// slab adds goff; a 3D slab cut along y maps layer by layer
__host__ __device__ inline long long global_elem(const DevPD& d, long long l) {
    return d.id_pl ? (l / d.id_pl) * d.id_pg + d.goff + l % d.id_pl : l + d.goff;
}
// does this rank own local element l (broken counts, break log)
__host__ __device__ inline bool owns_elem(const DevPD& d, long long l) {
    const long long r = d.id_pl ? l % d.id_pl : l;
    return r >= d.own_lo && r < d.own_hi;
}

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Per-bond critical stretch, BASELINE cfg3 extension: factor
// U[1-spread, 1+spread] from a counter hash of (min id, max id, seed).
// Explicit _rn intrinsics: never contracted, bitwise equal to the oracle.
__device__ inline double bond_s_crit(double s_crit, double spread, uint64_t seed, long long i,
                                     long long j) {
    if (spread == 0.0) return s_crit;
    const uint64_t key = ((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)j;
    const uint64_t hv = splitmix64(seed ^ splitmix64(key));
    const double u = __dmul_rn((double)(hv >> 11), 0x1.0p-53);
    const double factor = __dadd_rn(1.0 - spread, __dmul_rn(2.0 * spread, u));
    return __dmul_rn(s_crit, factor);
}

// launchers (pd_det.cu)
void launch_det_bond(const DevPD& d, const double* disp, int step, int do_break, int global_step,
                     cudaStream_t s);
void launch_node_update(const DevPD& d, double scale, int predict_next, cudaStream_t s);
void launch_predict(const DevPD& d, cudaStream_t s);
void launch_damage_node(const DevPD& d, const double* elem, const uint8_t* has, double* node,
                        cudaStream_t s);
void launch_init_acc(const DevPD& d, double scale, cudaStream_t s);
void launch_node_force(const DevPD& d, double* kx, cudaStream_t s);
void launch_damage(const DevPD& d, double* elem, double* node, cudaStream_t s);
void launch_gather(const double* src, const int32_t* idx, int n, double* dst, cudaStream_t s);
void launch_track(const double* src, const int32_t* idx, int n, double* trk_host,
                  const unsigned long long* cnt_dev, unsigned long long* cnt_host,
                  const double* scl_host_next, double* scl_dev_next, cudaStream_t s);
// launchers (pd_fast.cu)
void launch_fast_ubar(const DevPD& d, cudaStream_t s);
void launch_fast_bond(const DevPD& d, int step, int do_break, cudaStream_t s);

// neighbour build (pd_families.cu)
struct FamilyBuild {
    int32_t* col;  // K x E ELL, device
    int K;
    int64_t n_entries;
};
FamilyBuild build_families_device(int dim, int E, const double* d_cen, const double lo[3],
                                  double delta, double eps, int n_notch, const int32_t* notch_npts,
                                  const double* notch_pts, cudaStream_t s);

}  // namespace pmts
