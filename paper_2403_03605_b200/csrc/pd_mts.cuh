// Launchers of the MTS integrator kernels (pd_mts.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pmts {
struct DevPD;
namespace mtsk {

// PD substep kernels of the integrator: warp-per-element K^PD x (optional bond
// test into mask / cnt), node sum fused with the explicit solve, the predictor
// fused with zeroing the load, and scaled multiplier rows.
// Q / S (E x 2^dim x dim and E x 8 scratch, or null): the per-element node products
// computed once per call instead of per family entry -- bitwise the same force
void pd_force_warp(const DevPD& d, const double* x, uint32_t* mask, int do_break,
                   unsigned long long* cnt, cudaStream_t s, double* Q = nullptr,
                   double* S = nullptr, const int32_t* colT = nullptr,
                   const double* coefT = nullptr);  // colT / coefT: entry-major families
// linear (no bond test) K^PD x via centroid displacements; ubar: E x dim scratch
void pd_force_lin(const DevPD& d, const double* x, const uint32_t* mask, double* ubar,
                  cudaStream_t s);
void pd_node_explicit(const DevPD& d, const double* ra, double ra_scale, const double* M,
                      const uint8_t* cf, const double* rv, const double* rd, double gdt,
                      double bdt2, const double* bcvel, int homog, double* u, double* v,
                      double* a, cudaStream_t s);
void pd_node_lin(const DevPD& d, int with_force, const double* w, const int32_t* row_of, double f,
                 const double* M, const uint8_t* cf, double gdt, double bdt2, double dt, double cpv,
                 double cpd, double* u, double* v, double* a, double* rd, double* rv, double* out,
                 cudaStream_t s);
void pd_pre(int n, const double* u, const double* v, const double* a, double* rd, double* rv,
            double* ra, double dt, double cpv, double cpd, cudaStream_t s);
void scatter_scaled(int n, const int32_t* idx, const double* w, double f, double* dst,
                    cudaStream_t s);

void csr_spmv(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
              double* y, cudaStream_t s);
void predict(int n, const double* u, const double* v, const double* a, double* rd, double* rv,
             double dt, double cpv, double cpd, cudaStream_t s);
// ra (nullable) is scaled by ra_scale; homog: constrained velocities 0 instead of bcvel
void explicit_solve(int n, const double* ra, double ra_scale, const double* kd, const double* M,
                    const uint8_t* cf, const double* rv, const double* rd, double gdt, double bdt2,
                    const double* bcvel, int homog, double* u, double* v, double* a,
                    cudaStream_t s);
void rhs(int n, const double* ra, double ra_scale, const double* kd, const uint8_t* cf, double* b,
         cudaStream_t s);
void apply_a(int n, const double* x, const double* kx, const double* M, const uint8_t* cf,
             double bdt2, double* y, cudaStream_t s);
void finish(int n, const double* acc, const double* rv, const double* rd, double gdt, double bdt2,
            const uint8_t* cf, const double* bcvel, int homog, double* u, double* v, double* a,
            cudaStream_t s);
void zero_constrained(int n, const uint8_t* cf, double* x, cudaStream_t s);
void init_acc(int n, const double* p, const double* ku, const double* M, const uint8_t* cf,
              double* a, cudaStream_t s);
void scatter_add(int n, const int32_t* idx, const double* vals, double* dst, cudaStream_t s);
// idx[r] < 0: no load (scatter_add) / -0.0 (gather) -- rows a shard does not own
void gather(int n, const int32_t* idx, const double* src, double* dst, cudaStream_t s);
void fill(long long n, double v, double* x, cudaStream_t s);
// dst[didx[i]] = src[sidx[i]]; dst[idx[i]] = vals[i]
void copy_idx(int n, const double* src, const int32_t* sidx, double* dst, const int32_t* didx,
              cudaStream_t s);
void scatter_set(int n, const int32_t* idx, const double* vals, double* dst, cudaStream_t s);
void gather_csr(int n, const int32_t* rp, const int32_t* ci, const double* w, const double* src,
                double* dst, cudaStream_t s);
void scatter_csr(int nt, const int32_t* td, const int32_t* trp, const int32_t* tri,
                 const double* tw, const double* vals, double* dst, cudaStream_t s);
void scale(int n, const double* x, double sc, double* y, cudaStream_t s);
void add(int n, const double* x, double* y, cudaStream_t s);  // y += x
void add_states(int n, const double* a0, const double* a1, const double* a2, const double* b0,
                const double* b1, const double* b2, double* o0, double* o1, double* o2,
                cudaStream_t s);
void cg_update(int n, const double* alpha_dev, const double* p, const double* ap, double* x,
               double* r, cudaStream_t s);
void precond(int n, const double* r, const double* jac, double* z, cudaStream_t s);
void xpby(int n, const double* z, const double* beta_dev, double* p, cudaStream_t s);
int dot_partials();
void dot(int n, const double* x, const double* y, double* part, double* out, cudaStream_t s);
void ratio(const double* num, const double* den, double* out, cudaStream_t s);
// entry-major families (colT, coefT: E K; xiT: E K dim) and the linear force on them
void family_transpose(const DevPD& d, int32_t* colT, double* coefT, cudaStream_t s);
void pd_force_lin_t(const DevPD& d, const int32_t* colT, const double* coefT, const double* x,
                    const uint32_t* mask, double* ubar, cudaStream_t s);
// the same linear force on a 3D box lattice in lattice order (pd_mts_lat.cu): the
// coefficients in stencil order, the snapshot's bond states as stencil bits
struct LinLat {
    int nx = 0, ny = 0, nz = 0;
    double h = 0.0;
    double* coefS = nullptr;     // [61 E]: the positive offsets' coefficients
    uint32_t* maskS = nullptr;   // [4 E]
    const int8_t* slot = nullptr;  // [7^3] offset -> stencil slot (-1: none), device
};
void lin_lat_slot_table(int8_t* table343);
int lin_lat_stencil_size();
int lin_lat_coef_slots();
bool lin_lat_build(const DevPD& d, const LinLat& L, cudaStream_t s);  // false: an entry off the
                                                                     // stencil or an unsymmetric bond
void lin_lat_mask(const DevPD& d, const LinLat& L, const uint32_t* mask, cudaStream_t s);
void pd_force_lin_lat(const DevPD& d, const LinLat& L, const double* x, double* ubar,
                      cudaStream_t s);
void pd_ubar(const DevPD& d, const double* x, double* ubar, cudaStream_t s);
void iface_jac_csr(int n, const int32_t* rp, const int32_t* ci, const double* hv, int m,
                   double dt_pd, const int32_t* cpd, const double* Mpd, double* jd,
                   cudaStream_t s);
// the CG loop test on the device (conditional WHILE graph node); it_status: {iterations, status}
void cg_cond(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr,
             const double* s_pap, double tol, int max_iter, int* it_status, cudaStream_t s);
// fused CG steps (bitwise the unfused sequence): dot(s) + the CG scalar in one launch
// (part: 2 dot_partials() doubles, ticket: a zeroed counter), update + precondition
void dot_fin(int n, const double* x, const double* y, const double* x2, const double* y2,
             double* part, unsigned* ticket, double* out, double* out2, int mode, double* num,
             double* sc, cudaStream_t s);
void cg_update_precond(int n, const double* alpha_dev, const double* p, const double* ap,
                       double* x, double* r, const double* jac, double* z, cudaStream_t s);
void dense_matvec(int n, const double* A, const double* x, double* y, cudaStream_t s);
void csr_spmv_warp(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                   double* y, cudaStream_t s);

// coupled-step bookkeeping on the device (pd_mts.cu): S_j rows, interface rhs,
// energy terms, continuity maxima (as double bits), dense LU, H_FE assembly
void s_vectors(int nl, int m, double t, double dt_pd, double dt_fe, double ramp,
               const double* lamp, const double* gpfe, double* sv, cudaStream_t s);
void sub_idx(int n, const int32_t* idx, const double* x, double* b, cudaStream_t s);
void neg(int n, const double* x, double* y, cudaStream_t s);
void sub2(int n, const double* a, const double* b, double* o, cudaStream_t s);
void quad_w(int n, const double* da, const double* M, double f, const double* kda, double* w,
            cudaStream_t s);
void lpd_terms(int nl, int m, const double* gpf, const double* gpl, const double* sv,
               const double* lamp, const double* lam, double* A, double* B, cudaStream_t s);
void max_abs(int n, const double* x, const int32_t* idx, const double* y,
             unsigned long long* out, cudaStream_t s);
void lu_factor(int n, double* A, int* perm, unsigned long long* amax, int* flag, cudaStream_t s);
void lu_solve(int n, const double* A, const int* perm, const double* b, double* x, cudaStream_t s);
// more_out (nullable): the loop flag for a host-driven loop instead of the WHILE condition
void cg_start(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr, double tol,
              int max_iter, int* it_status, double* x, int n, cudaStream_t s,
              int* more_out = nullptr);
void col_neg(int n, int k, const double* x, double* D, cudaStream_t s);
void add_col_gather(int n, int k, const int32_t* idx, const double* x, double* H, cudaStream_t s);
void unit_row(int nf, const int32_t* rp, const int32_t* ci, const double* w, int k, double* ra,
              cudaStream_t s);
void unit_vec(int n, int k, double* x, cudaStream_t s);
// H_FE of an explicit FE side directly as CSR (candidates crp / cci, values bitwise the
// unit-column construction; exact zeros kept), then the nonzeros counted / compacted
void hfe_explicit(int nl, const long long* crp, const int32_t* cci, const int32_t* grp,
                  const int32_t* gci, const double* gw, const double* M, const uint8_t* cf,
                  double gdt, double* vals, cudaStream_t s);
void nz_count(int n, const long long* rp, const double* v, int* cnt, cudaStream_t s);
void nz_fill(int n, const long long* rp, const int32_t* ci, const double* v, const int32_t* orp,
             int32_t* oci, double* ov, cudaStream_t s);
void transpose(int n, const double* D, double* H, cudaStream_t s);
void row_nnz(int n, const double* D, int* cnt, cudaStream_t s);
void row_fill(int n, const double* D, const int* rp, int32_t* ci, double* v, cudaStream_t s);
void iface_jac(int n, const double* D, int m, double dt_pd, const int32_t* cpd, const double* Mpd,
               double* jd, cudaStream_t s);
// the implicit-FE unit columns k0 .. k0 + B - 1 of H_FE as B simultaneous CG solves
// (see pd_mts.cu); returns 0 or the first failing column's CG status
int batched_unit_columns(int nf, int nl, int k0, int B, const int32_t* krp, const int32_t* kci,
                         const double* kv, const double* M, const uint8_t* cf, const double* jac,
                         double bdt2, double gdt, const int32_t* grp, const int32_t* gci,
                         const double* gw, double tol, int max_iter, double* scratch, double* part,
                         double* sc, int* act, int* stat, int* n_active, int* h_count, double* D,
                         int* iters_out, cudaStream_t s);
int batched_partials();
// x[idx[i]] = 1 (i < n); dst[slots[i]] = g[rows[i]] (H_PD columns by colour)
void set_ones(int n, const int32_t* idx, double* x, cudaStream_t s);
void gather_slots(int n, const int32_t* rows, const int64_t* slots, const double* g, double* dst,
                  cudaStream_t s);
// C = A + B for two CSR matrices with sorted rows (count, then fill into rp from the
// exclusive scan of the counts); the diagonal of a CSR matrix (non-positive -> 0)
void merge_count(int n, const int32_t* arp, const int32_t* aci, const int32_t* brp,
                 const int32_t* bci, int* cnt, cudaStream_t s);
void merge_fill(int n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                const int32_t* bci, const double* bv, const int32_t* rp, int32_t* ci, double* v,
                cudaStream_t s);
void csr_diag(int n, const int32_t* rp, const int32_t* ci, const double* v, double* d,
              cudaStream_t s);
// fused CG stages: the implicit FE operator in one pass; the update + preconditioner +
// r.z / r.r + beta + the loop test (bitwise k_cg_update_precond, k_dot_fin mode 2 and
// k_cg_cond in sequence)
void csr_apply_a(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                 const double* M, const uint8_t* cf, double bdt2, double* y, cudaStream_t s);
void cg_update_dots(int n, const double* alpha_dev, const double* p, const double* ap, double* x,
                    double* r, const double* jac, double* z, double* part, unsigned* ticket,
                    double* s_rzn, double* s_rr, double* s_rz, double* s_beta, const double* s_bb,
                    const double* s_pap, double tol, int max_iter, int* it_status,
                    cudaGraphConditionalHandle h, cudaStream_t s, int* more_out = nullptr);
// the CG operator fused with p.Ap and alpha (part: pap_partials() doubles, ticket zeroed)
int pap_partials(int n, bool warp_rows);
void csr_apply_a_pap(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                     const double* M, const uint8_t* cf, double bdt2, double* y, double* part,
                     unsigned* ticket, double* s_pap, const double* s_rz, double* s_alpha,
                     cudaStream_t s);
void csr_warp_pap(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                  double* y, double* part, unsigned* ticket, double* s_pap, const double* s_rz,
                  double* s_alpha, cudaStream_t s);

}  // namespace mtsk
}  // namespace pmts
