/* ORACLE / TEST INFRASTRUCTURE ONLY -- not product code.
 *
 * CPU restatement (plain C, -ffp-contract=off) of the reference's PD fine-step
 * path, used only by tests/, bench.py's cpu_baseline leg and
 * __graft_entry__.smoke() as the checker.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/).
 *
 * Two step variants:
 *   PO_CSR -- the reference's own arithmetic: node-block CSR K^PD assembled in
 *             PE order, row SpMV in column order, downdates in broken (pe,qp)
 *             order.  Pinned bitwise against the reference (tests/golden).
 *   PO_MF  -- matrix-free gather in the order the CUDA deterministic kernel
 *             uses; equal to PO_CSR up to
 *             summation rounding and bitwise to the device.
 */
#ifndef PD_ORACLE_H
#define PD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PO_CSR = 0, PO_MF = 1 };
enum { PO_MICRO_EXP = 0, PO_MICRO_CONST = 1 };

/* prm[]: 0 delta, 1 l, 2 c0, 3 c_const, 4 h, 5 s_crit, 6 s_crit_spread,
 *        7 gamma, 8 beta, 9 dt
 * iprm[]: 0 micromodulus kind, 1 seed (per-bond s_crit factor), 2 variant,
 *         3 global id of local element 0 (slab decomposition tests),
 *         4, 5 elements per z layer, local and global (3D slabs cut along y; 0 = contiguous) */
typedef struct po_pd po_pd;

/* mesh.hpp:416-495 (find_pe_pairs) incl. notch predicates mesh.hpp:324-404.
 * notch_pts: n_notch notches, notch k has notch_npts[k] points (xyz each).
 * Returns the number of pairs; writes min(cap, n) (i,j) rows when out != 0. */
int64_t po_find_pairs(int dim, int n_elems, const double* centroid, const double* volume,
                      double delta, int n_notch, const int32_t* notch_npts,
                      const double* notch_pts, int32_t* out, int64_t cap);

po_pd* po_pd_create(int dim, int n_nodes, int n_elems, const int32_t* conn,
                    const double* centroid, const double* volume, int64_t n_pairs,
                    const int32_t* pairs, const double* mass, const double* p_ext, int n_bc,
                    const int32_t* bc_dofs, const double* bc_vel, const double* prm,
                    const int64_t* iprm);
void po_pd_destroy(po_pd* h);
/* newmark.hpp:110-116 -- a0 = (P*scale0 - K u0)/M, constrained rows 0 */
void po_pd_init(po_pd* h, double scale0);
/* n steps of driver_run.hpp:216-236; scales[k] = load_scale(t_k).
 * broken_out (optional, cap entries): pair indices in (step, pe) order;
 * broken_step (optional): step (1-based within this call) of each entry.
 * Returns number of newly broken bonds (all, even beyond cap). */
int64_t po_pd_step(po_pd* h, int n, const double* scales, int32_t* broken_out,
                   int32_t* broken_step, int64_t cap);
void po_pd_get_state(const po_pd* h, double* u, double* v, double* a);
void po_pd_set_state(po_pd* h, const double* u, const double* v, const double* a);
void po_pd_get_mu(const po_pd* h, uint8_t* mu);
/* perifem.hpp:202-231 */
void po_pd_damage(const po_pd* h, double* elem, double* node);
/* micromodulus material.hpp:84-88 (exp) or the BASELINE constant form */
double po_micromodulus(const po_pd* h, double r);
/* per-bond critical stretch (BASELINE cfg3 extension; spread 0 = scalar) */
double po_bond_s_crit(double s_crit, double spread, uint64_t seed, int32_t i, int32_t j);
/* perifem.hpp:144-166 for one pair (i<j) on displacement u */
double po_bond_stretch(const po_pd* h, int64_t pair, const double* u);
int64_t po_pd_nnz(const po_pd* h);
/* update_bond_states (perifem.hpp:170-193) on u; returns newly broken pairs */
int64_t po_pd_update_bond_states(po_pd* h, const double* u, int32_t* out, int64_t cap);
void po_pd_set_mu(po_pd* h, const uint8_t* mu);

#ifdef __cplusplus
}
#endif
#endif
