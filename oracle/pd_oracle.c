/* ORACLE / TEST INFRASTRUCTURE ONLY -- not product code.  See pd_oracle.h.
 *
 * Plain-C restatement of the reference's pure-PD (PeriFEM, one-point
 * quadrature) fine step.  Built with -ffp-contract=off so every expression
 * rounds exactly as the reference's.  Citations are
 * /root/reference/proj/<path>:<line>.
 */
#define _POSIX_C_SOURCE 200809L
#include "pd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MAXNN 8

struct po_pd {
    int dim, n_nodes, n_elems, nn, n_dof, variant, kind;
    int64_t n_pairs;
    const int32_t* conn_in;
    int32_t* conn;
    double *cen, *vol;
    int32_t* pairs;
    double *M, *P, *bc_vel;
    int32_t* bc_dofs;
    int n_bc;
    uint8_t* constrained;
    /* per pair (QuadPair, perifem.hpp:19-26) */
    double *xi, *xin, *w, *coef, *scrit;
    uint8_t* mu;
    /* kinematics (newmark.hpp:32-37) */
    double *u, *v, *a, *rd, *rv, *b;
    int32_t* brk;
    /* CSR (linalg.hpp:98-297) */
    int32_t *rp, *col;
    double* val;
    /* matrix-free families */
    int32_t *fptr, *fcol, *fpair, *nptr, *nel;
    double* G;
    double delta, l, c0, c_const, h, s_crit, spread, gamma, beta, dt, N;
    uint64_t seed;
    int64_t goff, id_pl, id_pg;
};

/* ------------------------------------------------------------------ */
/* geometry predicates: mesh.hpp:21-24, 322-404                        */

static double dist3(const double* a, const double* b) {
    const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

static double cross2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }
static double dmax(double a, double b) { return a < b ? b : a; }

/* mesh.hpp:324-347 */
static int segments_intersect_2d(const double* p1, const double* p2, const double* q1,
                                 const double* q2, double eps) {
    const double rx = p2[0] - p1[0], ry = p2[1] - p1[1];
    const double sx = q2[0] - q1[0], sy = q2[1] - q1[1];
    const double denom = cross2(rx, ry, sx, sy);
    const double qpx = q1[0] - p1[0], qpy = q1[1] - p1[1];
    const double tn = cross2(qpx, qpy, sx, sy);
    const double un = cross2(qpx, qpy, rx, ry);
    if (fabs(denom) > eps * eps) {
        const double t = tn / denom;
        const double u = un / denom;
        const double tol_t = eps / dmax(hypot(rx, ry), eps);
        const double tol_u = eps / dmax(hypot(sx, sy), eps);
        return t >= -tol_t && t <= 1.0 + tol_t && u >= -tol_u && u <= 1.0 + tol_u;
    }
    if (fabs(tn) > eps * dmax(hypot(sx, sy), eps)) return 0;
    const double rr = rx * rx + ry * ry;
    if (rr < eps * eps) return 0;
    double t0 = (qpx * rx + qpy * ry) / rr;
    double t1 = t0 + (sx * rx + sy * ry) / rr;
    if (t0 > t1) {
        const double s = t0;
        t0 = t1;
        t1 = s;
    }
    return t1 >= 0.0 && t0 <= 1.0;
}

/* mesh.hpp:349-395 */
static int segment_crosses_polygon_3d(const double* a, const double* b, const double* poly,
                                      int nv, double eps) {
    const double* o = poly;
    const double u[3] = {poly[3] - o[0], poly[4] - o[1], poly[5] - o[2]};
    const double v[3] = {poly[6] - o[0], poly[7] - o[1], poly[8] - o[2]};
    double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                   u[0] * v[1] - u[1] * v[0]};
    const double nlen = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (nlen == 0.0) return 0;
    for (int k = 0; k < 3; ++k) n[k] /= nlen;
    const double da = (a[0] - o[0]) * n[0] + (a[1] - o[1]) * n[1] + (a[2] - o[2]) * n[2];
    const double db = (b[0] - o[0]) * n[0] + (b[1] - o[1]) * n[1] + (b[2] - o[2]) * n[2];
    if ((da > eps && db > eps) || (da < -eps && db < -eps)) return 0;
    if (fabs(da - db) < eps) return 0;
    const double t = da / (da - db);
    if (t < -eps || t > 1.0 + eps) return 0;
    const double p[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]),
                         a[2] + t * (b[2] - a[2])};
    int drop = 0;
    double best = fabs(n[0]);
    for (int k = 1; k < 3; ++k)
        if (fabs(n[k]) > best) {
            best = fabs(n[k]);
            drop = k;
        }
    const int i0 = (drop + 1) % 3, i1 = (drop + 2) % 3;
    int inside = 0;
    for (int e = 0, f = nv - 1; e < nv; f = e++) {
        const double xi = poly[3 * e + i0], yi = poly[3 * e + i1];
        const double xj = poly[3 * f + i0], yj = poly[3 * f + i1];
        const double ex = xj - xi, ey = yj - yi;
        const double px = p[i0] - xi, py = p[i1] - yi;
        const double elen2 = ex * ex + ey * ey;
        if (elen2 > 0.0) {
            double s = (px * ex + py * ey) / elen2;
            s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
            const double ddx = px - s * ex, ddy = py - s * ey;
            if (ddx * ddx + ddy * ddy <= eps * eps) return 1;
        }
        if ((yi > p[i1]) != (yj > p[i1]) && p[i0] < (xj - xi) * (p[i1] - yi) / (yj - yi) + xi)
            inside = !inside;
    }
    return inside;
}

/* ------------------------------------------------------------------ */
/* mesh.hpp:416-495 find_pe_pairs                                      */

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int64_t po_find_pairs(int dim, int n_elems, const double* cen, const double* vol, double delta,
                      int n_notch, const int32_t* notch_npts, const double* notch_pts,
                      int32_t* out, int64_t cap) {
    if (delta <= 0.0 || n_elems <= 0) return 0;
    /* Mesh::char_length mesh.hpp:51-57 */
    double vs = 0.0;
    for (int e = 0; e < n_elems; ++e) vs += vol[e];
    vs /= (double)n_elems;
    const double cl = dim == 2 ? sqrt(vs) : cbrt(vs);
    const double eps = 1e-12 * dmax(cl, 1e-300);
    double lo[3] = {1e300, 1e300, 1e300};
    for (int e = 0; e < n_elems; ++e)
        for (int k = 0; k < 3; ++k)
            if (cen[3 * e + k] < lo[k]) lo[k] = cen[3 * e + k];
    /* cell_of mesh.hpp:441-446 -- dense grid over the occupied cell range */
    int* cell = (int*)malloc(sizeof(int) * 3 * (size_t)n_elems);
    int cmax[3] = {0, 0, 0};
    for (int e = 0; e < n_elems; ++e)
        for (int k = 0; k < 3; ++k) {
            int c = 0;
            if (k < dim) c = (int)floor((cen[3 * e + k] - lo[k]) / delta);
            cell[3 * e + k] = c;
            if (c > cmax[k]) cmax[k] = c;
        }
    const int64_t gx = cmax[0] + 1, gy = cmax[1] + 1, gz = cmax[2] + 1;
    const int64_t ncell = gx * gy * gz;
    int64_t* start = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
    int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_elems);
    for (int e = 0; e < n_elems; ++e)
        start[((int64_t)cell[3 * e + 2] * gy + cell[3 * e + 1]) * gx + cell[3 * e] + 1]++;
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
    memcpy(cur, start, sizeof(int64_t) * (size_t)ncell);
    for (int e = 0; e < n_elems; ++e)
        ids[cur[((int64_t)cell[3 * e + 2] * gy + cell[3 * e + 1]) * gx + cell[3 * e]]++] = e;
    free(cur);

    int64_t total = 0;
    int32_t buf[4096];
    const int zr = dim == 3 ? 1 : 0;
    for (int i = 0; i < n_elems; ++i) {
        const double* ci = cen + 3 * i;
        int nb = 0;
        for (int dz = -zr; dz <= zr; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t cx = cell[3 * i] + dx, cy = cell[3 * i + 1] + dy,
                                  cz = cell[3 * i + 2] + dz;
                    if (cx < 0 || cy < 0 || cz < 0 || cx >= gx || cy >= gy || cz >= gz) continue;
                    const int64_t c = (cz * gy + cy) * gx + cx;
                    for (int64_t s = start[c]; s < start[c + 1]; ++s) {
                        const int j = ids[s];
                        if (j <= i) continue;
                        const double* cj = cen + 3 * j;
                        if (dist3(ci, cj) > delta) continue;
                        int cut = 0;
                        const double* np = notch_pts;
                        for (int q = 0; q < n_notch && !cut; ++q) {
                            const int npts = notch_npts[q];
                            if (npts == 2) cut = segments_intersect_2d(ci, cj, np, np + 3, eps);
                            else if (npts >= 3) cut = segment_crosses_polygon_3d(ci, cj, np, npts, eps);
                            np += 3 * npts;
                        }
                        if (cut) continue;
                        if (nb < 4096) buf[nb++] = j;
                    }
                }
        qsort(buf, (size_t)nb, sizeof(int32_t), cmp_i32);
        for (int k = 0; k < nb; ++k) {
            if (out && total < cap) {
                out[2 * total] = i;
                out[2 * total + 1] = buf[k];
            }
            ++total;
        }
    }
    free(cell);
    free(start);
    free(ids);
    return total;
}

/* ------------------------------------------------------------------ */
/* per-bond critical stretch (BASELINE cfg3 extension)       */

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

double po_bond_s_crit(double s_crit, double spread, uint64_t seed, int32_t i, int32_t j) {
    if (spread == 0.0) return s_crit;
    const uint64_t key = ((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)j;
    const uint64_t hv = splitmix64(seed ^ splitmix64(key));
    const double u = (double)(hv >> 11) * 0x1.0p-53;
    const double factor = (1.0 - spread) + (2.0 * spread) * u;
    return s_crit * factor;
}

/* material.hpp:84-88; constant form c h / r^3 (2D) or c / r^3 (3D) */
double po_micromodulus(const po_pd* h, double r) {
    if (r > h->delta) return 0.0;
    if (h->kind == PO_MICRO_CONST) {
        const double r3 = (r * r) * r;
        return (h->dim == 2 ? h->c_const * h->h : h->c_const) / r3;
    }
    return h->c0 * exp(-r / h->l);
}

/* ------------------------------------------------------------------ */
/* CSR helpers: linalg.hpp:169-207                                      */

static void add_at(po_pd* h, int i, int j, double v) {
    int lo = h->rp[i], hi = h->rp[i + 1];
    while (lo < hi) { /* std::lower_bound */
        const int mid = lo + (hi - lo) / 2;
        if (h->col[mid] < j) lo = mid + 1;
        else hi = mid;
    }
    if (lo == h->rp[i + 1] || h->col[lo] != j) abort();
    h->val[lo] += v;
}

/* perifem.hpp:106-116 + 243-268 (scatter_pe_block) */
static void scatter_pe(po_pd* h, int64_t q, double coeff) {
    const int d = h->dim, nn = h->nn;
    const int ei = h->pairs[2 * q], ej = h->pairs[2 * q + 1];
    const double f = coeff * h->w[q] * h->coef[q];
    if (f == 0.0) return;
    double g[48];
    int rows[48];
    const double N = h->N;
    for (int a = 0; a < nn; ++a)
        for (int c = 0; c < d; ++c) {
            g[d * a + c] = N * h->xi[3 * q + c];
            rows[d * a + c] = h->conn[nn * ej + a] * d + c;
        }
    for (int a = 0; a < nn; ++a)
        for (int c = 0; c < d; ++c) {
            g[d * (nn + a) + c] = -N * h->xi[3 * q + c];
            rows[d * (nn + a) + c] = h->conn[nn * ei + a] * d + c;
        }
    const int ndof = 2 * d * nn;
    for (int r = 0; r < ndof; ++r) {
        const double gr = f * g[r];
        if (gr == 0.0) continue;
        for (int c = 0; c < ndof; ++c) {
            const double v = gr * g[c];
            if (v != 0.0) add_at(h, rows[r], rows[c], v);
        }
    }
}

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* perifem.hpp:285-315 pattern, then 317-329 scatter */
static void build_csr(po_pd* h) {
    const int d = h->dim, nn = h->nn, N = h->n_nodes;
    int* cnt = (int*)calloc((size_t)N, sizeof(int));
    for (int64_t q = 0; q < h->n_pairs; ++q)
        for (int s = 0; s < 2; ++s) {
            const int e = h->pairs[2 * q + s];
            for (int a = 0; a < nn; ++a) cnt[h->conn[nn * e + a]] += 2 * nn;
        }
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * ((size_t)N + 1));
    off[0] = 0;
    for (int n = 0; n < N; ++n) off[n + 1] = off[n] + cnt[n];
    int* adj = (int*)malloc(sizeof(int) * (size_t)off[N]);
    memset(cnt, 0, sizeof(int) * (size_t)N);
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        int nodes[16];
        int k = 0;
        for (int a = 0; a < nn; ++a) nodes[k++] = h->conn[nn * h->pairs[2 * q] + a];
        for (int a = 0; a < nn; ++a) nodes[k++] = h->conn[nn * h->pairs[2 * q + 1] + a];
        for (int r = 0; r < k; ++r)
            for (int c = 0; c < k; ++c) adj[off[nodes[r]] + cnt[nodes[r]]++] = nodes[c];
    }
    int* ulen = (int*)malloc(sizeof(int) * (size_t)N);
    int64_t nnz = 0;
    for (int n = 0; n < N; ++n) {
        int* row = adj + off[n];
        qsort(row, (size_t)cnt[n], sizeof(int), cmp_int);
        int w = 0;
        for (int r = 0; r < cnt[n]; ++r)
            if (w == 0 || row[w - 1] != row[r]) row[w++] = row[r];
        ulen[n] = w;
        nnz += (int64_t)w * d * d;
    }
    h->rp = (int32_t*)malloc(sizeof(int32_t) * ((size_t)h->n_dof + 1));
    h->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)nnz);
    h->val = (double*)calloc((size_t)nnz, sizeof(double));
    int64_t pos = 0;
    h->rp[0] = 0;
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < d; ++c) {
            for (int r = 0; r < ulen[n]; ++r)
                for (int cc = 0; cc < d; ++cc) h->col[pos++] = adj[off[n] + r] * d + cc;
            h->rp[n * d + c + 1] = (int32_t)pos;
        }
    free(cnt);
    free(off);
    free(adj);
    free(ulen);
    for (int64_t q = 0; q < h->n_pairs; ++q)
        if (h->mu[q]) scatter_pe(h, q, 1.0);
}

/* matrix-free families: per element ascending partners; per node ascending elements */
static void build_families(po_pd* h) {
    const int E = h->n_elems, N = h->n_nodes, nn = h->nn;
    h->fptr = (int32_t*)calloc((size_t)E + 1, sizeof(int32_t));
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        h->fptr[h->pairs[2 * q] + 1]++;
        h->fptr[h->pairs[2 * q + 1] + 1]++;
    }
    for (int e = 0; e < E; ++e) h->fptr[e + 1] += h->fptr[e];
    h->fcol = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)h->n_pairs + 4);
    h->fpair = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)h->n_pairs + 4);
    int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (size_t)E + 4);
    memcpy(cur, h->fptr, sizeof(int32_t) * (size_t)E);
    /* pairs sorted by (i,j): partners p<e arrive (from (p,e)) before p>e, each ascending */
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        const int i = h->pairs[2 * q], j = h->pairs[2 * q + 1];
        (void)i;
        h->fcol[cur[j]] = h->pairs[2 * q];
        h->fpair[cur[j]++] = (int32_t)q;
    }
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        const int i = h->pairs[2 * q];
        h->fcol[cur[i]] = h->pairs[2 * q + 1];
        h->fpair[cur[i]++] = (int32_t)q;
    }
    free(cur);
    h->nptr = (int32_t*)calloc((size_t)N + 1, sizeof(int32_t));
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < nn; ++a) h->nptr[h->conn[nn * e + a] + 1]++;
    for (int n = 0; n < N; ++n) h->nptr[n + 1] += h->nptr[n];
    h->nel = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->nptr[N] + 4);
    int32_t* nc = (int32_t*)malloc(sizeof(int32_t) * (size_t)N + 4);
    memcpy(nc, h->nptr, sizeof(int32_t) * (size_t)N);
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < nn; ++a) h->nel[nc[h->conn[nn * e + a]]++] = e;
    free(nc);
    h->G = (double*)calloc((size_t)E * 3, sizeof(double));
}

/* global element id of local element l: contiguous slabs add goff; 3D slabs cut
 * along y map layer by layer */
static int64_t global_id(const po_pd* h, int64_t l) {
    return h->id_pl ? (l / h->id_pl) * h->id_pg + h->goff + l % h->id_pl : l + h->goff;
}

po_pd* po_pd_create(int dim, int n_nodes, int n_elems, const int32_t* conn, const double* cen,
                    const double* vol, int64_t n_pairs, const int32_t* pairs, const double* mass,
                    const double* p_ext, int n_bc, const int32_t* bc_dofs, const double* bc_vel,
                    const double* prm, const int64_t* iprm) {
    po_pd* h = (po_pd*)calloc(1, sizeof(po_pd));
    h->dim = dim;
    h->nn = dim == 2 ? 4 : 8;
    h->N = dim == 2 ? 0.25 : 0.125; /* reference_shape at the centre, fem.hpp:22-47 */
    h->n_nodes = n_nodes;
    h->n_elems = n_elems;
    h->n_dof = n_nodes * dim;
    h->n_pairs = n_pairs;
    h->delta = prm[0];
    h->l = prm[1];
    h->c0 = prm[2];
    h->c_const = prm[3];
    h->h = prm[4];
    h->s_crit = prm[5];
    h->spread = prm[6];
    h->gamma = prm[7];
    h->beta = prm[8];
    h->dt = prm[9];
    h->kind = (int)iprm[0];
    h->seed = (uint64_t)iprm[1];
    h->variant = (int)iprm[2];
    h->goff = iprm[3]; /* global id of local element 0 (slab tests) */
    h->id_pl = iprm[4]; /* 3D slabs cut along y: local / global elements per z layer */
    h->id_pg = iprm[5];
    const size_t nd = (size_t)h->n_dof;
    h->conn = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_elems * h->nn);
    memcpy(h->conn, conn, sizeof(int32_t) * (size_t)n_elems * h->nn);
    h->cen = (double*)malloc(sizeof(double) * 3 * (size_t)n_elems);
    memcpy(h->cen, cen, sizeof(double) * 3 * (size_t)n_elems);
    h->vol = (double*)malloc(sizeof(double) * (size_t)n_elems);
    memcpy(h->vol, vol, sizeof(double) * (size_t)n_elems);
    h->pairs = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)n_pairs + 8);
    memcpy(h->pairs, pairs, sizeof(int32_t) * 2 * (size_t)n_pairs);
    h->M = (double*)malloc(sizeof(double) * nd);
    memcpy(h->M, mass, sizeof(double) * nd);
    h->P = (double*)malloc(sizeof(double) * nd);
    memcpy(h->P, p_ext, sizeof(double) * nd);
    h->n_bc = n_bc;
    h->bc_dofs = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n_bc + 1));
    h->bc_vel = (double*)malloc(sizeof(double) * ((size_t)n_bc + 1));
    if (n_bc) {
        memcpy(h->bc_dofs, bc_dofs, sizeof(int32_t) * (size_t)n_bc);
        memcpy(h->bc_vel, bc_vel, sizeof(double) * (size_t)n_bc);
    }
    h->constrained = (uint8_t*)calloc(nd, 1);
    for (int c = 0; c < n_bc; ++c) h->constrained[bc_dofs[c]] = 1;
    /* build_peri_elements perifem.hpp:87-97 (one-point rule) */
    const size_t P = (size_t)n_pairs + 1;
    h->xi = (double*)malloc(sizeof(double) * 3 * P);
    h->xin = (double*)malloc(sizeof(double) * P);
    h->w = (double*)malloc(sizeof(double) * P);
    h->coef = (double*)malloc(sizeof(double) * P);
    h->scrit = (double*)malloc(sizeof(double) * P);
    h->mu = (uint8_t*)malloc(P);
    h->brk = (int32_t*)malloc(sizeof(int32_t) * P);
    for (int64_t q = 0; q < n_pairs; ++q) {
        const int i = pairs[2 * q], j = pairs[2 * q + 1];
        double* x = h->xi + 3 * q;
        for (int k = 0; k < 3; ++k) x[k] = cen[3 * j + k] - cen[3 * i + k];
        h->xin[q] = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
        h->w[q] = vol[i] * vol[j];
        h->coef[q] = po_micromodulus(h, h->xin[q]);
        h->scrit[q] = po_bond_s_crit(h->s_crit, h->spread, h->seed, (int32_t)global_id(h, i),
                                     (int32_t)global_id(h, j));
        h->mu[q] = 1;
    }
    h->u = (double*)calloc(nd, sizeof(double));
    h->v = (double*)calloc(nd, sizeof(double));
    h->a = (double*)calloc(nd, sizeof(double));
    h->rd = (double*)calloc(nd, sizeof(double));
    h->rv = (double*)calloc(nd, sizeof(double));
    h->b = (double*)calloc(nd, sizeof(double));
    for (int c = 0; c < n_bc; ++c) h->v[bc_dofs[c]] = bc_vel[c];
    if (h->variant == PO_CSR) build_csr(h);
    else build_families(h);
    return h;
}

void po_pd_destroy(po_pd* h) {
    if (!h) return;
    void* ptrs[] = {h->conn, h->cen, h->vol, h->pairs, h->M, h->P, h->bc_dofs, h->bc_vel,
                    h->constrained, h->xi, h->xin, h->w, h->coef, h->scrit, h->mu, h->u, h->v,
                    h->a, h->rd, h->rv, h->b, h->rp, h->col, h->val, h->fptr, h->fcol, h->fpair,
                    h->nptr, h->nel, h->G, h->brk};
    for (size_t k = 0; k < sizeof(ptrs) / sizeof(ptrs[0]); ++k) free(ptrs[k]);
    free(h);
}

int64_t po_pd_nnz(const po_pd* h) { return h->rp ? h->rp[h->n_dof] : 0; }

/* perifem.hpp:144-166: eta = sum_j N u - sum_i N u in node order */
static double stretch_q(const po_pd* h, int64_t q, const double* u) {
    const int d = h->dim, nn = h->nn;
    const int ei = h->pairs[2 * q], ej = h->pairs[2 * q + 1];
    double eta[3] = {0, 0, 0};
    for (int a = 0; a < nn; ++a) {
        const int base = h->conn[nn * ej + a] * d;
        for (int c = 0; c < d; ++c) eta[c] += h->N * u[base + c];
    }
    for (int a = 0; a < nn; ++a) {
        const int base = h->conn[nn * ei + a] * d;
        for (int c = 0; c < d; ++c) eta[c] -= h->N * u[base + c];
    }
    double len2 = 0.0;
    for (int c = 0; c < d; ++c) {
        const double v = h->xi[3 * q + c] + eta[c];
        len2 += v * v;
    }
    const double len = sqrt(len2);
    if (len <= 0.0) return -1.0;
    return (len - h->xin[q]) / h->xin[q];
}

double po_bond_stretch(const po_pd* h, int64_t pair, const double* u) {
    return stretch_q(h, pair, u);
}

/* Independent-iteration loops over a few host threads (pthreads; no OpenMP
 * runtime in this image).  Every iteration writes only its own outputs, so the
 * results do not depend on the thread count.  PO_THREADS overrides the count. */
typedef struct { po_pd* h; const double* x; double* y; } mf_ctx;
typedef void (*range_fn)(void*, int64_t, int64_t);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } par_job;
static void* par_run(void* a) {
    par_job* j = (par_job*)a;
    j->fn(j->ctx, j->lo, j->hi);
    return 0;
}
static void par_for(int64_t n, range_fn fn, void* ctx) {
    static int nt = 0;
    if (!nt) {
        const char* e = getenv("PO_THREADS");
        nt = e ? atoi(e) : (int)sysconf(_SC_NPROCESSORS_ONLN);
        if (nt < 1) nt = 1;
        if (nt > 64) nt = 64;
    }
    int t = n < 65536 ? 1 : nt;
    if (t == 1) { fn(ctx, 0, n); return; }
    pthread_t th[64];
    par_job jb[64];
    for (int k = 0; k < t; ++k) {
        jb[k].fn = fn; jb[k].ctx = ctx;
        jb[k].lo = n * k / t; jb[k].hi = n * (k + 1) / t;
        if (k) pthread_create(&th[k], 0, par_run, &jb[k]);
    }
    par_run(&jb[0]);
    for (int k = 1; k < t; ++k) pthread_join(th[k], 0);
}
static void mf_elems(void* vc, int64_t e0, int64_t e1);
static void mf_nodes(void* vc, int64_t n0, int64_t n1);

/* K*x into y: CSR row sums in column order (linalg.hpp:209-221) or the
 * matrix-free element/node gathers (DESIGN.md deterministic order). */
static void apply_k(po_pd* h, const double* x, double* y) {
    if (h->variant == PO_CSR) {
        for (int r = 0; r < h->n_dof; ++r) {
            double s = 0.0;
            for (int p = h->rp[r]; p < h->rp[r + 1]; ++p) s += h->val[p] * x[h->col[p]];
            y[r] = s;
        }
        return;
    }
    /* per element / per node gathers are independent: threads change nothing */
    mf_ctx ctx = {h, x, y};
    par_for(h->n_elems, mf_elems, &ctx);
    par_for(h->n_nodes, mf_nodes, &ctx);
}

static void mf_elems(void* vc, int64_t e0, int64_t e1) {
    const mf_ctx* cx = (const mf_ctx*)vc;
    po_pd* h = cx->h;
    const double* x = cx->x;
    const int d = h->dim, nn = h->nn;
    for (int e = (int)e0; e < (int)e1; ++e) {
        double G[3] = {0.0, 0.0, 0.0};
        for (int k = h->fptr[e]; k < h->fptr[e + 1]; ++k) {
            const int64_t q = h->fpair[k];
            if (!h->mu[q]) continue;
            const int p = h->fcol[k];
            const int ei = p < e ? p : e, ej = p < e ? e : p;
            double eta[3] = {0, 0, 0};
            for (int a = 0; a < nn; ++a) {
                const int base = h->conn[nn * ej + a] * d;
                for (int c = 0; c < d; ++c) eta[c] += h->N * x[base + c];
            }
            for (int a = 0; a < nn; ++a) {
                const int base = h->conn[nn * ei + a] * d;
                for (int c = 0; c < d; ++c) eta[c] -= h->N * x[base + c];
            }
            const double* xi = h->xi + 3 * q;
            double dot = xi[0] * eta[0] + xi[1] * eta[1];
            if (d == 3) dot = dot + xi[2] * eta[2];
            const double t = h->coef[q] * h->w[q] * dot;
            for (int c = 0; c < d; ++c) {
                if (e == ej) G[c] = G[c] + t * xi[c];
                else G[c] = G[c] - t * xi[c];
            }
        }
        for (int c = 0; c < d; ++c) h->G[3 * e + c] = G[c];
    }
}

static void mf_nodes(void* vc, int64_t n0, int64_t n1) {
    const mf_ctx* cx = (const mf_ctx*)vc;
    const po_pd* h = cx->h;
    double* y = cx->y;
    const int d = h->dim;
    for (int n = (int)n0; n < (int)n1; ++n)
        for (int c = 0; c < d; ++c) {
            double s = 0.0;
            for (int k = h->nptr[n]; k < h->nptr[n + 1]; ++k)
                s = s + h->N * h->G[3 * h->nel[k] + c];
            y[n * d + c] = s;
        }
}

static void mark_breaks(void* vc, int64_t q0, int64_t q1) {
    po_pd* h = ((mf_ctx*)vc)->h;
    for (int64_t q = q0; q < q1; ++q)
        if (h->mu[q] && stretch_q(h, q, h->u) >= h->scrit[q]) h->mu[q] = 2;
}

void po_pd_init(po_pd* h, double scale0) {
    double* ku = h->b;
    apply_k(h, h->u, ku);
    for (int i = 0; i < h->n_dof; ++i) {
        const double p = h->P[i] * scale0;
        h->a[i] = h->constrained[i] ? 0.0 : (p - ku[i]) / h->M[i];
    }
}

int64_t po_pd_step(po_pd* h, int n, const double* scales, int32_t* broken_out,
                   int32_t* broken_step, int64_t cap) {
    const double dt = h->dt, gm = h->gamma, bt = h->beta;
    int64_t nb = 0;
    for (int s = 0; s < n; ++s) {
        /* newmark_predictor newmark.hpp:61-69 */
        for (int i = 0; i < h->n_dof; ++i) {
            h->rv[i] = h->v[i] + dt * (1.0 - gm) * h->a[i];
            h->rd[i] = h->u[i] + dt * h->v[i] + dt * dt * (0.5 - bt) * h->a[i];
        }
        /* BlockOperator::solve explicit branch newmark.hpp:122-159 */
        apply_k(h, h->rd, h->b);
        for (int i = 0; i < h->n_dof; ++i) {
            double pt = h->P[i];
            pt *= scales[s];
            const double bi = h->constrained[i] ? 0.0 : pt - h->b[i];
            const double acc = h->constrained[i] ? 0.0 : bi / h->M[i];
            h->a[i] = acc;
            h->v[i] = h->rv[i] + gm * dt * acc;
            h->u[i] = h->rd[i] + bt * dt * dt * acc;
        }
        for (int c = 0; c < h->n_bc; ++c) h->v[h->bc_dofs[c]] = h->bc_vel[c];
        /* update_bond_states perifem.hpp:170-193 (s >= s_crit inclusive) */
        if (!(h->s_crit > 0.0 && isfinite(h->s_crit))) continue;
        /* the per-pair test in parallel (mu 2 = breaks this step), then the
         * delta list in ascending pe order, as the reference appends it */
        mf_ctx bx = {h, 0, 0};
        par_for(h->n_pairs, mark_breaks, &bx);
        int64_t nnew = 0;
        for (int64_t q = 0; q < h->n_pairs; ++q)
            if (h->mu[q] == 2) {
                h->mu[q] = 0;
                h->brk[nnew++] = (int32_t)q;
            }
        /* incremental_stiffness_update perifem.hpp:356-364, broken (pe,qp) order */
        if (h->variant == PO_CSR)
            for (int64_t k = 0; k < nnew; ++k) scatter_pe(h, h->brk[k], -1.0);
        for (int64_t k = 0; k < nnew; ++k, ++nb)
            if (broken_out && nb < cap) {
                broken_out[nb] = h->brk[k];
                if (broken_step) broken_step[nb] = s + 1;
            }
    }
    return nb;
}

void po_pd_get_state(const po_pd* h, double* u, double* v, double* a) {
    const size_t nd = sizeof(double) * (size_t)h->n_dof;
    if (u) memcpy(u, h->u, nd);
    if (v) memcpy(v, h->v, nd);
    if (a) memcpy(a, h->a, nd);
}

void po_pd_set_state(po_pd* h, const double* u, const double* v, const double* a) {
    const size_t nd = sizeof(double) * (size_t)h->n_dof;
    if (u) memcpy(h->u, u, nd);
    if (v) memcpy(h->v, v, nd);
    if (a) memcpy(h->a, a, nd);
}

void po_pd_get_mu(const po_pd* h, uint8_t* mu) { memcpy(mu, h->mu, (size_t)h->n_pairs); }

/* perifem.hpp:202-231 */
void po_pd_damage(const po_pd* h, double* elem, double* node) {
    const int E = h->n_elems, N = h->n_nodes, nn = h->nn;
    double* total = (double*)calloc((size_t)E, sizeof(double));
    double* intact = (double*)calloc((size_t)E, sizeof(double));
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        const int i = h->pairs[2 * q], j = h->pairs[2 * q + 1];
        total[i] += h->w[q];
        total[j] += h->w[q];
        if (h->mu[q]) {
            intact[i] += h->w[q];
            intact[j] += h->w[q];
        }
    }
    int* count = (int*)calloc((size_t)N, sizeof(int));
    for (int e = 0; e < E; ++e) elem[e] = total[e] > 0.0 ? 1.0 - intact[e] / total[e] : 0.0;
    for (int n = 0; n < N; ++n) node[n] = 0.0;
    for (int e = 0; e < E; ++e) {
        if (total[e] == 0.0) continue;
        for (int a = 0; a < nn; ++a) {
            node[h->conn[nn * e + a]] += elem[e];
            ++count[h->conn[nn * e + a]];
        }
    }
    for (int n = 0; n < N; ++n)
        if (count[n] > 0) node[n] /= count[n];
    free(total);
    free(intact);
    free(count);
}

/* update_bond_states (perifem.hpp:170-193) on an explicit displacement */
int64_t po_pd_update_bond_states(po_pd* h, const double* u, int32_t* out, int64_t cap) {
    int64_t n = 0;
    for (int64_t q = 0; q < h->n_pairs; ++q) {
        if (!h->mu[q]) continue;
        if (stretch_q(h, q, u) >= h->scrit[q]) {
            h->mu[q] = 0;
            if (out && n < cap) out[n] = (int32_t)q;
            ++n;
        }
    }
    return n;
}

void po_pd_set_mu(po_pd* h, const uint8_t* mu) { memcpy(h->mu, mu, (size_t)h->n_pairs); }
