// Host-side setup of the coupled multi-time-step (Arlequin) run behind
// pmts_mts_create (include/pmts_capi.h) -- SURVEY.md 8(f) row 1.
//
// Native C++ restatement of the reference's coupled build, compiled with
// -ffp-contract=off so every assembled value (alpha weights, the FE stiffness
// in CSR, lumped masses, surface loads, coupling rows) is bit-identical to the
// reference's; tests/test_mts_setup.py pins that against the reference's own
// dump (oracle/ref_mts_driver).  Citations: /root/reference/proj/include/perimts/.
//   build_scenario coupled part       driver.hpp:211-222
//   label_subdomains / region          mesh.hpp:509-627
//   WeightFunction                     coupling.hpp:25-41
//   elastic_matrix                     material.hpp:55-81
//   element_stiffness / lumped_mass    fem.hpp:133-179
//   boundary_faces / face tractions    fem.hpp:229-337
//   build_dof_map / assemble_global    fem.hpp:381-474
//   SparseMatrix::from_triplets        linalg.hpp:102-155
//   M, P of assemble_pd_global         perifem.hpp:331-349
//   resolve_bcs_quiet                  driver.hpp:133-150
//   build_coupling_map                 coupling.hpp:72-105
#include "pmts_mts_setup.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <map>

namespace pmts {

namespace {

bool box_contains(const MtsBox& b, const double* p, int dim, double tol = 0.0) {
    for (int k = 0; k < dim; ++k)
        if (p[k] < b.lo[k] - tol || p[k] > b.hi[k] + tol) return false;
    return true;
}

// BoundsBox::distance (mesh.hpp:152-159)
double box_distance(const MtsBox& b, const double* p, int dim) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) {
        const double d = std::max({b.lo[k] - p[k], p[k] - b.hi[k], 0.0});
        s += d * d;
    }
    return std::sqrt(s);
}

bool box_empty(const MtsBox& b, int dim) {
    for (int k = 0; k < dim; ++k)
        if (b.hi[k] <= b.lo[k]) return true;
    return false;
}

// detail::shrunk_box (mesh.hpp:524-535)
MtsBox shrunk_box(const MtsBox& box, const MtsSystem& s) {
    MtsBox core = box;
    const double tol = 1e-9 * std::max(1.0, s.overlap_width);
    for (int k = 0; k < s.dim; ++k) {
        if (box.lo[k] > s.domain.lo[k] + tol) core.lo[k] += s.overlap_width;
        if (box.hi[k] < s.domain.hi[k] - tol) core.hi[k] -= s.overlap_width;
    }
    return core;
}

bool inside_pd(const MtsSystem& s, const double* p) {
    for (const auto& b : s.pd_boxes)
        if (box_contains(b, p, s.dim)) return true;
    return false;
}

// region_distance_to_core (mesh.hpp:553-571), boxes only
double distance_to_core(const MtsSystem& s, const double* p) {
    double d = 1e300;
    for (const auto& b : s.pd_boxes) {
        const MtsBox core = shrunk_box(b, s);
        if (!box_empty(core, s.dim)) d = std::min(d, box_distance(core, p, s.dim));
    }
    return d;
}

// build_dof_map (fem.hpp:392-411)
void dof_map(const MtsSystem& s, const std::vector<int>& active, std::vector<int32_t>& node_dof,
             int& n_dof, std::vector<int>& active_nodes) {
    const int nn = s.dim == 2 ? 4 : 8;
    const int N = int(s.nodes.size() / 3);
    node_dof.assign(N, -1);
    for (int e : active)
        for (int a = 0; a < nn; ++a) node_dof[s.conn[std::size_t(e) * nn + a]] = 0;
    n_dof = 0;
    active_nodes.clear();
    for (int n = 0; n < N; ++n) {
        if (node_dof[n] == 0) {
            node_dof[n] = n_dof;
            n_dof += s.dim;
            active_nodes.push_back(n);
        } else {
            node_dof[n] = -1;
        }
    }
}

// elastic_matrix (material.hpp:55-81), row-major
std::vector<double> elastic_matrix(double E, double nu, int formulation, int& rows) {
    if (formulation == 0) {
        rows = 3;
        std::vector<double> d(9, 0.0);
        const double f = E / (1.0 - nu * nu);
        d[0] = d[4] = f;
        d[1] = d[3] = f * nu;
        d[8] = f * (1.0 - nu) / 2.0;
        return d;
    }
    if (std::abs(1.0 - 2.0 * nu) < 1e-12) throw ConfigError("nu = 0.5 is singular for plane strain / 3D");
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    if (formulation == 1) {
        rows = 3;
        std::vector<double> d(9, 0.0);
        d[0] = d[4] = lam + 2.0 * mu;
        d[1] = d[3] = lam;
        d[8] = mu;
        return d;
    }
    rows = 6;
    std::vector<double> d(36, 0.0);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) d[i * 6 + j] = i == j ? lam + 2.0 * mu : lam;
    for (int i = 3; i < 6; ++i) d[i * 6 + i] = mu;
    return d;
}

std::vector<std::array<double, 3>> gauss_points(int dim) {
    const double g = 1.0 / std::sqrt(3.0);
    std::vector<std::array<double, 3>> pts;
    if (dim == 2) {
        for (int j = 0; j < 2; ++j)
            for (int i = 0; i < 2; ++i) pts.push_back({i ? g : -g, j ? g : -g, 0.0});
    } else {
        for (int k = 0; k < 2; ++k)
            for (int j = 0; j < 2; ++j)
                for (int i = 0; i < 2; ++i) pts.push_back({i ? g : -g, j ? g : -g, k ? g : -g});
    }
    return pts;
}

// shape_and_gradients (fem.hpp:51-97): physical gradients and detJ
void shape_gradients(const MtsSystem& s, const int32_t* en, const double* xi, double dNdx[8][3],
                     double& detJ) {
    const int d = s.dim, nn = d == 2 ? 4 : 8;
    double gref[8][3];
    for (int a = 0; a < nn; ++a) corner_gradient(d, xi, a, gref[a]);
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 0; a < nn; ++a) {
        const double* p = s.nodes.data() + 3 * std::size_t(en[a]);
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) J[i][j] += p[i] * gref[a][j];
    }
    double inv[3][3];
    if (d == 2) {
        detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        if (detJ <= 0.0) throw ConfigError("inverted element (non-positive Jacobian)");
        const double r = 1.0 / detJ;
        inv[0][0] = J[1][1] * r;
        inv[0][1] = -J[0][1] * r;
        inv[1][0] = -J[1][0] * r;
        inv[1][1] = J[0][0] * r;
    } else {
        detJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
               J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
               J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        if (detJ <= 0.0) throw ConfigError("inverted element (non-positive Jacobian)");
        const double r = 1.0 / detJ;
        inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * r;
        inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
        inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
        inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * r;
        inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
        inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
        inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * r;
        inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
        inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
    }
    for (int a = 0; a < nn; ++a)
        for (int i = 0; i < d; ++i) {
            double v = 0.0;
            for (int j = 0; j < d; ++j) v += gref[a][j] * inv[j][i];
            dNdx[a][i] = v;
        }
}

// element_stiffness (fem.hpp:156-167) with strain_matrix (fem.hpp:118-146)
std::vector<double> element_stiffness(const MtsSystem& s, const int32_t* en,
                                      const std::vector<double>& D, int rows) {
    const int dim = s.dim, nn = dim == 2 ? 4 : 8, ndof = dim * nn;
    std::vector<double> k(std::size_t(ndof) * ndof, 0.0), b(std::size_t(rows) * ndof),
        db(std::size_t(rows) * ndof);
    for (const auto& xi : gauss_points(dim)) {
        double dNdx[8][3], detJ;
        shape_gradients(s, en, xi.data(), dNdx, detJ);
        std::fill(b.begin(), b.end(), 0.0);
        for (int a = 0; a < nn; ++a) {
            const int c = dim * a;
            if (dim == 2) {
                b[0 * ndof + c] = dNdx[a][0];
                b[1 * ndof + c + 1] = dNdx[a][1];
                b[2 * ndof + c] = dNdx[a][1];
                b[2 * ndof + c + 1] = dNdx[a][0];
            } else {
                b[0 * ndof + c] = dNdx[a][0];
                b[1 * ndof + c + 1] = dNdx[a][1];
                b[2 * ndof + c + 2] = dNdx[a][2];
                b[3 * ndof + c] = dNdx[a][1];
                b[3 * ndof + c + 1] = dNdx[a][0];
                b[4 * ndof + c + 1] = dNdx[a][2];
                b[4 * ndof + c + 2] = dNdx[a][1];
                b[5 * ndof + c] = dNdx[a][2];
                b[5 * ndof + c + 2] = dNdx[a][0];
            }
        }
        for (int i = 0; i < rows; ++i)
            for (int j = 0; j < ndof; ++j) {
                double v = 0.0;
                for (int r = 0; r < rows; ++r) v += D[std::size_t(i) * rows + r] * b[std::size_t(r) * ndof + j];
                db[std::size_t(i) * ndof + j] = v;
            }
        for (int i = 0; i < ndof; ++i)
            for (int j = 0; j < ndof; ++j) {
                double v = 0.0;
                for (int r = 0; r < rows; ++r) v += b[std::size_t(r) * ndof + i] * db[std::size_t(r) * ndof + j];
                k[std::size_t(i) * ndof + j] += v * detJ;
            }
    }
    return k;
}

// lumped_mass (fem.hpp:172-179)
std::array<double, 8> lumped_mass(const MtsSystem& s, const int32_t* en, double rho) {
    std::array<double, 8> m{};
    const int nn = s.dim == 2 ? 4 : 8;
    for (const auto& xi : gauss_points(s.dim)) {
        double dNdx[8][3], detJ;
        shape_gradients(s, en, xi.data(), dNdx, detJ);
        for (int a = 0; a < nn; ++a) m[a] += rho * shape_value(s.dim, xi.data(), a) * detJ;
    }
    return m;
}

struct Face {
    int element = -1;
    std::array<int, 4> nodes{};
    int nn = 0;
    double center[3] = {0, 0, 0};
};

// boundary_faces (fem.hpp:229-266): faces referenced once, sorted by node list
std::vector<Face> boundary_faces(const MtsSystem& s) {
    static const int quad_edges[4][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}};
    static const int hex_faces[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4},
                                        {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
    const int dim = s.dim, nn = dim == 2 ? 4 : 8;
    const int E = int(s.volume.size());
    std::map<std::array<int, 4>, std::pair<int, Face>> faces;
    for (int e = 0; e < E; ++e) {
        const int32_t* en = s.conn.data() + std::size_t(e) * nn;
        const int nf = dim == 2 ? 4 : 6;
        for (int f = 0; f < nf; ++f) {
            Face bf;
            bf.element = e;
            bf.nn = dim == 2 ? 2 : 4;
            for (int a = 0; a < bf.nn; ++a)
                bf.nodes[a] = en[dim == 2 ? quad_edges[f][a] : hex_faces[f][a]];
            std::array<int, 4> key = bf.nodes;
            std::sort(key.begin(), key.begin() + bf.nn);
            for (int a = bf.nn; a < 4; ++a) key[a] = -1;
            auto [it, inserted] = faces.try_emplace(key, std::make_pair(0, bf));
            ++it->second.first;
        }
    }
    std::vector<Face> out;
    for (auto& [key, entry] : faces) {
        if (entry.first != 1) continue;
        Face& bf = entry.second;
        for (int k = 0; k < 3; ++k) bf.center[k] = 0.0;
        for (int a = 0; a < bf.nn; ++a)
            for (int k = 0; k < 3; ++k) bf.center[k] += s.nodes[3 * std::size_t(bf.nodes[a]) + k] / bf.nn;
        out.push_back(bf);
    }
    std::sort(out.begin(), out.end(), [](const Face& a, const Face& b) { return a.nodes < b.nodes; });
    return out;
}

// integrate_face_traction (fem.hpp:294-337)
void face_traction(const MtsSystem& s, const Face& face, const double* t,
                   std::vector<std::pair<int, std::array<double, 3>>>& out) {
    if (s.dim == 2) {
        const double* a = s.nodes.data() + 3 * std::size_t(face.nodes[0]);
        const double* b = s.nodes.data() + 3 * std::size_t(face.nodes[1]);
        double d2 = 0.0;
        for (int k = 0; k < 3; ++k) d2 += (a[k] - b[k]) * (a[k] - b[k]);
        const double len = std::sqrt(d2);
        for (int n = 0; n < 2; ++n)
            out.push_back({face.nodes[n], {t[0] * len / 2, t[1] * len / 2, t[2] * len / 2}});
        return;
    }
    const double g = 1.0 / std::sqrt(3.0);
    std::array<double, 4> nodal{};
    for (int q = 0; q < 4; ++q) {
        const double xi = (q & 1) ? g : -g, eta = (q & 2) ? g : -g;
        const double N[4] = {0.25 * (1 - xi) * (1 - eta), 0.25 * (1 + xi) * (1 - eta),
                             0.25 * (1 + xi) * (1 + eta), 0.25 * (1 - xi) * (1 + eta)};
        const double dxi[4] = {-0.25 * (1 - eta), 0.25 * (1 - eta), 0.25 * (1 + eta),
                               -0.25 * (1 + eta)};
        const double deta[4] = {-0.25 * (1 - xi), -0.25 * (1 + xi), 0.25 * (1 + xi),
                                0.25 * (1 - xi)};
        double tu[3] = {0, 0, 0}, tv[3] = {0, 0, 0};
        for (int a = 0; a < 4; ++a) {
            const double* p = s.nodes.data() + 3 * std::size_t(face.nodes[a]);
            for (int k = 0; k < 3; ++k) {
                tu[k] += dxi[a] * p[k];
                tv[k] += deta[a] * p[k];
            }
        }
        const double cx = tu[1] * tv[2] - tu[2] * tv[1];
        const double cy = tu[2] * tv[0] - tu[0] * tv[2];
        const double cz = tu[0] * tv[1] - tu[1] * tv[0];
        const double dA = std::sqrt(cx * cx + cy * cy + cz * cz);
        for (int a = 0; a < 4; ++a) nodal[a] += N[a] * dA;
    }
    for (int a = 0; a < 4; ++a)
        out.push_back({face.nodes[a], {t[0] * nodal[a], t[1] * nodal[a], t[2] * nodal[a]}});
}

// add_surface_loads (fem.hpp:344-378), tractions only (pressure patches are out
// of scope)
void surface_loads(const MtsSystem& s, const std::vector<Face>& faces,
                   const std::vector<int32_t>& node_dof, bool pd_side, bool require_hit,
                   std::vector<double>& p_ext) {
    if (s.tractions.empty()) return;
    const double tol = 1e-12 * s.cl;
    std::vector<std::pair<int, std::array<double, 3>>> nodal;
    for (const auto& patch : s.tractions) {
        bool hit = false;
        for (const auto& f : faces) {
            if (!box_contains(patch.box, f.center, s.dim, tol)) continue;
            if (node_dof[f.nodes[0]] < 0) continue;
            const double w = pd_side ? 1.0 - s.alpha[f.element] : s.alpha[f.element];
            nodal.clear();
            face_traction(s, f, patch.value, nodal);
            for (const auto& [node, force] : nodal)
                for (int ci = 0; ci < s.dim; ++ci) p_ext[node_dof[node] + ci] += w * force[ci];
            hit = true;
        }
        if (!hit && require_hit) throw ConfigError("traction patch selects no boundary face");
    }
}

struct Triplet {
    int row, col;
    double value;
};

// SparseMatrix::from_triplets (linalg.hpp:102-155): counting sort by row, per
// row std::sort by column (the same library sort on the same sequence, so the
// same summation order of duplicates), merge, drop exact zeros
void csr_from_triplets(int n, const std::vector<Triplet>& triplets, std::vector<int32_t>& rowptr,
                       std::vector<int32_t>& col, std::vector<double>& val) {
    std::vector<int> count(n, 0);
    for (const auto& t : triplets) {
        if (t.row < 0 || t.row >= n || t.col < 0 || t.col >= n)
            throw ConfigError("sparse assembly: index out of range");
        ++count[t.row];
    }
    std::vector<int> ptr(n + 1, 0);
    for (int i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + count[i];
    std::vector<int> cursor(ptr.begin(), ptr.end() - 1);
    std::vector<int> cols(triplets.size());
    std::vector<double> vals(triplets.size());
    for (const auto& t : triplets) {
        const int p = cursor[t.row]++;
        cols[p] = t.col;
        vals[p] = t.value;
    }
    col.clear();
    val.clear();
    col.reserve(triplets.size());
    val.reserve(triplets.size());
    rowptr.assign(n + 1, 0);
    std::vector<std::pair<int, double>> row;
    for (int i = 0; i < n; ++i) {
        row.clear();
        for (int p = ptr[i]; p < ptr[i + 1]; ++p) row.emplace_back(cols[p], vals[p]);
        std::sort(row.begin(), row.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first; });
        std::size_t w = 0;
        for (std::size_t r = 0; r < row.size(); ++r) {
            if (w > 0 && row[w - 1].first == row[r].first) {
                row[w - 1].second += row[r].second;
            } else {
                row[w++] = row[r];
            }
        }
        for (std::size_t r = 0; r < w; ++r) {
            if (row[r].second == 0.0) continue;
            col.push_back(row[r].first);
            val.push_back(row[r].second);
        }
        rowptr[i + 1] = int32_t(col.size());
    }
}

// resolve_bcs_quiet (driver.hpp:133-150) on one subdomain's dof numbering
void resolve_bcs(const MtsSystem& s, const std::vector<int32_t>& node_dof,
                 const std::vector<int>& active_nodes, std::vector<int32_t>& dofs,
                 std::vector<double>& vel) {
    std::map<int, double> table;
    const double tol = 1e-9 * std::max(s.cl, 1e-300);
    for (const auto& bc : s.kinematic)
        for (int n : active_nodes) {
            if (!box_contains(bc.box, &s.nodes[3 * std::size_t(n)], s.dim, tol)) continue;
            if (bc.fix_all)
                for (int c = 0; c < s.dim; ++c) table[node_dof[n] + c] = 0.0;
            else
                table[node_dof[n] + bc.comp] = bc.vel;
        }
    dofs.clear();
    vel.clear();
    for (const auto& [dof, v] : table) {
        dofs.push_back(dof);
        vel.push_back(v);
    }
}

}  // namespace

// WeightFunction::operator() (coupling.hpp:31-40)
double mts_alpha_at(const MtsSystem& s, const double* x) {
    if (s.pd_boxes.empty()) return 1.0;
    if (!inside_pd(s, x)) return 1.0;
    const double l1 = distance_to_core(s, x);
    if (l1 <= 0.0) return 0.0;
    if (s.weight_kind == 0) return 0.5;
    const double r = std::min(l1 / s.overlap_width, 1.0);
    return s.weight_kind == 1 ? r : r * r * r;
}

void build_mts_system(MtsSystem& s) {
    const int dim = s.dim, nn = dim == 2 ? 4 : 8;
    const int N = int(s.nodes.size() / 3), E = int(s.volume.size());
    // build_scenario coupled part (driver.hpp:211-222): domain = mesh bounding box
    for (int k = 0; k < 3; ++k) {
        s.domain.lo[k] = 1e300;
        s.domain.hi[k] = -1e300;
    }
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < 3; ++k) {
            s.domain.lo[k] = std::min(s.domain.lo[k], s.nodes[3 * std::size_t(n) + k]);
            s.domain.hi[k] = std::max(s.domain.hi[k], s.nodes[3 * std::size_t(n) + k]);
        }
    s.overlap_width = s.overlap_width_factor * s.cl;
    // label_subdomains (mesh.hpp:599-626)
    if (s.pd_boxes.empty()) throw ConfigError("subdomain labeling needs a PD region");
    if (s.overlap_width <= 0.0) throw ConfigError("overlap width must be positive");
    s.label.assign(E, 0);
    s.node_in_overlap.assign(N, 0);
    int n_overlap = 0, n_pd = 0;
    for (int e = 0; e < E; ++e) {
        const double* c = s.centroid.data() + 3 * std::size_t(e);
        if (!inside_pd(s, c)) continue;
        if (distance_to_core(s, c) == 0.0) {
            s.label[e] = 1;
            ++n_pd;
        } else {
            s.label[e] = 2;
            ++n_overlap;
            // coupling rows sit on the PD side's overlap nodes
            if (s.fe_mesh_elems < 0 || e >= s.fe_mesh_elems)
                for (int a = 0; a < nn; ++a) s.node_in_overlap[s.conn[std::size_t(e) * nn + a]] = 1;
        }
    }
    if (n_pd + n_overlap == 0) throw ConfigError("PD region contains no elements");
    if (n_overlap == 0) throw ConfigError("overlap must contain at least one element layer");
    if (n_pd == 0) throw ConfigError("PD region must keep a core beyond the overlap bands");
    s.alpha.resize(E);
    for (int e = 0; e < E; ++e) s.alpha[e] = mts_alpha_at(s, s.centroid.data() + 3 * std::size_t(e));
    s.node_alpha.resize(N);
    for (int n = 0; n < N; ++n) s.node_alpha[n] = mts_alpha_at(s, s.nodes.data() + 3 * std::size_t(n));
    s.fe_active.clear();
    s.pd_active.clear();
    for (int e = 0; e < E; ++e) {
        const bool fe_mesh = s.fe_mesh_elems < 0 || e < s.fe_mesh_elems;
        const bool pd_mesh = s.fe_mesh_elems < 0 || e >= s.fe_mesh_elems;
        if (s.label[e] != 1 && fe_mesh) s.fe_active.push_back(e);
        if (s.label[e] != 0 && pd_mesh) s.pd_active.push_back(e);
    }
    if (s.fe_mesh_elems >= 0 && (s.fe_active.empty() || s.pd_active.empty()))
        throw ConfigError("non-matching coupling: an empty FE or PD subdomain");

    const auto faces = boundary_faces(s);
    // tractions must select some boundary face overall (driver.hpp:195-209)
    {
        const double ftol = 1e-12 * s.cl;
        for (const auto& p : s.tractions) {
            bool covered = false;
            for (const auto& f : faces)
                if (box_contains(p.box, f.center, dim, ftol)) {
                    covered = true;
                    break;
                }
            if (!covered) throw ConfigError("traction patch selects no boundary face");
        }
    }

    // ---- FE: assemble_global (fem.hpp:421-474) ----
    dof_map(s, s.fe_active, s.fe_node_dof, s.fe_n_dof, s.fe_active_nodes);
    int rows = 0;
    const std::vector<double> D = elastic_matrix(s.E, s.nu, s.formulation, rows);
    std::vector<Triplet> triplets;
    s.fe_mass.assign(s.fe_n_dof, 0.0);
    s.fe_p_ext.assign(s.fe_n_dof, 0.0);
    const int ndof_e = dim * nn;
    for (int eid : s.fe_active) {
        const int32_t* en = s.conn.data() + std::size_t(eid) * nn;
        const std::vector<double> blk = element_stiffness(s, en, D, rows);
        const std::array<double, 8> masses = lumped_mass(s, en, s.rho);
        const double a = s.alpha[eid];
        if (a <= 0.0) {
            if (s.label[eid] == 0) throw InternalError("zero weight on an FE-only element");
            if (a < 0.0) throw InternalError("negative weight on an element");
        }
        for (int p = 0; p < nn; ++p) {
            const int prow = s.fe_node_dof[en[p]];
            for (int q = 0; q < nn; ++q) {
                const int qcol = s.fe_node_dof[en[q]];
                for (int ci = 0; ci < dim; ++ci)
                    for (int cj = 0; cj < dim; ++cj)
                        triplets.push_back({prow + ci, qcol + cj,
                                            a * blk[std::size_t(dim * p + ci) * ndof_e + dim * q + cj]});
            }
            for (int ci = 0; ci < dim; ++ci) s.fe_mass[prow + ci] += a * masses[p];
            double b[3] = {s.body_force[0], s.body_force[1], s.body_force[2]};
            const double* c = s.centroid.data() + 3 * std::size_t(eid);
            for (const auto& patch : s.body_patches)
                if (box_contains(patch.box, c, dim))
                    for (int ci = 0; ci < dim; ++ci) b[ci] += patch.value[ci];
            for (int ci = 0; ci < dim; ++ci) s.fe_p_ext[prow + ci] += a * b[ci] * masses[p] / s.rho;
        }
    }
    csr_from_triplets(s.fe_n_dof, triplets, s.fe_rowptr, s.fe_col, s.fe_val);
    surface_loads(s, faces, s.fe_node_dof, false, false, s.fe_p_ext);

    // ---- PD: M and P of assemble_pd_global (perifem.hpp:331-350) ----
    dof_map(s, s.pd_active, s.pd_node_dof, s.pd_n_dof, s.pd_active_nodes);
    s.pd_mass.assign(s.pd_n_dof, 0.0);
    s.pd_p_ext.assign(s.pd_n_dof, 0.0);
    for (int eid : s.pd_active) {
        const int32_t* en = s.conn.data() + std::size_t(eid) * nn;
        const double w = 1.0 - s.alpha[eid];
        const std::array<double, 8> masses = lumped_mass(s, en, s.rho);
        double b[3] = {s.body_force[0], s.body_force[1], s.body_force[2]};
        const double* c = s.centroid.data() + 3 * std::size_t(eid);
        for (const auto& patch : s.body_patches)
            if (box_contains(patch.box, c, dim))
                for (int ci = 0; ci < dim; ++ci) b[ci] += patch.value[ci];
        for (int a = 0; a < nn; ++a) {
            const int base = s.pd_node_dof[en[a]];
            for (int ci = 0; ci < dim; ++ci) {
                s.pd_mass[base + ci] += w * masses[a];
                s.pd_p_ext[base + ci] += w * b[ci] * masses[a] / s.rho;
            }
        }
    }
    surface_loads(s, faces, s.pd_node_dof, true, false, s.pd_p_ext);

    // ---- kinematic constraints per subdomain, coupling rows ----
    {
        const double tol = 1e-9 * std::max(s.cl, 1e-300);
        for (const auto& bc : s.kinematic) {
            bool hit = false;
            for (int n = 0; n < N && !hit; ++n) hit = box_contains(bc.box, &s.nodes[3 * std::size_t(n)], dim, tol);
            if (!hit) throw ConfigError("kinematic constraint selects no node");
        }
    }
    resolve_bcs(s, s.fe_node_dof, s.fe_active_nodes, s.fe_bc_dofs, s.fe_bc_vel);
    resolve_bcs(s, s.pd_node_dof, s.pd_active_nodes, s.pd_bc_dofs, s.pd_bc_vel);
    // build_coupling_map (coupling.hpp:72-105); non-matching: the row of a PD overlap
    // node interpolates the FE velocity with the shape functions of the FE element
    // containing it (local coordinates from lattice indices: exact, so a PD node on
    // an FE node gets the single weight 1 -- the conforming map)
    s.cpl_fe.clear();
    s.cpl_pd.clear();
    s.cpl_fe_rp.assign(1, 0);
    s.cpl_fe_ci.clear();
    s.cpl_fe_w.clear();
    int n_on = 0;
    for (int n = 0; n < N; ++n) n_on += s.node_in_overlap[n];
    if (n_on == 0) throw ConfigError("empty overlap: no coupling possible");
    auto fe_bc = [&](int fd) {
        return std::binary_search(s.fe_bc_dofs.begin(), s.fe_bc_dofs.end(), fd);
    };
    for (int n = 0; n < N; ++n) {
        if (!s.node_in_overlap[n]) continue;
        if (s.pd_node_dof[n] < 0) throw InternalError("overlap node missing from the PD dof map");
        int fn[8], nfe = 0;  // FE nodes and weights of this row
        double fw[8];
        if (s.fe_mesh_elems < 0) {
            if (s.fe_node_dof[n] < 0)
                throw InternalError("overlap node missing from a subdomain dof map");
            fn[0] = n;
            fw[0] = 1.0;
            nfe = 1;
        } else {
            // PD node (lattice index) -> FE element and local coordinates
            const int q = n - s.fe_mesh_nodes;
            const int pnx = s.pd_n[0] + 1, pny = s.pd_n[1] + 1;
            const int pi[3] = {q % pnx, (q / pnx) % pny, q / (pnx * pny)};
            int ei[3] = {0, 0, 0}, li[3] = {0, 0, 0};
            for (int k = 0; k < dim; ++k) {
                // fine index on the FE lattice: (pd_lo - fe_lo) / pd_h + pi, an integer
                const long long g = std::llround((s.pd_lo[k] - s.fe_lo[k]) / s.pd_h) + pi[k];
                long long c = g / s.fe_ratio;
                if (c >= s.fe_n[k]) c = s.fe_n[k] - 1;  // the far face: last element
                ei[k] = int(c);
                li[k] = int(g - c * s.fe_ratio);  // 0 .. fe_ratio
            }
            // prefer an FE-active element among those sharing the point (ascending id)
            int best = -1;
            int cand[3][2], nc[3];
            for (int k = 0; k < 3; ++k) {
                nc[k] = 1;
                cand[k][0] = ei[k];
                if (k < dim && li[k] == 0 && ei[k] > 0) {
                    cand[k][0] = ei[k] - 1;
                    cand[k][1] = ei[k];
                    nc[k] = 2;
                }
            }
            int bl[3] = {0, 0, 0};
            for (int a = 0; a < nc[2] && best < 0; ++a)
                for (int b = 0; b < nc[1] && best < 0; ++b)
                    for (int c = 0; c < nc[0] && best < 0; ++c) {
                        const int ex = cand[0][c], ey = cand[1][b], ez = dim == 3 ? cand[2][a] : 0;
                        const int e = (ez * s.fe_n[1] + ey) * s.fe_n[0] + ex;
                        if (s.label[e] == 1) continue;  // FE-inactive (PD core)
                        best = e;
                        bl[0] = li[0] + (ex < ei[0] ? s.fe_ratio : 0);
                        bl[1] = li[1] + (ey < ei[1] ? s.fe_ratio : 0);
                        bl[2] = dim == 3 ? li[2] + (ez < ei[2] ? s.fe_ratio : 0) : 0;
                    }
            if (best < 0) throw ConfigError("a PD overlap node lies in no FE-active element");
            const int32_t* en = s.conn.data() + std::size_t(best) * nn;
            double xi[3] = {0, 0, 0};
            for (int k = 0; k < dim; ++k) xi[k] = 2.0 * bl[k] / s.fe_ratio - 1.0;  // exact
            for (int a = 0; a < nn; ++a) {
                const double w = shape_value(dim, xi, a);
                if (w == 0.0) continue;
                fn[nfe] = en[a];
                fw[nfe] = w;
                ++nfe;
            }
        }
        for (int c = 0; c < dim; ++c) {
            const int pdof = s.pd_node_dof[n] + c;
            if (std::binary_search(s.pd_bc_dofs.begin(), s.pd_bc_dofs.end(), pdof)) continue;
            bool all_bc = true;
            for (int a = 0; a < nfe; ++a) {
                if (s.fe_node_dof[fn[a]] < 0) throw InternalError("FE node without a dof");
                all_bc = all_bc && fe_bc(s.fe_node_dof[fn[a]] + c);
            }
            if (all_bc) continue;
            s.cpl_fe.push_back(s.fe_node_dof[fn[0]] + c);
            s.cpl_pd.push_back(pdof);
            for (int a = 0; a < nfe; ++a) {
                s.cpl_fe_ci.push_back(s.fe_node_dof[fn[a]] + c);
                s.cpl_fe_w.push_back(fw[a]);
            }
            s.cpl_fe_rp.push_back(int32_t(s.cpl_fe_ci.size()));
        }
    }
    if (s.cpl_fe.empty()) throw ConfigError("empty overlap: all coupling rows constrained");
    // BlockOperator ctor checks (newmark.hpp:84-93)
    auto check_mass = [](const std::vector<double>& M, const std::vector<int32_t>& bc) {
        for (std::size_t i = 0; i < M.size(); ++i)
            if (M[i] <= 0.0 && !std::binary_search(bc.begin(), bc.end(), int32_t(i)))
                throw SolverError("non-positive lumped mass at dof " + std::to_string(i));
    };
    check_mass(s.fe_mass, s.fe_bc_dofs);
    check_mass(s.pd_mass, s.pd_bc_dofs);
}

}  // namespace pmts
