// Host-side scenario setup behind pmts_scenario_* (include/pmts_capi.h).
//
// Native C++ restatement of the reference's setup for a generated pure-PD run
// (once per run; the fine-step hot path is on the device).  Compiled with
// -ffp-contract=off so every value (centroids, volumes, masses, loads, c0) is
// bit-identical to the reference's; tests/test_setup_*.py pin that against the
// reference's own dumps.  Citations: /root/reference/proj/include/perimts/.
#include <algorithm>
#include <cstdlib>
#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <vector>

#include "pmts_internal.h"

namespace pmts {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

// corner_gradient (mesh.hpp:74-89) == reference_shape gradients (fem.hpp:22-47)
void corner_gradient(int dim, const double* xi, int a, double* g) {
    if (dim == 2) {
        static const double sx[4] = {-1, 1, 1, -1};
        static const double sy[4] = {-1, -1, 1, 1};
        g[0] = 0.25 * sx[a] * (1 + sy[a] * xi[1]);
        g[1] = 0.25 * sy[a] * (1 + sx[a] * xi[0]);
        g[2] = 0.0;
    } else {
        static const double sx[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
        static const double sy[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
        static const double sz[8] = {-1, -1, -1, -1, 1, 1, 1, 1};
        g[0] = 0.125 * sx[a] * (1 + sy[a] * xi[1]) * (1 + sz[a] * xi[2]);
        g[1] = 0.125 * sy[a] * (1 + sx[a] * xi[0]) * (1 + sz[a] * xi[2]);
        g[2] = 0.125 * sz[a] * (1 + sx[a] * xi[0]) * (1 + sy[a] * xi[1]);
    }
}

double shape_value(int dim, const double* xi, int a) {
    if (dim == 2) {
        static const double sx[4] = {-1, 1, 1, -1};
        static const double sy[4] = {-1, -1, 1, 1};
        return 0.25 * (1 + sx[a] * xi[0]) * (1 + sy[a] * xi[1]);
    }
    static const double sx[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
    static const double sy[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
    static const double sz[8] = {-1, -1, -1, -1, 1, 1, 1, 1};
    return 0.125 * (1 + sx[a] * xi[0]) * (1 + sy[a] * xi[1]) * (1 + sz[a] * xi[2]);
}

// jacobian_det (mesh.hpp:91-105) == shape_and_gradients' detJ (fem.hpp:51-79)
double jacobian_det(int dim, const int32_t* en, const double* nodes, const double* xi) {
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double g[3];
    const int nn = dim == 2 ? 4 : 8;
    for (int a = 0; a < nn; ++a) {
        corner_gradient(dim, xi, a, g);
        const double* p = nodes + 3 * std::size_t(en[a]);
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) J[i][j] += p[i] * g[j];
    }
    if (dim == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

// compute_element_geometry (mesh.hpp:112-139)
void element_geometry(int dim, int n_elems, const int32_t* conn, const double* nodes,
                      double* centroid, double* volume) {
    const double gp = 1.0 / std::sqrt(3.0);
    const int nn = dim == 2 ? 4 : 8;
    for (int e = 0; e < n_elems; ++e) {
        const int32_t* en = conn + std::size_t(e) * nn;
        double c[3] = {0, 0, 0};
        for (int a = 0; a < nn; ++a)
            for (int k = 0; k < 3; ++k) c[k] += nodes[3 * std::size_t(en[a]) + k];
        for (int k = 0; k < 3; ++k) c[k] /= nn;
        for (int k = 0; k < 3; ++k) centroid[3 * std::size_t(e) + k] = c[k];
        double vol = 0.0;
        const int ng = dim == 2 ? 4 : 8;
        for (int q = 0; q < ng; ++q) {
            const double xi[3] = {(q & 1) ? gp : -gp, (q & 2) ? gp : -gp, (q & 4) ? gp : -gp};
            const double dj = jacobian_det(dim, en, nodes, xi);
            if (dj <= 0.0)
                throw ConfigError("inverted element " + std::to_string(e) +
                                  " (non-positive Jacobian)");
            vol += dj;
        }
        volume[e] = vol;
    }
}

// Mesh::char_length (mesh.hpp:51-57)
double char_length(int dim, int n_elems, const double* volume) {
    if (n_elems <= 0) return 0.0;
    double v = 0.0;
    for (int e = 0; e < n_elems; ++e) v += volume[e];
    v /= static_cast<double>(n_elems);
    return dim == 2 ? std::sqrt(v) : std::cbrt(v);
}

// Mesh::char_length (mesh.hpp:51-57) of the generated lattice n[0] x n[1] (x n[2])
// at spacing h from lo, without storing it: the volume sum on the device when
// one is present, else the same sum streamed on the host
double lattice_char_length(int dim, const int n[3], const double lo[3], double h, bool host) {
    const long long E = (long long)n[0] * n[1] * (dim == 3 ? n[2] : 1);
    if (E <= 0) return 0.0;
    double v = 0.0;
    if (!host && device_available()) {
        v = lattice_volume_sum_device(dim, n, lo, h);
    } else {
        const double gp = 1.0 / std::sqrt(3.0);
        const int nx = n[0] + 1, ny = n[1] + 1;
        std::vector<double> nodes(3 * 8);
        int32_t en[8];
        for (long long e = 0; e < E; ++e) {
            const int i = int(e % n[0]), j = int((e / n[0]) % n[1]), k = int(e / ((long long)n[0] * n[1]));
            const int ii[8] = {i, i + 1, i + 1, i, i, i + 1, i + 1, i};
            const int jj[8] = {j, j, j + 1, j + 1, j, j, j + 1, j + 1};
            for (int a = 0; a < (dim == 2 ? 4 : 8); ++a) {
                const int kk = a >= 4 ? k + 1 : k;
                nodes[3 * a] = lo[0] + ii[a] * h;
                nodes[3 * a + 1] = lo[1] + jj[a] * h;
                nodes[3 * a + 2] = dim == 3 ? lo[2] + kk * h : 0.0;
                en[a] = a;
            }
            (void)nx;
            (void)ny;
            double vol = 0.0;
            for (int q = 0; q < (dim == 2 ? 4 : 8); ++q) {
                const double xi[3] = {(q & 1) ? gp : -gp, (q & 2) ? gp : -gp, (q & 4) ? gp : -gp};
                vol += jacobian_det(dim, en, nodes.data(), xi);
            }
            v += vol;
        }
    }
    v /= static_cast<double>(E);
    return dim == 2 ? std::sqrt(v) : std::cbrt(v);
}

// GK15 adaptive quadrature (material.hpp:92-142) and calibrate_c0 (:150-165)
namespace {
const double kXk[15] = {-0.991455371120813, -0.949107912342759, -0.864864423359769,
                        -0.741531185599394, -0.586087235467691, -0.405845151377397,
                        -0.207784955007898, 0.0, 0.207784955007898, 0.405845151377397,
                        0.586087235467691, 0.741531185599394, 0.864864423359769,
                        0.949107912342759, 0.991455371120813};
const double kWk[15] = {0.022935322010529, 0.063092092629979, 0.104790010322250,
                        0.140653259715525, 0.169004726639267, 0.190350578064785,
                        0.204432940075298, 0.209482141084728, 0.204432940075298,
                        0.190350578064785, 0.169004726639267, 0.140653259715525,
                        0.104790010322250, 0.063092092629979, 0.022935322010529};
const double kWg[7] = {0.129484966168870, 0.279705391489277, 0.381830050505119,
                       0.417959183673469, 0.381830050505119, 0.279705391489277,
                       0.129484966168870};

struct C0Integrand {
    double delta, l;
    int power;
    double operator()(double s) const {
        const double r = s * delta;
        return std::pow(r, power) * std::exp(-r / l);
    }
};

void gk15(const C0Integrand& f, double a, double b, double& value, double& error) {
    const double h = 0.5 * (b - a), c = 0.5 * (a + b);
    double sk = 0.0, sg = 0.0;
    for (int i = 0; i < 15; ++i) {
        const double fv = f(c + h * kXk[i]);
        sk += kWk[i] * fv;
        if (i % 2 == 1) sg += kWg[i / 2] * fv;
    }
    value = sk * h;
    error = std::abs((sk - sg) * h);
}

double adaptive(const C0Integrand& f, double a, double b, double rel_tol, int depth) {
    double v, e;
    gk15(f, a, b, v, e);
    if (e <= rel_tol * std::max(std::abs(v), 1e-300) || depth > 48) return v;
    const double m = 0.5 * (a + b);
    return adaptive(f, a, m, rel_tol, depth + 1) + adaptive(f, m, b, rel_tol, depth + 1);
}
}  // namespace

double calibrate_c0(double E, double delta, double l, int formulation) {
    if (E <= 0.0) throw ConfigError("elastic modulus must be positive");
    if (l <= 0.0 || l > delta) throw ConfigError("length scale must satisfy 0 < l <= delta");
    const int power = formulation == 2 ? 6 : 5;
    const double integral = adaptive(C0Integrand{delta, l, power}, 0.0, 1.0, 1e-12, 0) * delta;
    constexpr double pi = 3.14159265358979323846;
    return 3.0 * E / (pi * integral);
}

}  // namespace pmts

using namespace pmts;

struct Box {
    double lo[3], hi[3];
    // BoundsBox::contains (mesh.hpp:145-149)
    bool contains(const double* p, int dim, double tol = 0.0) const {
        for (int k = 0; k < dim; ++k)
            if (p[k] < lo[k] - tol || p[k] > hi[k] + tol) return false;
        return true;
    }
};

struct pmts_scenario {
    int dim = 2;
    int n[3] = {1, 1, 1};
    std::vector<double> nodes, centroid, volume, mass, p_ext, bc_vel;
    std::vector<int32_t> conn, bc_dofs;
    double delta = 0, l = 0, c0 = 0, cl = 0, dt = 0, gamma = 0.5, beta = 0, s_crit = 0, ramp = 0;
    int n_steps = 0;
};

namespace {

// generate_structured (mesh.hpp:170-219)
void generate(pmts_scenario& s, const pmts_scenario_desc& d) {
    if (d.spacing <= 0.0) throw ConfigError("mesh spacing must be positive");
    if (d.dim != 2 && d.dim != 3) throw ConfigError("mesh dimension must be 2 or 3");
    s.dim = d.dim;
    for (int k = 0; k < d.dim; ++k) {
        const double len = d.hi[k] - d.lo[k];
        if (len <= 0.0) throw ConfigError("degenerate extent along an axis");
        const double cells = len / d.spacing;
        const double rounded = std::round(cells);
        if (std::abs(cells - rounded) > 1e-9 * std::max(1.0, cells) || rounded < 1.0)
            throw ConfigError("extent along an axis is not a multiple of the spacing");
        s.n[k] = static_cast<int>(rounded);
    }
    const int nx = s.n[0] + 1, ny = s.n[1] + 1, nz = d.dim == 3 ? s.n[2] + 1 : 1;
    s.nodes.reserve(std::size_t(nx) * ny * nz * 3);
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                s.nodes.push_back(d.lo[0] + i * d.spacing);
                s.nodes.push_back(d.lo[1] + j * d.spacing);
                s.nodes.push_back(d.dim == 3 ? d.lo[2] + k * d.spacing : 0.0);
            }
    auto nid = [&](int i, int j, int k) { return (k * ny + j) * nx + i; };
    for (int k = 0; k < (d.dim == 3 ? s.n[2] : 1); ++k)
        for (int j = 0; j < s.n[1]; ++j)
            for (int i = 0; i < s.n[0]; ++i) {
                if (d.dim == 2) {
                    const int32_t e[4] = {nid(i, j, 0), nid(i + 1, j, 0), nid(i + 1, j + 1, 0),
                                          nid(i, j + 1, 0)};
                    s.conn.insert(s.conn.end(), e, e + 4);
                } else {
                    const int32_t e[8] = {nid(i, j, k),         nid(i + 1, j, k),
                                          nid(i + 1, j + 1, k), nid(i, j + 1, k),
                                          nid(i, j, k + 1),     nid(i + 1, j, k + 1),
                                          nid(i + 1, j + 1, k + 1), nid(i, j + 1, k + 1)};
                    s.conn.insert(s.conn.end(), e, e + 8);
                }
            }
    const int nn = d.dim == 2 ? 4 : 8;
    const int E = int(s.conn.size() / nn);
    s.centroid.resize(3 * std::size_t(E));
    s.volume.resize(E);
    element_geometry(d.dim, E, s.conn.data(), s.nodes.data(), s.centroid.data(),
                     s.volume.data());
}

void build(pmts_scenario& s, const pmts_scenario_desc& d) {
    // geometry and lumped masses on the device when one is present (pd_setup.cu,
    // bitwise the host restatement's values); the host loops otherwise
    DeviceSetup* dev = nullptr;
    struct DevGuard {
        DeviceSetup*& p;
        ~DevGuard() {
            if (p) setup_device_end(p);
        }
    } dev_guard{dev};
    if (!d.host_setup && device_available()) {
        if (d.spacing <= 0.0) throw ConfigError("mesh spacing must be positive");
        if (d.dim != 2 && d.dim != 3) throw ConfigError("mesh dimension must be 2 or 3");
        s.dim = d.dim;
        for (int k = 0; k < d.dim; ++k) {
            const double len = d.hi[k] - d.lo[k];
            if (len <= 0.0) throw ConfigError("degenerate extent along an axis");
            const double cells = len / d.spacing;
            const double rounded = std::round(cells);
            if (std::abs(cells - rounded) > 1e-9 * std::max(1.0, cells) || rounded < 1.0)
                throw ConfigError("extent along an axis is not a multiple of the spacing");
            s.n[k] = static_cast<int>(rounded);
        }
        dev = setup_device_begin(d.dim, s.n, d.lo, d.spacing, d.rho, s.nodes, s.conn, s.centroid,
                                 s.volume);
    } else {
        generate(s, d);
    }
    const int dim = s.dim, nn = dim == 2 ? 4 : 8;
    const int N = int(s.nodes.size() / 3), E = int(s.volume.size());
    s.cl = char_length(dim, E, s.volume.data());
    // build_scenario (driver.hpp:179-191)
    s.delta = d.delta_factor * s.cl;
    s.l = s.delta / d.l_factor;
    s.c0 = calibrate_c0(d.E, s.delta, s.l, d.formulation);
    s.s_crit = d.s_crit;
    if (s.delta <= 0.0) throw ConfigError("horizon must be positive");
    if (d.rho <= 0.0) throw ConfigError("density must be positive");
    s.ramp = d.load_ramp >= 0.0 ? d.load_ramp : d.m * d.dt_pd;
    s.dt = d.dt_pd;
    s.gamma = d.gamma;
    s.beta = d.beta;
    if (d.dt_pd <= 0.0) throw ConfigError("time.dt_pd must be positive");
    s.n_steps = static_cast<int>(std::llround(d.total_time / d.dt_pd));

    // bounding box (mesh.hpp:59-67)
    double blo[3] = {1e300, 1e300, 1e300}, bhi[3] = {-1e300, -1e300, -1e300};
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < 3; ++k) {
            blo[k] = std::min(blo[k], s.nodes[3 * std::size_t(n) + k]);
            bhi[k] = std::max(bhi[k], s.nodes[3 * std::size_t(n) + k]);
        }
    // body patches, then tractions as horizon bands (driver.hpp:76-116)
    std::vector<Box> patch_box;
    std::vector<std::array<double, 3>> patch_val;
    for (int p = 0; p < d.n_body_patch; ++p) {
        const double* v = d.body_patch + 9 * p;
        patch_box.push_back(Box{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}});
        patch_val.push_back({v[6], v[7], v[8]});
    }
    const double tol = 1e-9 * std::max(s.cl, 1e-300);
    for (int p = 0; p < d.n_traction; ++p) {
        const double* v = d.traction + 9 * p;
        Box box{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}};
        int axis = -1;
        bool high = false;
        for (int k = 0; k < dim; ++k) {
            if (std::abs(box.lo[k] - box.hi[k]) < 2.0 * s.cl) {
                if (std::abs(box.lo[k] - blo[k]) < s.cl || std::abs(box.hi[k] - blo[k]) < s.cl) {
                    axis = k;
                    high = false;
                }
                if (std::abs(box.lo[k] - bhi[k]) < s.cl || std::abs(box.hi[k] - bhi[k]) < s.cl) {
                    axis = k;
                    high = true;
                }
            }
        }
        if (axis < 0)
            throw ConfigError("cannot map a traction patch to a boundary plane for the PD "
                              "body-force band");
        Box band = box;
        if (high) {
            band.hi[axis] = bhi[axis] + tol;
            band.lo[axis] = bhi[axis] - s.delta + tol;
        } else {
            band.lo[axis] = blo[axis] - tol;
            band.hi[axis] = blo[axis] + s.delta - tol;
        }
        std::array<double, 3> val{0, 0, 0};
        for (int k = 0; k < dim; ++k) val[k] = v[6 + k] / s.delta;
        patch_box.push_back(band);
        patch_val.push_back(val);
    }
    // M and P_ext (perifem.hpp:331-348) with w = 1 - alpha = 1
    const std::size_t nd = std::size_t(N) * dim;
    if (dev) {
        std::vector<double> boxes;
        for (std::size_t p = 0; p < patch_box.size(); ++p) {
            for (int k = 0; k < 3; ++k) boxes.push_back(patch_box[p].lo[k]);
            for (int k = 0; k < 3; ++k) boxes.push_back(patch_box[p].hi[k]);
            for (int k = 0; k < 3; ++k) boxes.push_back(patch_val[p][k]);
        }
        setup_device_loads(dev, d.body_force, int(patch_box.size()), boxes.data(), s.mass, s.p_ext);
    } else {
        s.mass.assign(nd, 0.0);
        s.p_ext.assign(nd, 0.0);
    }
    const double g = 1.0 / std::sqrt(3.0);
    for (int e = 0; e < E && !dev; ++e) {
        const int32_t* en = s.conn.data() + std::size_t(e) * nn;
        const double w = 1.0 - 0.0;
        // lumped_mass (fem.hpp:172-179) over gauss_points (fem.hpp:101-115)
        double masses[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int ng = dim == 2 ? 4 : 8;
        for (int q = 0; q < ng; ++q) {
            const int i = q & 1, j = (q >> 1) & 1, k = (q >> 2) & 1;
            const double xi[3] = {i ? g : -g, j ? g : -g, dim == 3 ? (k ? g : -g) : 0.0};
            const double detJ = jacobian_det(dim, en, s.nodes.data(), xi);
            if (detJ <= 0.0) throw ConfigError("inverted element (non-positive Jacobian)");
            for (int a = 0; a < nn; ++a) masses[a] += d.rho * shape_value(dim, xi, a) * detJ;
        }
        double b[3] = {d.body_force[0], d.body_force[1], d.body_force[2]};
        const double* c = s.centroid.data() + 3 * std::size_t(e);
        for (std::size_t p = 0; p < patch_box.size(); ++p)
            if (patch_box[p].contains(c, dim))
                for (int k = 0; k < dim; ++k) b[k] += patch_val[p][k];
        for (int a = 0; a < nn; ++a) {
            const std::size_t base = std::size_t(en[a]) * dim;
            for (int k = 0; k < dim; ++k) {
                s.mass[base + k] += w * masses[a];
                s.p_ext[base + k] += w * b[k] * masses[a] / d.rho;
            }
        }
    }
    // kinematic constraints (driver.hpp:121-149)
    std::map<int, double> table;
    struct Kin {
        Box box;
        int comp;
        double vel;
        bool fix_all;
    };
    std::vector<Kin> kin;
    for (int b = 0; b < d.n_velocity_bc; ++b) {
        const double* v = d.velocity_bc + 8 * b;
        const int comp = int(v[6]);
        if (comp < 0 || comp >= dim) throw ConfigError("velocity_bc component out of range");
        kin.push_back({Box{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}}, comp, v[7], false});
    }
    for (int b = 0; b < d.n_fixed; ++b) {
        const double* v = d.fixed + 6 * b;
        kin.push_back({Box{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}}, 0, 0.0, true});
    }
    for (const auto& k : kin) {
        bool hit = false;
        for (int n = 0; n < N && !hit; ++n) hit = k.box.contains(&s.nodes[3 * std::size_t(n)], dim, tol);
        if (!hit) throw ConfigError("kinematic constraint selects no node");
        for (int n = 0; n < N; ++n) {
            if (!k.box.contains(&s.nodes[3 * std::size_t(n)], dim, tol)) continue;
            if (k.fix_all)
                for (int c = 0; c < dim; ++c) table[n * dim + c] = 0.0;
            else
                table[n * dim + k.comp] = k.vel;
        }
    }
    for (const auto& [dof, v] : table) {
        s.bc_dofs.push_back(dof);
        s.bc_vel.push_back(v);
    }
    for (std::size_t i = 0; i < nd; ++i)
        if (s.mass[i] <= 0.0 && !table.count(int(i)))
            throw SolverError("non-positive lumped mass at dof " + std::to_string(i));
}

}  // namespace

extern "C" {

const char* pmts_last_error(void) { return g_last_error.c_str(); }
int pmts_abi_version(void) { return PMTS_ABI_VERSION; }

int pmts_scenario_build(const pmts_scenario_desc* desc, pmts_scenario** out) {
    return guard([&] {
        if (!desc || !out) throw ConfigError("null argument");
        auto s = std::make_unique<pmts_scenario>();
        build(*s, *desc);
        *out = s.release();
    });
}

int pmts_scenario_get(const pmts_scenario* s, pmts_scenario_view* v) {
    return guard([&] {
        if (!s || !v) throw ConfigError("null argument");
        v->dim = s->dim;
        v->n_nodes = int32_t(s->nodes.size() / 3);
        v->n_elems = int32_t(s->volume.size());
        v->n_dof = v->n_nodes * s->dim;
        v->n_bc = int32_t(s->bc_dofs.size());
        v->n_steps = s->n_steps;
        for (int k = 0; k < 3; ++k) v->lattice[k] = k < s->dim ? s->n[k] : 1;
        v->delta = s->delta;
        v->l = s->l;
        v->c0 = s->c0;
        v->char_length = s->cl;
        v->dt = s->dt;
        v->gamma = s->gamma;
        v->beta = s->beta;
        v->s_crit = s->s_crit;
        v->load_ramp = s->ramp;
        v->node_xyz = s->nodes.data();
        v->elem_nodes = s->conn.data();
        v->centroid = s->centroid.data();
        v->volume = s->volume.data();
        v->mass = s->mass.data();
        v->p_ext = s->p_ext.data();
        v->bc_dofs = s->bc_dofs.data();
        v->bc_vel = s->bc_vel.data();
    });
}

double pmts_scenario_load_scale(const pmts_scenario* s, double t) {
    if (s->ramp <= 0.0) return 1.0;
    return std::clamp(t / s->ramp, 0.0, 1.0);
}

void pmts_scenario_destroy(pmts_scenario* s) { delete s; }

}  // extern "C"
