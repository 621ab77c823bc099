// Internal helpers shared by the host translation units of libpmts.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pmts_capi.h"

namespace pmts {

// Exception types mirror the reference's (errors.hpp:8-21); they never cross
// the C ABI -- guard() maps them onto status codes.
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InternalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

// f(i) for i in [0, n) over the host's cores (independent iterations); the first
// exception is rethrown
template <class F>
void par_range(int n, F&& f) {
    const int nth = int(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
    if (n < 4096 || nth == 1) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(nth);
    for (int t = 0; t < nth; ++t)
        th.emplace_back([&, t] {
            try {
                for (int i = int((long long)n * t / nth); i < int((long long)n * (t + 1) / nth); ++i)
                    f(i);
            } catch (...) {
                err[t] = std::current_exception();
            }
        });
    for (auto& x : th) x.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}


template <class F>
int guard(F&& f) {
    try {
        f();
        set_last_error("");
        return PMTS_OK;
    } catch (const ConfigError& e) {
        set_last_error(e.what());
        return PMTS_ERR_CONFIG;
    } catch (const SolverError& e) {
        set_last_error(e.what());
        return PMTS_ERR_SOLVER;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PMTS_ERR_INTERNAL;
    } catch (...) {
        set_last_error("unknown error");
        return PMTS_ERR_INTERNAL;
    }
}

// Bit-exact host restatements used by both the setup and the PD handle.
void element_geometry(int dim, int n_elems, const int32_t* conn, const double* nodes,
                      double* centroid, double* volume);
double char_length(int dim, int n_elems, const double* volume);
double lattice_char_length(int dim, const int n[3], const double lo[3], double h, bool host);
double calibrate_c0(double E, double delta, double l, int formulation);
// reference_shape gradients / values (fem.hpp:22-47) and the Jacobian
// determinant of shape_and_gradients (fem.hpp:51-79); nodes are xyz triples
void corner_gradient(int dim, const double* xi, int a, double* g);
double shape_value(int dim, const double* xi, int a);
double jacobian_det(int dim, const int32_t* en, const double* nodes, const double* xi);

// Device restatement of the generated-mesh setup (pd_setup.cu), bitwise equal to
// the host one; used when a CUDA device is present (PMTS_HOST_SETUP=1: host).
#include <vector>
struct DeviceSetup;
bool device_available();
DeviceSetup* setup_device_begin(int dim, const int n[3], const double lo[3], double spacing,
                                double rho, std::vector<double>& nodes,
                                std::vector<int32_t>& conn, std::vector<double>& centroid,
                                std::vector<double>& volume);
// boxes: n_patch x (lo[3] hi[3] value[3]) in the host loop's patch order
void setup_device_loads(DeviceSetup* ds, const double body[3], int n_patch, const double* boxes,
                        std::vector<double>& mass, std::vector<double>& p_ext);
void setup_device_end(DeviceSetup* ds);
// sum of the element volumes of a generated lattice in element order (the first
// half of Mesh::char_length, mesh.hpp:51-57), computed on the device
double lattice_volume_sum_device(int dim, const int n[3], const double lo[3], double spacing);

}  // namespace pmts
