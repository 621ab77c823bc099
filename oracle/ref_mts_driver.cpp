// ORACLE / TEST INFRASTRUCTURE ONLY -- not product code.
//
// Thin driver over the UNMODIFIED reference headers (compiled in place from
// /root/reference/proj/include by oracle/Makefile; no reference source is
// copied into this repository) for the coupled multi-time-step path
// (SURVEY.md 8(f) row 1).  It runs the reference's own coupled macro loop and
// either dumps the assembled systems and the per-macro-step states (--dump
// DIR) to pin the device integrator, or times the macro steps (--time) for
// the bench's reference arm.
//
// The setup and loop restate run_built's coupled branch call for call
// (reference: proj/include/perimts/driver_run.hpp:247-295):
//   assemble_global (alpha-weighted FE)   fem.hpp:421-474
//   find_pe_pairs(..., pd_active)          mesh.hpp:416-495
//   build_peri_elements                    perifem.hpp:42-100
//   assemble_pd_global ((1-alpha) weights) perifem.hpp:276-351
//   resolve_bcs_quiet                      driver.hpp:133-150
//   build_coupling_map                     coupling.hpp:72-105
//   CoupledIntegrator + macro_step         mts.hpp:81-118, 244-306
//
// Usage:
//   ref_mts_driver CFG [--override sec.key=val]... [--steps N] [--dump DIR]
//                  [--checkpoints k1,k2,...] [--time] [--warmup N]
#include "perimts/driver.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

using namespace perimts;

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

template <class T>
void dump_vec(const std::string& path, const std::vector<T>& v) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot write " + path);
    f.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
}

std::vector<int> parse_list(const std::string& s) {
    std::vector<int> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ','))
        if (!tok.empty()) out.push_back(std::stoi(tok));
    return out;
}

void dump_state(const std::string& dir, const std::string& tag, const KinematicState& s) {
    dump_vec(dir + "/" + tag + "_u.f64", s.disp);
    dump_vec(dir + "/" + tag + "_v.f64", s.vel);
    dump_vec(dir + "/" + tag + "_a.f64", s.acc);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_mts_driver CFG [--override k=v]... [--steps N] "
                             "[--dump DIR] [--checkpoints a,b] [--time] [--warmup N]\n");
        return 2;
    }
    std::string cfg_path = argv[1], dump_dir;
    std::vector<std::string> overrides;
    std::vector<int> checkpoints;
    int steps_override = -1, warmup = 0;
    bool time_only = false;
    for (int a = 2; a < argc; ++a) {
        std::string s = argv[a];
        if (s == "--override" && a + 1 < argc) overrides.push_back(argv[++a]);
        else if (s == "--steps" && a + 1 < argc) steps_override = std::atoi(argv[++a]);
        else if (s == "--dump" && a + 1 < argc) dump_dir = argv[++a];
        else if (s == "--checkpoints" && a + 1 < argc) checkpoints = parse_list(argv[++a]);
        else if (s == "--time") time_only = true;
        else if (s == "--warmup" && a + 1 < argc) warmup = std::atoi(argv[++a]);
        else {
            std::fprintf(stderr, "unknown argument %s\n", s.c_str());
            return 2;
        }
    }
    try {
        Config cfg = Config::parse_file(cfg_path);
        for (const auto& o : overrides) cfg.apply_override(o);
        const ScenarioConfig sc = load_scenario(cfg);
        if (sc.mode != RunMode::coupled_mts)
            throw ConfigError("ref_mts_driver runs run.mode = coupled_mts");

        const double t_setup0 = now_s();
        BuiltScenario b = build_scenario(sc);
        const Mesh& mesh = b.mesh;
        FeSystem fe_sys = assemble_global(mesh, b.fe_active, b.alpha_elem,
                                          &b.labels.element_label, b.sc.material, b.loads);
        const auto pairs = find_pe_pairs(mesh, b.pd_mat.delta, b.sc.notches, b.pd_active);
        std::vector<PeriElement> pes = build_peri_elements(mesh, pairs, b.sc.pe_quadrature);
        PdSystem pd_sys = assemble_pd_global(
            mesh, b.pd_active, b.alpha_elem, [&](const Point& p) { return b.weight(p); }, pes,
            b.pd_mat, b.sc.material, b.loads);
        BcTable fe_bcs = detail::resolve_bcs_quiet(mesh, fe_sys.dofs, b.loads);
        BcTable pd_bcs = detail::resolve_bcs_quiet(mesh, pd_sys.dofs, b.loads);
        const CouplingMap coupling =
            build_coupling_map(mesh, b.labels, fe_sys.dofs, pd_sys.dofs, &fe_bcs, &pd_bcs);
        // the PD stiffness as assembled, before any bond breaks (dumped below)
        const SparseMatrix k_pd0 = pd_sys.K;

        MtsOptions opts;
        opts.interface_mode = b.sc.interface_mode;
        opts.enforce_continuity = b.sc.enforce_continuity;
        opts.track_energy = b.sc.track_energy;
        MacroStepPlan plan{b.sc.m, b.sc.dt_pd};
        CoupledIntegrator integ(mesh, fe_sys, pd_sys, pes, coupling, b.pd_mat, plan, b.sc.fe_nm,
                                b.sc.pd_nm, fe_bcs, pd_bcs, b.load_scale, opts);
        integ.initialize_accelerations();
        const double t_setup = now_s() - t_setup0;

        int n_macro = static_cast<int>(std::llround(b.sc.total_time / b.sc.dt_fe()));
        if (steps_override >= 0) n_macro = steps_override;

        if (!dump_dir.empty()) {
            std::vector<int> labels(mesh.element_count()), pr, fe_nd, pd_nd;
            for (int e = 0; e < mesh.element_count(); ++e)
                labels[e] = static_cast<int>(b.labels.element_label[e]);
            for (const auto& p : pairs) {
                pr.push_back(p.i);
                pr.push_back(p.j);
            }
            dump_vec(dump_dir + "/labels.i32", labels);
            dump_vec(dump_dir + "/alpha.f64", b.alpha_elem);
            dump_vec(dump_dir + "/fe_node_dof.i32", fe_sys.dofs.node_dof);
            dump_vec(dump_dir + "/pd_node_dof.i32", pd_sys.dofs.node_dof);
            dump_vec(dump_dir + "/fe_k_rowptr.i32", fe_sys.K.row_ptr());
            dump_vec(dump_dir + "/fe_k_col.i32", fe_sys.K.col_idx());
            dump_vec(dump_dir + "/fe_k_val.f64", fe_sys.K.values());
            dump_vec(dump_dir + "/fe_mass.f64", fe_sys.M);
            dump_vec(dump_dir + "/fe_p_ext.f64", fe_sys.P_ext);
            dump_vec(dump_dir + "/pd_k_rowptr.i32", k_pd0.row_ptr());
            dump_vec(dump_dir + "/pd_k_col.i32", k_pd0.col_idx());
            dump_vec(dump_dir + "/pd_k_val.f64", k_pd0.values());
            dump_vec(dump_dir + "/pd_mass.f64", pd_sys.M);
            dump_vec(dump_dir + "/pd_p_ext.f64", pd_sys.P_ext);
            dump_vec(dump_dir + "/pairs.i32", pr);
            dump_vec(dump_dir + "/pe_weight.f64", pd_sys.pe_weight);
            dump_vec(dump_dir + "/fe_bc_dofs.i32", fe_bcs.dofs);
            dump_vec(dump_dir + "/fe_bc_vel.f64", fe_bcs.velocity);
            dump_vec(dump_dir + "/pd_bc_dofs.i32", pd_bcs.dofs);
            dump_vec(dump_dir + "/pd_bc_vel.f64", pd_bcs.velocity);
            dump_vec(dump_dir + "/fe_dof.i32", coupling.fe_dof);
            dump_vec(dump_dir + "/pd_dof.i32", coupling.pd_dof);
            dump_state(dump_dir, "fe0", integ.fe_state());
            dump_state(dump_dir, "pd0", integ.pd_state());
            std::vector<double> scales;
            for (int i = 0; i <= n_macro * b.sc.m; ++i) scales.push_back(b.load_scale(i * b.sc.dt_pd));
            dump_vec(dump_dir + "/scale.f64", scales);
            std::ofstream meta(dump_dir + "/meta.txt");
            meta.precision(17);
            meta << "dim " << mesh.dim << "\n"
                 << "n_nodes " << mesh.node_count() << "\n"
                 << "n_elems " << mesh.element_count() << "\n"
                 << "n_pairs " << pairs.size() << "\n"
                 << "fe_n_dof " << fe_sys.dofs.n_dof << "\n"
                 << "pd_n_dof " << pd_sys.dofs.n_dof << "\n"
                 << "n_lambda " << coupling.n_lambda << "\n"
                 << "n_macro " << n_macro << "\n"
                 << "m " << b.sc.m << "\n"
                 << "dt_pd " << b.sc.dt_pd << "\n"
                 << "delta " << b.pd_mat.delta << "\n"
                 << "c0 " << b.pd_mat.c0 << "\n"
                 << "l " << b.pd_mat.l << "\n"
                 << "s_crit " << b.pd_mat.s_crit << "\n"
                 << "dense " << (integ.dense_interface() ? 1 : 0) << "\n";
        }

        std::vector<int> broken_log;  // (macro step, pe) rows
        std::vector<double> lambdas, continuity, energy;
        std::vector<int> iters;
        long long broken_total = 0;
        double t_k = 0.0, t_u = 0.0, t_l = 0.0, t_y = 0.0;
        double t_loop0 = now_s();
        for (int i = 1; i <= n_macro; ++i) {
            if (i == warmup + 1) t_loop0 = now_s();
            // the broken bonds of this macro step, in the order macro_step records
            // them, come from the live mu flags: diff them around the step
            std::vector<std::uint8_t> before;
            if (!time_only)
                for (const auto& pe : pes) before.push_back(pe.quad_pairs[0].mu);
            const MacroReport rep = integ.macro_step();
            if (i > warmup) {
                t_k += rep.timing.t_kinematic;
                t_u += rep.timing.t_update;
                t_l += rep.timing.t_lambda;
                t_y += rep.timing.t_unit;
            }
            broken_total += rep.newly_broken;
            if (!time_only) {
                for (std::size_t p = 0; p < pes.size(); ++p)
                    if (before[p] && !pes[p].quad_pairs[0].mu) {
                        broken_log.push_back(i);
                        broken_log.push_back(static_cast<int>(p));
                    }
                continuity.push_back(rep.continuity_residual);
                energy.push_back(rep.energy.quad_fe);
                energy.push_back(rep.energy.quad_pd);
                energy.push_back(rep.energy.lambda_fe);
                energy.push_back(rep.energy.lambda_pd);
                iters.push_back(rep.interface_iterations);
            }
            if (!dump_dir.empty())
                for (int k : checkpoints)
                    if (k == i) {
                        dump_state(dump_dir, "fe_" + std::to_string(i), integ.fe_state());
                        dump_state(dump_dir, "pd_" + std::to_string(i), integ.pd_state());
                        dump_vec(dump_dir + "/lambda_" + std::to_string(i) + ".f64",
                                 integ.lambda());
                    }
        }
        const double t_loop = now_s() - t_loop0;
        if (!dump_dir.empty()) {
            dump_state(dump_dir, "fe", integ.fe_state());
            dump_state(dump_dir, "pd", integ.pd_state());
            dump_vec(dump_dir + "/lambda.f64", integ.lambda());
            dump_vec(dump_dir + "/broken.i32", broken_log);
            dump_vec(dump_dir + "/continuity.f64", continuity);
            dump_vec(dump_dir + "/energy.f64", energy);
            dump_vec(dump_dir + "/iterations.i32", iters);
        }
        const int timed = n_macro - std::min(warmup, n_macro);
        std::printf("{\"macro_steps\": %d, \"warmup\": %d, \"m\": %d, \"n_lambda\": %d, "
                    "\"dense\": %d, \"fe_dof\": %d, \"pd_dof\": %d, \"bonds\": %zu, "
                    "\"setup_s\": %.6f, \"loop_s\": %.6f, \"t_k_s\": %.6f, \"t_u_s\": %.6f, "
                    "\"t_lambda_s\": %.6f, \"t_unit_s\": %.6f, \"macro_steps_per_s\": %.6e, "
                    "\"workers\": %d, \"broken\": %lld}\n",
                    n_macro, warmup, b.sc.m, coupling.n_lambda, integ.dense_interface() ? 1 : 0,
                    fe_sys.dofs.n_dof, pd_sys.dofs.n_dof, pairs.size(), t_setup, t_loop, t_k,
                    t_u, t_l, t_y, timed > 0 ? timed / t_loop : 0.0, worker_count(),
                    broken_total);
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const SolverError& e) {
        std::fprintf(stderr, "solver error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
