// ORACLE / TEST INFRASTRUCTURE ONLY -- not product code.
//
// Thin driver over the UNMODIFIED reference headers (compiled in place from
// /root/reference/proj/include by oracle/Makefile; no reference source is
// copied into this repository).  It runs the reference's own pure-PD step
// loop -- the hot path of SURVEY.md section 8(a) -- and either dumps every
// input/output needed to pin the CPU restatement and the CUDA path
// (--dump DIR), or times the loop (--time) for the bench's reference arm.
//
// The loop below restates run_built's pure-PD branch call for call
// (reference: proj/include/perimts/driver_run.hpp:160-246):
//   find_pe_pairs            mesh.hpp:416-495
//   build_peri_elements      perifem.hpp:42-100
//   assemble_pd_global       perifem.hpp:276-351
//   BlockOperator            newmark.hpp:77-181
//   advance_dynamic_step     newmark.hpp:185-190
//   update_bond_states       perifem.hpp:170-193
//   incremental_stiffness_update perifem.hpp:356-364
//   damage_field             perifem.hpp:202-231
//
// Usage:
//   ref_driver CFG_FILE [--override sec.key=val]... [--steps N]
//              [--dump DIR] [--checkpoints k1,k2,...] [--time] [--setup-only]
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

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_driver CFG [--override k=v]... [--steps N] [--dump DIR] "
                             "[--checkpoints a,b] [--time] [--setup-only]\n");
        return 2;
    }
    std::string cfg_path = argv[1], dump_dir;
    std::vector<std::string> overrides;
    std::vector<int> checkpoints;
    int steps_override = -1, warmup = 0;
    bool time_only = false, setup_only = false;
    for (int a = 2; a < argc; ++a) {
        std::string s = argv[a];
        if (s == "--override" && a + 1 < argc) overrides.push_back(argv[++a]);
        else if (s == "--steps" && a + 1 < argc) steps_override = std::atoi(argv[++a]);
        else if (s == "--dump" && a + 1 < argc) dump_dir = argv[++a];
        else if (s == "--checkpoints" && a + 1 < argc) checkpoints = parse_list(argv[++a]);
        else if (s == "--time") time_only = true;
        else if (s == "--setup-only") setup_only = true;
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
        if (sc.mode != RunMode::pure_pd) throw ConfigError("ref_driver runs run.mode = pure_pd");

        const double t_setup0 = now_s();
        BuiltScenario b = build_scenario(sc);
        const Mesh& mesh = b.mesh;
        std::vector<int> active(mesh.element_count());
        for (int e = 0; e < mesh.element_count(); ++e) active[e] = e;
        const std::vector<double> alpha_field(mesh.element_count(), 0.0);

        const double t_pairs0 = now_s();
        const auto pairs = find_pe_pairs(mesh, b.pd_mat.delta, b.sc.notches);
        const double t_pairs = now_s() - t_pairs0;
        auto pes = build_peri_elements(mesh, pairs, b.sc.pe_quadrature);
        PdSystem sys = assemble_pd_global(mesh, active, alpha_field,
                                          [](const Point&) { return 0.0; }, pes, b.pd_mat,
                                          b.sc.material, b.loads);
        NewmarkParams nm = b.sc.pd_nm;
        nm.dt = b.sc.dt_pd;
        BcTable bcs = detail::resolve_bcs_quiet(mesh, sys.dofs, b.loads);
        BlockOperator op(&sys.K, sys.M, nm, bcs);
        KinematicState state = KinematicState::zero(sys.dofs.n_dof);
        for (std::size_t c = 0; c < bcs.dofs.size(); ++c) state.vel[bcs.dofs[c]] = bcs.velocity[c];
        {
            Vector p0 = sys.P_ext;
            scale(p0, b.load_scale(0.0));
            state.acc = op.initial_acceleration(p0, state.disp);
        }
        const double t_setup = now_s() - t_setup0;

        int n_steps = static_cast<int>(std::llround(b.sc.total_time / b.sc.dt_pd));
        if (steps_override >= 0) n_steps = steps_override;

        if (!dump_dir.empty()) {
            std::vector<double> nodes, cen, vol;
            std::vector<int> conn, pr;
            const int nn = mesh.dim == 2 ? 4 : 8;
            for (const auto& p : mesh.nodes) nodes.insert(nodes.end(), p.begin(), p.end());
            for (const auto& e : mesh.elements) {
                for (int a = 0; a < nn; ++a) conn.push_back(e.node_ids[a]);
                cen.insert(cen.end(), e.centroid.begin(), e.centroid.end());
                vol.push_back(e.volume);
            }
            for (const auto& p : pairs) {
                pr.push_back(p.i);
                pr.push_back(p.j);
            }
            std::vector<double> xi_norm, weight;
            for (const auto& pe : pes) {
                xi_norm.push_back(pe.quad_pairs[0].xi_norm);
                weight.push_back(pe.quad_pairs[0].weight);
            }
            dump_vec(dump_dir + "/nodes.f64", nodes);
            dump_vec(dump_dir + "/conn.i32", conn);
            dump_vec(dump_dir + "/centroid.f64", cen);
            dump_vec(dump_dir + "/volume.f64", vol);
            dump_vec(dump_dir + "/pairs.i32", pr);
            dump_vec(dump_dir + "/xi_norm.f64", xi_norm);
            dump_vec(dump_dir + "/weight.f64", weight);
            dump_vec(dump_dir + "/mass.f64", sys.M);
            dump_vec(dump_dir + "/p_ext.f64", sys.P_ext);
            dump_vec(dump_dir + "/bc_dofs.i32", bcs.dofs);
            dump_vec(dump_dir + "/bc_vel.f64", bcs.velocity);
            dump_vec(dump_dir + "/a0.f64", state.acc);
            std::vector<double> scales;
            for (int i = 0; i <= n_steps; ++i) scales.push_back(b.load_scale(i * b.sc.dt_pd));
            dump_vec(dump_dir + "/scale.f64", scales);
            std::ofstream meta(dump_dir + "/meta.txt");
            meta.precision(17);
            meta << "dim " << mesh.dim << "\n"
                 << "n_nodes " << mesh.node_count() << "\n"
                 << "n_elems " << mesh.element_count() << "\n"
                 << "n_pairs " << pairs.size() << "\n"
                 << "n_dof " << sys.dofs.n_dof << "\n"
                 << "n_steps " << n_steps << "\n"
                 << "delta " << b.pd_mat.delta << "\n"
                 << "l " << b.pd_mat.l << "\n"
                 << "c0 " << b.pd_mat.c0 << "\n"
                 << "s_crit " << b.pd_mat.s_crit << "\n"
                 << "dt " << nm.dt << "\n"
                 << "gamma " << nm.gamma << "\n"
                 << "beta " << nm.beta << "\n"
                 << "rho " << b.sc.material.rho << "\n"
                 << "char_length " << mesh.char_length() << "\n"
                 << "nnz " << sys.K.nnz() << "\n";
        }
        if (setup_only) {
            std::printf("{\"setup_s\": %.6f, \"pairs_s\": %.6f, \"bonds\": %zu, \"nnz\": %d}\n",
                        t_setup, t_pairs, pairs.size(), sys.K.nnz());
            return 0;
        }

        std::vector<int> broken_log;  // (step, pe) rows
        std::size_t broken_total = 0;
        double t_k = 0.0, t_u = 0.0;
        Vector warm;
        double t_loop0 = now_s();
        for (int i = 1; i <= n_steps; ++i) {
            if (i == warmup + 1) t_loop0 = now_s();  // steps 1..warmup untimed
            const double t = i * b.sc.dt_pd;
            const double tick = now_s();
            Vector p_t = sys.P_ext;
            scale(p_t, b.load_scale(t));
            state = advance_dynamic_step(op, state, p_t, &warm);
            const double tick_u = now_s();
            t_k += tick_u - tick;
            if (b.pd_mat.fracture_enabled()) {
                const auto broken =
                    update_bond_states(mesh, pes, state.disp, sys.dofs, b.pd_mat.s_crit);
                if (!broken.empty()) {
                    incremental_stiffness_update(sys.K, mesh, sys.dofs, pes, sys.pe_weight,
                                                 broken, b.pd_mat);
                    if (!nm.explicit_scheme()) op.refresh_diagonal();
                }
                broken_total += broken.size();
                if (!time_only)
                    for (const auto& bb : broken) {
                        broken_log.push_back(i);
                        broken_log.push_back(bb.pe);
                    }
            }
            t_u += now_s() - tick_u;
            if (!dump_dir.empty())
                for (int k : checkpoints)
                    if (k == i) {
                        dump_vec(dump_dir + "/u_" + std::to_string(i) + ".f64", state.disp);
                        dump_vec(dump_dir + "/v_" + std::to_string(i) + ".f64", state.vel);
                        dump_vec(dump_dir + "/a_" + std::to_string(i) + ".f64", state.acc);
                    }
        }
        const double t_loop = now_s() - t_loop0;

        if (!dump_dir.empty()) {
            dump_vec(dump_dir + "/u.f64", state.disp);
            dump_vec(dump_dir + "/v.f64", state.vel);
            dump_vec(dump_dir + "/a.f64", state.acc);
            dump_vec(dump_dir + "/broken.i32", broken_log);
            const DamageField dmg = damage_field(mesh, pes);
            dump_vec(dump_dir + "/damage_elem.f64", dmg.element);
            dump_vec(dump_dir + "/damage_node.f64", dmg.node);
        }
        const double bonds = double(pairs.size());
        const int timed = n_steps - std::min(warmup, n_steps);
        std::printf("{\"steps\": %d, \"warmup\": %d, \"bonds\": %zu, \"nnz\": %d, "
                    "\"setup_s\": %.6f, \"loop_s\": %.6f, \"t_k_s\": %.6f, \"t_u_s\": %.6f, "
                    "\"bond_updates_per_s\": %.6e, \"workers\": %d, \"broken\": %zu}\n",
                    n_steps, warmup, pairs.size(), sys.K.nnz(), t_setup, t_loop, t_k, t_u,
                    timed > 0 ? bonds * timed / t_loop : 0.0, worker_count(), broken_total);
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
