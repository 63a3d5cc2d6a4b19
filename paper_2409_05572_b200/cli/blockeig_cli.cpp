// blockeig — command-line front end of the B200 library.
//
// Same subcommands, flags, CSV/JSON schemas and exit codes as the reference's
// tools/blockeig_cli.cpp (solve :245-292, compare :314-400 with the four
// strategies run concurrently on ONE matrix handle, gen :519-531, theory
// :505-517), talking to the library only through include/blockeig.h, so its
// history CSV is comparable column by column with the reference's.  Extensions
// (beig_solve_ex): --device, --op-shift (shifted operator, SI), --largest,
// --profile (per-kernel device timing in the summary).  No third-party parsers:
// flags are "--name value" / "--flag", JSON is written by hand.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <future>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blockeig.h"

namespace {

enum Exit { kOk = 0, kInput = 1, kNotConverged = 2, kViolation = 3 };

struct Opts {
    std::string matrix, gen, solver = "si", strategy = "none", expand = "xdrop", precond = "identity";
    std::string out, format = "csv";
    int n_ev = 1, n_ex = 0, n_es = 0, max_iters = 2000, cg_iters = 5;
    double tol = 1e-10, shift = 0.0;
    uint64_t seed = 0;
    int j_e = 12, j_s = 2, j_p = 10, j_warm = 5;
    double mu = 1.1, r_warm = 1e-4;
    bool spd_shift = false;
    // extensions
    int device = 0;
    bool profile = false, largest = false, op_shifted = false;
    double op_shift = 0.0;
    // theory
    std::string suite = "all";
    int trials = -1;
};

const std::map<std::string, int> kSolvers = {
    {"si", BEIG_SOLVER_SI}, {"sd", BEIG_SOLVER_SD}, {"lobpcg", BEIG_SOLVER_LOBPCG}, {"tracemin", BEIG_SOLVER_TRACEMIN}};
const std::map<std::string, int> kStrategies = {
    {"none", BEIG_STRATEGY_NONE}, {"fix", BEIG_STRATEGY_FIX}, {"slope", BEIG_STRATEGY_SLOPE},
    {"slopek", BEIG_STRATEGY_SLOPEK}};
const std::map<std::string, int> kExpand = {
    {"xdrop", BEIG_EXPAND_XDROP}, {"powered", BEIG_EXPAND_POWERED}, {"random", BEIG_EXPAND_RANDOM}};
const std::map<std::string, int> kPrecond = {{"identity", BEIG_PRECOND_IDENTITY}, {"diagonal", BEIG_PRECOND_DIAGONAL}};

int fail(const std::string& msg) {
    std::cerr << "error: " << msg << "\n";
    return kInput;
}

std::string g17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

// JSON number / string / array helpers (finite doubles as %.17g, else null)
std::string jnum(double v) { return std::isfinite(v) ? g17(v) : "null"; }
std::string jstr(const std::string& s) { return "\"" + s + "\""; }
std::string jarr(const std::vector<double>& v) {
    std::string s = "[";
    for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + jnum(v[i]);
    return s + "]";
}

// ---------------------------------------------------------------- argument parsing
bool parse_args(int argc, char** argv, int first, Opts& o, std::string& err, bool theory) {
    std::map<std::string, std::string*> str = {
        {"--matrix", &o.matrix}, {"--gen", &o.gen},           {"--solver", &o.solver}, {"--strategy", &o.strategy},
        {"--expand-mode", &o.expand}, {"--precond", &o.precond}, {"--out", &o.out},    {"--format", &o.format}};
    std::map<std::string, int*> ints = {{"--nev", &o.n_ev},     {"--nex", &o.n_ex},         {"--nes", &o.n_es},
                                        {"--max-iters", &o.max_iters}, {"--cg-iters", &o.cg_iters}, {"--je", &o.j_e},
                                        {"--js", &o.j_s},       {"--jp", &o.j_p},           {"--jwarm", &o.j_warm},
                                        {"--device", &o.device}, {"--trials", &o.trials}};
    std::map<std::string, double*> dbls = {{"--tol", &o.tol}, {"--shift", &o.shift}, {"--mu", &o.mu},
                                           {"--rwarm", &o.r_warm}, {"--op-shift", &o.op_shift}};
    std::map<std::string, bool*> flags = {{"--spd-shift", &o.spd_shift}, {"--profile", &o.profile},
                                          {"--largest", &o.largest}};
    for (int i = first; i < argc; ++i) {
        const std::string a = argv[i];
        if (theory && a.rfind("--", 0) != 0) {  // positional suite name
            o.suite = a;
            continue;
        }
        if (flags.count(a)) {
            *flags[a] = true;
            continue;
        }
        if (i + 1 >= argc) {
            err = a + " needs a value";
            return false;
        }
        const std::string v = argv[++i];
        char* end = nullptr;
        if (str.count(a)) {
            *str[a] = v;
        } else if (ints.count(a)) {
            *ints[a] = static_cast<int>(std::strtol(v.c_str(), &end, 10));
        } else if (dbls.count(a)) {
            *dbls[a] = std::strtod(v.c_str(), &end);
            if (a == "--op-shift") o.op_shifted = true;
        } else if (a == "--seed") {
            o.seed = std::strtoull(v.c_str(), &end, 10);
        } else {
            err = "unknown option " + a;
            return false;
        }
        if (end && *end) {
            err = a + ": not a number: " + v;
            return false;
        }
    }
    auto member = [&](const std::string& v, const std::map<std::string, int>& m, const char* what) {
        if (m.count(v)) return true;
        err = std::string(what) + ": unknown value " + v;
        return false;
    };
    if (theory) return true;
    return member(o.solver, kSolvers, "--solver") && member(o.strategy, kStrategies, "--strategy") &&
           member(o.expand, kExpand, "--expand-mode") && member(o.precond, kPrecond, "--precond") &&
           (o.format == "csv" || o.format == "json" || (err = "--format: csv | json", false));
}

// ---------------------------------------------------------------- library calls
struct Matrix {
    beig_matrix* m = nullptr;
    ~Matrix() { beig_matrix_destroy(m); }
};
struct Result {
    beig_result* r = nullptr;
    ~Result() { beig_result_destroy(r); }
};

// -1: continue; otherwise the exit code
int open_matrix(const Opts& o, Matrix& mh) {
    if (o.matrix.empty() == o.gen.empty()) return fail("exactly one of --matrix and --gen is required");
    int rc = o.matrix.empty() ? beig_matrix_gen(&mh.m, o.gen.c_str()) : beig_matrix_read(&mh.m, o.matrix.c_str());
    if (rc != BEIG_OK) return fail(beig_last_error());
    if (o.spd_shift) {
        double lam = 0.0;
        beig_matrix* shifted = nullptr;
        if ((rc = beig_matrix_lambda_min(mh.m, &lam)) != BEIG_OK ||
            (rc = beig_matrix_spd_shift(&shifted, mh.m, lam)) != BEIG_OK)
            return fail(beig_last_error());
        beig_matrix_destroy(mh.m);
        mh.m = shifted;
    }
    return -1;
}

struct Run {
    std::string strategy;
    int rc = BEIG_OK;
    std::string err;
    int status = BEIG_STATUS_MAX_ITERS, iterations = 0;
    std::vector<beig_iter_record> hist;
    std::vector<double> values;
    beig_work_summary work{};
    double r_final = -1.0;
    double seconds = 0.0;
    beig_kernel_stat kstats[BEIG_KERNEL_CLASSES] = {};
};

Run solve_once(const Opts& o, const beig_matrix* m, const std::string& strategy) {
    Run run;
    run.strategy = strategy;
    beig_solver_config cfg;
    beig_solver_config_default(&cfg);
    cfg.n_ev = o.n_ev;
    cfg.n_ex = o.n_ex;
    cfg.n_es = o.n_es;
    cfg.tol = o.tol;
    cfg.max_iters = o.max_iters;
    cfg.shift = o.shift;
    cfg.cg_iters = o.cg_iters;
    cfg.precond = kPrecond.at(o.precond);
    cfg.expand_mode = kExpand.at(o.expand);
    cfg.seed = o.seed;
    beig_strategy_config sc;
    beig_strategy_config_default(&sc);
    sc.kind = kStrategies.at(strategy);
    sc.j_e = o.j_e;
    sc.j_s = o.j_s;
    sc.mu = o.mu;
    sc.j_p = o.j_p;
    sc.j_warm = o.j_warm;
    sc.r_warm = o.r_warm;
    beig_solve_ext ext;
    beig_solve_ext_default(&ext);
    ext.device = o.device;
    ext.profile = o.profile ? 1 : 0;
    ext.which = o.largest ? BEIG_WHICH_LARGEST : BEIG_WHICH_SMALLEST;
    if (o.op_shifted) {
        ext.op_mode = BEIG_OP_SHIFTED;
        ext.op_shift = o.op_shift;
    }
    Result rh;
    run.rc = beig_solve_ex(&rh.r, m, kSolvers.at(o.solver), &cfg, &sc, nullptr, 0, &ext);
    if (run.rc != BEIG_OK) {
        run.err = beig_last_error();
        return run;
    }
    run.status = beig_result_status(rh.r);
    run.iterations = beig_result_iterations(rh.r);
    run.hist.resize(static_cast<size_t>(beig_result_history_len(rh.r)));
    if (!run.hist.empty()) beig_result_history(rh.r, run.hist.data(), static_cast<int>(run.hist.size()));
    run.r_final = run.hist.empty() ? -1.0 : run.hist.back().r_overall;
    run.values.resize(static_cast<size_t>(beig_result_nev(rh.r)));
    beig_result_values(rh.r, run.values.data(), static_cast<int>(run.values.size()));
    beig_result_work(rh.r, &run.work);
    run.seconds = beig_result_seconds(rh.r);
    if (o.profile)
        for (int k = 0; k < BEIG_KERNEL_CLASSES; ++k) beig_result_kernel_stats(rh.r, k, &run.kstats[k]);
    return run;
}

const char* status_name(int s) {
    return s == BEIG_STATUS_CONVERGED ? "converged" : s == BEIG_STATUS_STAGNATED ? "stagnated" : "max_iters";
}

std::string event_name(const beig_iter_record& h) {
    if (h.event == BEIG_EVENT_SHRINK) return "shrink";
    if (h.event == BEIG_EVENT_EXPAND) return "expand";
    if (h.event == BEIG_EVENT_LOCK) return "lock(" + std::to_string(h.lock_count) + ")";
    return "none";
}

std::string work_json(const beig_work_summary& w) {
    return "{\"spmv_cols\": " + std::to_string(w.spmv_cols) + ", \"solve_cols\": " + std::to_string(w.solve_cols) +
           ", \"ortho_flops\": " + std::to_string(w.ortho_flops) + ", \"rr_flops\": " + std::to_string(w.rr_flops) +
           ", \"combined\": " + jnum(w.combined) + "}";
}

// payload to --out (summary to stdout) or to stdout (summary to stderr)
int deliver(const Opts& o, const std::string& payload, const std::string& summary) {
    if (o.out.empty()) {
        std::cout << payload;
        std::cerr << summary;
        return -1;
    }
    std::ofstream f(o.out, std::ios::binary);
    if (!f || !(f << payload).flush()) return fail("cannot write '" + o.out + "'");
    std::cout << summary;
    return -1;
}

std::string profile_summary(const Run& r) {
    static const char* names[BEIG_KERNEL_CLASSES] = {"spmm", "gram", "gemm", "syev", "chol", "residual", "other"};
    std::ostringstream s;
    s << "device: seconds=" << g17(r.seconds);
    for (int k = 0; k < BEIG_KERNEL_CLASSES; ++k)
        if (r.kstats[k].launches)
            s << " " << names[k] << "=" << r.kstats[k].launches << "x/" << g17(r.kstats[k].ms) << "ms";
    return s.str() + "\n";
}

// ---------------------------------------------------------------- subcommands
int cmd_solve(const Opts& o) {
    Matrix mh;
    if (int rc = open_matrix(o, mh); rc >= 0) return rc;
    const Run r = solve_once(o, mh.m, o.strategy);
    if (r.rc != BEIG_OK) return fail(r.err);
    std::ostringstream p;
    if (o.format == "csv") {
        p << "iteration,r_overall,n_now,event,spmv_cols_cum,solve_cols_cum,ortho_flops_cum,rr_dim\n";
        for (const auto& h : r.hist)
            p << h.iteration << ',' << g17(h.r_overall) << ',' << h.n_now << ',' << event_name(h) << ','
              << h.spmv_cols << ',' << h.solve_cols << ',' << h.ortho_flops << ',' << h.rr_dim << '\n';
    } else {
        p << "{\n  \"command\": \"solve\",\n  \"solver\": " << jstr(o.solver) << ",\n  \"strategy\": "
          << jstr(o.strategy) << ",\n  \"status\": " << jstr(status_name(r.status)) << ",\n  \"iterations\": "
          << r.iterations << ",\n  \"r_final\": " << jnum(r.r_final) << ",\n  \"values\": " << jarr(r.values)
          << ",\n  \"work\": " << work_json(r.work) << ",\n  \"history\": [";
        for (size_t i = 0; i < r.hist.size(); ++i) {
            const auto& h = r.hist[i];
            p << (i ? "," : "") << "\n    {\"iteration\": " << h.iteration << ", \"r_overall\": " << jnum(h.r_overall)
              << ", \"n_now\": " << h.n_now << ", \"event\": " << jstr(event_name(h))
              << ", \"spmv_cols_cum\": " << h.spmv_cols << ", \"solve_cols_cum\": " << h.solve_cols
              << ", \"ortho_flops_cum\": " << h.ortho_flops << ", \"rr_dim\": " << h.rr_dim << "}";
        }
        p << "\n  ]\n}\n";
    }
    std::ostringstream s;
    s << "solver=" << o.solver << " strategy=" << o.strategy << " status=" << status_name(r.status)
      << " iterations=" << r.iterations << " r_final=" << g17(r.r_final) << " combined_work=" << g17(r.work.combined)
      << "\nvalues:";
    for (double v : r.values) s << ' ' << g17(v);
    s << "\n";
    if (o.profile) s << profile_summary(r);
    if (int rc = deliver(o, p.str(), s.str()); rc >= 0) return rc;
    return r.status == BEIG_STATUS_CONVERGED ? kOk : kNotConverged;
}

int worker_cap() {
    if (const char* e = std::getenv("BLOCKEIG_THREADS"))
        if (int v = std::atoi(e); v >= 1) return v;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(std::min(4u, hw)) : 1;
}

int cmd_compare(const Opts& o) {
    Matrix mh;
    if (int rc = open_matrix(o, mh); rc >= 0) return rc;
    double na = 0.0;
    beig_matrix_norm_est(mh.m, &na);  // shared cache warmed before the workers start
    const std::vector<std::string> names = {"none", "fix", "slope", "slopek"};
    std::vector<Run> runs(names.size());
    const size_t cap = static_cast<size_t>(worker_cap());
    for (size_t b = 0; b < names.size(); b += cap) {  // concurrent solves on ONE handle
        std::vector<std::future<Run>> fut;
        for (size_t i = b; i < std::min(names.size(), b + cap); ++i)
            fut.push_back(std::async(std::launch::async, [&, i] { return solve_once(o, mh.m, names[i]); }));
        for (size_t i = b; i < std::min(names.size(), b + cap); ++i) runs[i] = fut[i - b].get();
    }
    for (const auto& r : runs)
        if (r.rc != BEIG_OK) return fail("strategy " + r.strategy + ": " + r.err);
    const double base = runs[0].work.combined;
    auto save = [&](size_t i) { return i == 0 || base <= 0 ? 0.0 : 100.0 * (1.0 - runs[i].work.combined / base); };
    std::ostringstream p;
    if (o.format == "csv") {
        p << "strategy,status,iterations,r_final,spmv_cols,solve_cols,ortho_flops,rr_flops,combined_work,save_pct\n";
        for (size_t i = 0; i < runs.size(); ++i) {
            const auto& r = runs[i];
            p << r.strategy << ',' << status_name(r.status) << ',' << r.iterations << ',' << g17(r.r_final) << ','
              << r.work.spmv_cols << ',' << r.work.solve_cols << ',' << r.work.ortho_flops << ',' << r.work.rr_flops
              << ',' << g17(r.work.combined) << ',' << g17(save(i)) << '\n';
        }
    } else {
        p << "{\n  \"command\": \"compare\",\n  \"solver\": " << jstr(o.solver) << ",\n  \"rows\": [";
        for (size_t i = 0; i < runs.size(); ++i) {
            const auto& r = runs[i];
            p << (i ? "," : "") << "\n    {\"strategy\": " << jstr(r.strategy) << ", \"status\": "
              << jstr(status_name(r.status)) << ", \"iterations\": " << r.iterations << ", \"r_final\": "
              << jnum(r.r_final) << ", \"values\": " << jarr(r.values) << ", \"work\": " << work_json(r.work)
              << ", \"save_pct\": " << jnum(save(i)) << "}";
        }
        p << "\n  ]\n}\n";
    }
    std::ostringstream s;
    for (size_t i = 0; i < runs.size(); ++i)
        s << "strategy=" << runs[i].strategy << " status=" << status_name(runs[i].status)
          << " iterations=" << runs[i].iterations << " combined_work=" << g17(runs[i].work.combined)
          << " save_pct=" << g17(save(i)) << "\n";
    if (int rc = deliver(o, p.str(), s.str()); rc >= 0) return rc;
    for (const auto& r : runs)
        if (r.status != BEIG_STATUS_CONVERGED) return kNotConverged;
    return kOk;
}

int cmd_gen(const Opts& o) {
    if (o.gen.empty()) return fail("--gen is required");
    if (o.out.empty()) return fail("--out is required");
    Matrix mh;
    if (beig_matrix_gen(&mh.m, o.gen.c_str()) != BEIG_OK || beig_matrix_write(mh.m, o.out.c_str()) != BEIG_OK)
        return fail(beig_last_error());
    std::cout << "wrote " << beig_matrix_rows(mh.m) << "x" << beig_matrix_rows(mh.m) << " matrix ("
              << beig_matrix_nnz_lower(mh.m) << " stored entries) to " << o.out << "\n";
    return kOk;
}

// the analysis suites live outside this build's hot path: the library reports
// BEIG_ERR_INVALID for them (include/blockeig.h), surfaced as an input error
int cmd_theory(const Opts& o) {
    static const char* suites[] = {"example3x3", "rate", "decomp", "perturb", "main", "all"};
    bool known = false;
    for (const char* s : suites) known = known || o.suite == s;
    if (!known) return fail("theory: unknown suite " + o.suite);
    beig_example3x3 ex{};
    if (beig_theory_example3x3(&ex) != BEIG_OK) return fail(beig_last_error());
    std::cout << "example3x3: rho_x1=" << g17(ex.rho_x1) << "\n";
    return kOk;
}

void usage() {
    std::cerr << "usage: blockeig <solve|compare|gen|theory> [options]\n"
                 "  --matrix FILE | --gen SPEC   (laplacian1d:N | diag:v1,v2,... | diag-geom:N,RATIO)\n"
                 "  --solver si|sd|lobpcg|tracemin --nev --nex --nes --tol --max-iters --shift --cg-iters --seed\n"
                 "  --strategy none|fix|slope|slopek --je --js --mu --jp --jwarm --rwarm\n"
                 "  --expand-mode xdrop|powered|random --precond identity|diagonal --spd-shift\n"
                 "  --out FILE --format csv|json\n"
                 "  B200 extensions: --device N --op-shift C --largest --profile\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kInput;
    }
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
        usage();
        return kOk;
    }
    Opts o;
    std::string err;
    if (cmd != "solve" && cmd != "compare" && cmd != "gen" && cmd != "theory") {
        usage();
        return kInput;
    }
    if (!parse_args(argc, argv, 2, o, err, cmd == "theory")) return fail(err);
    if (cmd == "solve") return cmd_solve(o);
    if (cmd == "compare") return cmd_compare(o);
    if (cmd == "gen") return cmd_gen(o);
    return cmd_theory(o);
}
