// sewald-cli: command-line front end of the B200 Spectral Ewald engine
// (SURVEY §8 f row 2; SPEC.md module `cli`). The reference
// ships it as a stub (proj/tools/main.cpp:1, CMakeLists.txt:35 `sewald-cli`).
//
//   sewald-cli params   print the full EstimateReport of select_parameters (--json: one JSON line)
//   sewald-cli gen      write a seeded synthetic particle file
//   sewald-cli compute  full potential of a particle file (or a seeded system) -> CSV
//   sewald-cli validate SE against the analytic oracles (direct 0P / Ewald 3P / q-sums 2P, 1P)
//   sewald-cli sweep    --axis tol|P|rc|kinf: CSV of (parameter, measured error, estimated error)
//   sewald-cli bench    fixed-N_rc scaling runs: CSV of (N, xi, wall time, time / N)
//
// Everything numeric goes through the drop-in C++ API (include/sewald/*.h ->
// libsewald_gpu.so: sm_100a kernels). Exit codes: 0 ok, 2 usage
// or input error, 3 validation failure, 4 infeasible parameters.
#include "sewald/estimates.h"
#include "sewald/fourier.h"
#include "sewald/realspace.h"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace sewald;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Infeasible : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const char* kUsage =
    "usage: sewald-cli <params|gen|compute|validate|sweep|bench> [options]\n"
    "  --kernel stokeslet|stresslet|rotlet   --periodicity 0..3   --cell Lx,Ly,Lz\n"
    "  --tol-abs T | --tol-rel T              --xi X | --nrc N    --window pkb|kb|tg   --fm F\n"
    "  --n N --seed S --Q Q (generated systems)   --in FILE   --out FILE   --json\n"
    "  --no-pollution-adjust   --threads T (accepted; the sums run on the GPU)\n"
    "  sweep: --axis tol|P|rc|kinf     bench: --n0 N --doublings J --reps R\n"
    "  validate: --oracle auto|direct0p|ewald3p|qsum2p|qsum1p\n";

// ------------------------------------------------------------ options

struct Opts {
    std::string cmd;
    std::map<std::string, std::string> kv;
    bool has(const std::string& k) const { return kv.count(k) > 0; }
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    double num(const std::string& k, double def) const {
        if (!has(k)) return def;
        try {
            size_t pos = 0;
            const double v = std::stod(get(k), &pos);
            if (pos != get(k).size()) throw std::invalid_argument("");
            return v;
        } catch (const std::exception&) {
            throw Usage("--" + k + " expects a number, got '" + get(k) + "'");
        }
    }
    long integer(const std::string& k, long def) const {
        const double v = num(k, (double)def);
        if (v != std::floor(v)) throw Usage("--" + k + " expects an integer");
        return (long)v;
    }
};

const std::map<std::string, bool> kFlags = {  // name -> takes a value
    {"kernel", true}, {"periodicity", true}, {"cell", true}, {"tol-abs", true}, {"tol-rel", true},
    {"xi", true}, {"nrc", true}, {"window", true}, {"fm", true}, {"seed", true}, {"in", true},
    {"out", true}, {"no-pollution-adjust", false}, {"threads", true}, {"n", true}, {"Q", true},
    {"json", false}, {"axis", true}, {"n0", true}, {"doublings", true}, {"reps", true}, {"oracle", true},
    {"kmax", true}};

Opts parse(int argc, char** argv) {
    if (argc < 2) throw Usage("missing subcommand");
    Opts o;
    o.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) throw Usage("unexpected argument '" + a + "'");
        a = a.substr(2);
        auto it = kFlags.find(a);
        if (it == kFlags.end()) throw Usage("unknown option --" + a);
        if (it->second) {
            if (i + 1 >= argc) throw Usage("--" + a + " needs a value");
            o.kv[a] = argv[++i];
        } else {
            o.kv[a] = "1";
        }
    }
    if (o.has("tol-abs") && o.has("tol-rel")) throw Usage("--tol-abs and --tol-rel are mutually exclusive");
    if (o.has("xi") && o.has("nrc")) throw Usage("--xi and --nrc are mutually exclusive");
    return o;
}

Kernel parse_kernel(const std::string& s) {
    Kernel k;
    if (!kernel_from_name(s, k)) throw Usage("unknown kernel '" + s + "'");
    return k;
}

Cell parse_cell(const std::string& s) {
    Cell c;
    std::stringstream ss(s);
    std::string tok;
    int i = 0;
    while (std::getline(ss, tok, ',')) {
        if (i >= 3) throw Usage("--cell takes three lengths");
        try {
            c.L[i++] = std::stod(tok);
        } catch (const std::exception&) {
            throw Usage("--cell: bad length '" + tok + "'");
        }
    }
    if (i != 3) throw Usage("--cell takes three lengths Lx,Ly,Lz");
    return c;
}

// ------------------------------------------------------ particle files

// Format: header `# kernel=<k> D=<d> L=<L1> <L2> <L3> N=<n>`,
// then `x y z s1 s2 s3` (stokeslet / rotlet) or `x y z q1 q2 q3 n1 n2 n3`
// (stresslet) per particle; other `#` lines are comments.
SourceSystem read_particles(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Usage("cannot open particle file '" + path + "'");
    SourceSystem s;
    bool header = false;
    long n_decl = -1;
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const auto first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos) continue;
        if (line[first] == '#') {
            if (line.find("kernel=") == std::string::npos) continue;
            std::stringstream ss(line.substr(first + 1));
            std::string tok;
            while (ss >> tok) {
                const auto eq = tok.find('=');
                if (eq == std::string::npos) continue;
                const std::string key = tok.substr(0, eq), val = tok.substr(eq + 1);
                try {
                    if (key == "kernel") s.kind = parse_kernel(val);
                    else if (key == "D") s.d = std::stoi(val);
                    else if (key == "N") n_decl = std::stol(val);
                    else if (key == "L") {
                        s.cell.L[0] = std::stod(val);
                        if (!(ss >> s.cell.L[1] >> s.cell.L[2])) throw std::invalid_argument("L");
                    }
                } catch (const Usage&) {
                    throw;
                } catch (const std::exception&) {
                    throw Usage(path + ":" + std::to_string(lineno) + ": bad header field '" + tok + "'");
                }
            }
            header = true;
            continue;
        }
        if (!header) throw Usage(path + ":" + std::to_string(lineno) + ": data before the '# kernel=...' header");
        std::stringstream ss(line);
        const int cols = s.kind == Kernel::stresslet ? 9 : 6;
        double v[9];
        for (int c = 0; c < cols; ++c)
            if (!(ss >> v[c]))
                throw Usage(path + ":" + std::to_string(lineno) + ": expected " + std::to_string(cols) + " numbers");
        std::string extra;
        if (ss >> extra) throw Usage(path + ":" + std::to_string(lineno) + ": trailing text '" + extra + "'");
        s.x.push_back({v[0], v[1], v[2]});
        s.f.push_back({v[3], v[4], v[5]});
        if (s.kind == Kernel::stresslet) s.nu.push_back({v[6], v[7], v[8]});
    }
    if (!header) throw Usage(path + ": missing '# kernel=... D=... L=... N=...' header");
    if (n_decl >= 0 && (size_t)n_decl != s.x.size())
        throw Usage(path + ": header declares N=" + std::to_string(n_decl) + " but the file has " +
                    std::to_string(s.x.size()) + " particles");
    return s;
}

std::string fmt17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

void write_particles(std::ostream& out, const SourceSystem& s) {
    out << "# kernel=" << kernel_name(s.kind) << " D=" << s.d << " L=" << fmt17(s.cell.L[0]) << ' '
        << fmt17(s.cell.L[1]) << ' ' << fmt17(s.cell.L[2]) << " N=" << s.size() << '\n';
    for (size_t i = 0; i < s.size(); ++i) {
        out << fmt17(s.x[i][0]) << ' ' << fmt17(s.x[i][1]) << ' ' << fmt17(s.x[i][2]) << ' ' << fmt17(s.f[i][0])
            << ' ' << fmt17(s.f[i][1]) << ' ' << fmt17(s.f[i][2]);
        if (s.kind == Kernel::stresslet)
            out << ' ' << fmt17(s.nu[i][0]) << ' ' << fmt17(s.nu[i][1]) << ' ' << fmt17(s.nu[i][2]);
        out << '\n';
    }
}

// Seeded system: std::mt19937_64, positions uniform in the cell,
// strength components uniform in [-1, 1] rescaled a posteriori to the target Q
// (§4.1.1), stresslet normals uniform on the sphere.
SourceSystem generate(Kernel kind, int d, const Cell& cell, long N, unsigned long long seed, double Q) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u01(0.0, 1.0), usym(-1.0, 1.0);
    std::normal_distribution<double> gauss;
    SourceSystem s;
    s.kind = kind;
    s.d = d;
    s.cell = cell;
    s.x.resize(N);
    s.f.resize(N);
    for (auto& p : s.x)
        for (int a = 0; a < 3; ++a) p[a] = u01(rng) * cell.L[a];
    for (auto& f : s.f)
        for (int a = 0; a < 3; ++a) f[a] = usym(rng);
    if (kind == Kernel::stresslet) {
        s.nu.resize(N);
        for (auto& n : s.nu) {
            Vec3 g{gauss(rng), gauss(rng), gauss(rng)};
            const double r = std::sqrt(norm2(g));
            n = (1.0 / r) * g;
        }
    }
    if (N > 0 && Q > 0.0) {
        const double q0 = source_quantity(s);
        const double sc = std::sqrt(Q / q0);
        for (auto& f : s.f) f = sc * f;
    }
    return s;
}

// ------------------------------------------------------- parameters

// N_rc defaults (PAPER.md Table "Expected average number of points within a
// ball", uniform system): stokeslet / rotlet 2500, 950, 450, 400 for D = 0..3;
// stresslet 6000, 1600, 800, 800.
double default_nrc(Kernel kind, int d) {
    static const double sr[4] = {2500, 950, 450, 400}, st[4] = {6000, 1600, 800, 800};
    return kind == Kernel::stresslet ? st[d] : sr[d];
}

// xi from a fixed N_rc: r_c = (3 N_rc V / (4 pi N))^(1/3),
// then the xi whose real-space truncation estimate at r_c equals tau.
double xi_from_nrc(Kernel kind, const Cell& cell, long N, double Q, double nrc, const ToleranceSpec& tol) {
    const double V = cell.volume(), L = std::cbrt(V);
    const double rc = std::cbrt(3.0 * nrc * V / (4.0 * M_PI * (double)N));
    // the absolute tolerance depends on xi through U for relative tolerances; iterate
    double lo = 1e-3 / rc, hi = 1e3 / rc;
    for (int it = 0; it < 200; ++it) {
        const double xi = std::sqrt(lo * hi);
        const double tau = tol.absolute(potential_rms(kind, L, Q, xi));
        if (realspace_trunc_error(kind, xi, rc, L, Q) > tau) lo = xi; else hi = xi;
        if (hi / lo < 1 + 1e-13) break;
    }
    return hi;
}

struct Setup {
    SourceSystem sys;
    ToleranceSpec tol;
    SelectionOptions sel;
    double xi = 10.0;
    double Q = 1.0;
};

Setup setup(const Opts& o, bool need_system) {
    Setup s;
    if (o.has("in")) {
        s.sys = read_particles(o.get("in"));
        if (o.has("kernel") && parse_kernel(o.get("kernel")) != s.sys.kind)
            throw Usage("--kernel disagrees with the particle file header");
        if (o.has("periodicity") && o.integer("periodicity", 3) != s.sys.d)
            throw Usage("--periodicity disagrees with the particle file header");
    } else {
        if (!o.has("kernel") || !o.has("periodicity")) throw Usage("--kernel and --periodicity are required");
        const Kernel kind = parse_kernel(o.get("kernel"));
        const long d = o.integer("periodicity", 3);
        if (d < 0 || d > 3) throw Usage("--periodicity must be 0..3");
        const Cell cell = o.has("cell") ? parse_cell(o.get("cell")) : Cell{};
        const long N = o.integer("n", need_system ? 1000 : 0);
        if (N < 0) throw Usage("--n must be >= 0");
        s.sys = generate(kind, (int)d, cell, N, (unsigned long long)o.integer("seed", 1), o.num("Q", 1.0));
    }
    s.tol.value = o.has("tol-rel") ? o.num("tol-rel", 1e-8) : o.num("tol-abs", 1e-8);
    s.tol.relative = o.has("tol-rel");
    if (!(s.tol.value > 0.0)) throw Usage("tolerance must be positive");
    s.sel.f_m = (int)o.integer("fm", 4);
    s.sel.pollution_fix = !o.has("no-pollution-adjust");
    const std::string w = o.get("window", "pkb");
    if (w != "pkb" && w != "kb" && w != "tg") throw Usage("--window must be pkb, kb or tg");
    s.sel.window = window_kind_from_name(w);
    s.Q = s.sys.size() > 0 ? source_quantity(s.sys) : o.num("Q", 1.0);
    if (!(s.Q > 0.0)) s.Q = 1.0;  // all-zero strengths: any Q selects valid parameters
    if (o.has("nrc")) {
        const double nrc = o.num("nrc", 0.0);
        if (!(nrc > 0.0)) throw Usage("--nrc must be positive");
        const long N = std::max<long>(1, (long)s.sys.size());
        s.xi = xi_from_nrc(s.sys.kind, s.sys.cell, N, s.Q, nrc, s.tol);
    } else {
        s.xi = o.num("xi", 10.0);
        if (!(s.xi > 0.0)) throw Usage("--xi must be positive");
    }
    return s;
}

ParameterSelection select(const Setup& s, double tol_value) {
    ToleranceSpec t = s.tol;
    t.value = tol_value;
    try {
        return select_parameters(s.sys.kind, s.sys.d, s.sys.cell, s.Q, s.xi, t, s.sel);
    } catch (const std::invalid_argument& e) {
        throw Infeasible(e.what());
    } catch (const std::domain_error& e) {
        throw Infeasible(e.what());
    }
}

// ------------------------------------------------------------ report

std::vector<std::pair<std::string, std::string>> report_fields(const ParameterSelection& ps) {
    const EwaldParams& p = ps.params;
    const EstimateReport& r = ps.report;
    std::vector<std::pair<std::string, std::string>> f;
    auto add = [&](const std::string& k, double v) { f.emplace_back(k, fmt17(v)); };
    auto addi = [&](const std::string& k, long v) { f.emplace_back(k, std::to_string(v)); };
    auto add3 = [&](const std::string& k, const std::array<int, 3>& v) {
        f.emplace_back(k, std::to_string(v[0]) + "," + std::to_string(v[1]) + "," + std::to_string(v[2]));
    };
    f.emplace_back("kernel", kernel_name(p.kind));
    addi("d", p.d);
    add("xi", p.xi);
    add("rc", p.rc);
    add("h", p.grid.h);
    add3("M", p.grid.M);
    f.emplace_back("window", window_kind_name(p.window.kind));
    addi("P", p.window.P);
    add("beta", p.window.beta);
    addi("nu", p.window.nu);
    add("alpha", p.window.alpha);
    addi("f_m", p.grid.f_m);
    add("tau_abs", r.tau_abs);
    add("U", r.U);
    add("kinf", r.kinf);
    add("kinf_grid", p.grid.kinf());
    add("fourier_trunc", r.fourier_trunc);
    add("realspace_trunc", r.realspace_trunc);
    add("window_err", r.window_err);
    add("h_estimate", r.h_estimate);
    addi("P_estimate", r.P_estimate);
    add("h_target", r.h_target);  // pollution-adjusted (raw: h_estimate, P_estimate)
    addi("P_target", r.P_target);
    addi("rc_clamped", r.rc_clamped);
    addi("kinf_clamped", r.kinf_clamped);
    addi("window_saturated", r.window_saturated);
    addi("tg_support_from_pkb", r.tg_support_from_pkb);
    if (p.d < 3) {  // SPEC: the d = 3 report omits padding / upsampling (§4.6 step 5)
        add("R", p.R);
        add3("M_ext", p.grid.M_ext);
        add("s0", p.upsampling.s0);
        add("s_star", p.upsampling.s_star);
        add3("k_star", p.upsampling.k_star);
        add("s0_raw", p.upsampling.s0_raw);
        add("s_star_raw", p.upsampling.s_star_raw);
    }
    return f;
}

void print_report(std::ostream& out, const ParameterSelection& ps, bool json, const char* prefix = "") {
    const auto f = report_fields(ps);
    if (json) {
        out << '{';
        for (size_t i = 0; i < f.size(); ++i) {
            const bool str = f[i].first == "kernel" || f[i].first == "window" || f[i].second.find(',') != std::string::npos;
            out << (i ? ", " : "") << '"' << f[i].first << "\": ";
            if (str) out << '"' << f[i].second << '"'; else out << f[i].second;
        }
        out << "}\n";
        return;
    }
    for (const auto& kv : f) out << prefix << kv.first << " = " << kv.second << '\n';
}

// ----------------------------------------------------------- commands

std::ostream* open_out(const Opts& o, std::ofstream& file) {
    if (!o.has("out")) return &std::cout;
    file.open(o.get("out"));
    if (!file) throw Usage("cannot write '" + o.get("out") + "'");
    return &file;
}

int cmd_params(const Opts& o) {
    Setup s = setup(o, false);
    const ParameterSelection ps = select(s, s.tol.value);
    print_report(std::cout, ps, o.has("json"));
    return 0;
}

int cmd_gen(const Opts& o) {
    Setup s = setup(o, true);
    std::ofstream file;
    write_particles(*open_out(o, file), s.sys);
    return 0;
}

int cmd_compute(const Opts& o) {
    Setup s = setup(o, true);
    const ParameterSelection ps = select(s, s.tol.value);
    const TargetSet t = TargetSet::from_sources(s.sys);
    const std::vector<Vec3> u = s.sys.size() ? full_potential(s.sys, t, ps.params) : std::vector<Vec3>{};
    std::ofstream file;
    std::ostream& out = *open_out(o, file);
    print_report(out, ps, false, "# ");
    out << "index,x,y,z,u1,u2,u3\n";
    for (size_t i = 0; i < u.size(); ++i)
        out << i << ',' << fmt17(s.sys.x[i][0]) << ',' << fmt17(s.sys.x[i][1]) << ',' << fmt17(s.sys.x[i][2]) << ','
            << fmt17(u[i][0]) << ',' << fmt17(u[i][1]) << ',' << fmt17(u[i][2]) << '\n';
    return 0;
}

struct Measured {
    double abs_err, rel_err;
};

// The SE part a given oracle checks (targets = sources):
//   D = 0: full potential vs the direct sum (starred);
//   D = 1, 2, 3: Fourier part vs the q-sums / direct Ewald (D = 3 stresslet:
//   both with the zero mode of PAPER.md:775).
Measured measure(const SourceSystem& sys, const EwaldParams& p, const std::array<int, 3>& kmax) {
    const TargetSet t = TargetSet::from_sources(sys);
    std::vector<Vec3> u, ref;
    if (sys.d == 0) {
        u = full_potential(sys, t, p);
        ref = direct_sum_0p(sys, t, true);
    } else {
        u = se_fourier_potential(sys, t, p);
        if (sys.kind == Kernel::stresslet && sys.d == 3) {
            const std::vector<Vec3> z = stresslet_zero_mode_3p(t, sys);
            for (size_t i = 0; i < u.size(); ++i) u[i] += z[i];
        }
        ref = fourier_reference_potential(sys, t, p.xi, kmax);
    }
    double rel = 0.0;
    try {
        rel = rel_rms_error(u, ref);
    } catch (const std::domain_error&) {
        rel = 0.0;
    }
    return {rms_error(u, ref), rel};
}

std::array<int, 3> kmax_of(const Opts& o, double xi, const Cell& cell) {
    std::array<int, 3> k = oracle_kmax(xi, cell);
    if (o.has("kmax")) k = {(int)o.integer("kmax", 0), (int)o.integer("kmax", 0), (int)o.integer("kmax", 0)};
    for (int v : k)
        if (v < 1) throw Usage("--kmax must be >= 1");
    return k;
}

const char* oracle_name(int d) {
    static const char* n[4] = {"direct0p", "qsum1p", "qsum2p", "ewald3p"};
    return n[d];
}

int cmd_validate(const Opts& o) {
    Setup s = setup(o, true);
    if (s.sys.size() > 5000) throw Usage("validate: the oracles are direct sums; use N <= 5000");
    if (s.sys.size() == 0) throw Usage("validate: empty system");
    const std::string want = o.get("oracle", "auto");
    if (want != "auto" && want != oracle_name(s.sys.d))
        throw Usage("--oracle " + want + " does not match periodicity " + std::to_string(s.sys.d) + " (use " +
                    oracle_name(s.sys.d) + ")");
    const ParameterSelection ps = select(s, s.tol.value);
    const Measured m = measure(s.sys, ps.params, kmax_of(o, ps.params.xi, s.sys.cell));
    const double tau = ps.report.tau_abs;
    std::cout << "oracle = " << oracle_name(s.sys.d) << "\nN = " << s.sys.size() << "\ntau_abs = " << fmt17(tau)
              << "\nabs_rms_error = " << fmt17(m.abs_err) << "\nrel_rms_error = " << fmt17(m.rel_err) << '\n';
    if (tau < 1e-13)
        std::cerr << "warning: tolerance at the double-precision floor; the error saturates near 1e-14 relative\n";
    if (m.abs_err > 10.0 * tau) {
        std::cout << "status = FAIL (error > 10 tau)\n";
        return 3;
    }
    std::cout << "status = ok\n";
    return 0;
}

// Rebuild the grid / window tail of select_parameters (estimates.cpp:250-266)
// for a forced window support or grid spacing.
EwaldParams with_grid(const Setup& s, const ParameterSelection& base, double h, int P) {
    EwaldParams p = base.params;
    p.grid = build_grid(s.sys.cell, s.sys.d, h, P, s.sys.kind, s.sel.f_m);
    p.window = WindowSpec::make(s.sel.window, P, p.grid.h);
    if (p.d < 3) {
        p.R = truncation_radius(p.grid.L_ext, p.d);
        p.upsampling = upsampling_params(p.grid, base.report.tau_abs, base.report.U);
    }
    return p;
}

int cmd_sweep(const Opts& o) {
    Setup s = setup(o, true);
    if (s.sys.size() > 5000) throw Usage("sweep: the oracles are direct sums; use N <= 5000");
    const std::string axis = o.get("axis");
    std::ofstream file;
    std::ostream& out = *open_out(o, file);
    const double L = std::cbrt(s.sys.cell.volume());
    const auto kmax = kmax_of(o, s.xi, s.sys.cell);
    if (axis == "tol") {
        out << "tol,measured,estimated\n";
        for (double t = 1e-3; t >= 0.99e-12; t /= 10.0) {
            const ParameterSelection ps = select(s, t);
            const Measured m = measure(s.sys, ps.params, kmax);
            const double est = s.sys.d == 0 ? ps.report.fourier_trunc + ps.report.window_err + ps.report.realspace_trunc
                                            : ps.report.fourier_trunc + ps.report.window_err;
            out << fmt17(t) << ',' << fmt17(m.abs_err) << ',' << fmt17(est) << '\n';
        }
    } else if (axis == "P") {
        // truncation negligible: the grid of a tight tolerance, window support varied
        const ParameterSelection ps = select(s, 1e-13);
        out << "P,measured,estimated\n";
        for (int P = 4; P <= 16; P += 2) {
            const EwaldParams p = with_grid(s, ps, ps.params.grid.h, P);
            const Measured m = measure(s.sys, p, kmax);
            const double P_eff = s.sel.window == WindowKind::tg ? 0.6 * P : (double)P;
            out << P << ',' << fmt17(m.abs_err) << ',' << fmt17(window_error(P_eff, ps.report.U)) << '\n';
        }
    } else if (axis == "kinf") {
        const ParameterSelection ps = select(s, 1e-13);
        out << "kinf,measured,estimated\n";
        for (int Mx = 8; Mx <= ps.params.grid.M[0]; Mx += 4) {
            const EwaldParams p = with_grid(s, ps, s.sys.cell.L[0] / Mx, ps.params.window.P);
            const Measured m = measure(s.sys, p, kmax);
            out << fmt17(p.grid.kinf()) << ',' << fmt17(m.abs_err) << ','
                << fmt17(fourier_trunc_error(s.sys.kind, s.xi, p.grid.kinf(), L, s.Q)) << '\n';
        }
    } else if (axis == "rc") {
        // real-space truncation: u_R(rc) against u_R at a cutoff with negligible tail
        const TargetSet t = TargetSet::from_sources(s.sys);
        const ParameterSelection ps = select(s, 1e-15);
        const double rc_ref = std::min(ps.params.rc, 0.5 * std::min({s.sys.cell.L[0], s.sys.cell.L[1], s.sys.cell.L[2]}));
        const std::vector<Vec3> ref = realspace_potential(s.sys, t, s.xi, rc_ref * 1.3, true, 1);
        out << "rc,measured,estimated\n";
        for (int i = 1; i <= 10; ++i) {
            const double rc = rc_ref * i / 10.0;
            const std::vector<Vec3> u = realspace_potential(s.sys, t, s.xi, rc, true, 1);
            out << fmt17(rc) << ',' << fmt17(rms_error(u, ref)) << ','
                << fmt17(realspace_trunc_error(s.sys.kind, s.xi, rc, L, s.Q)) << '\n';
        }
    } else {
        throw Usage("--axis must be tol, P, rc or kinf");
    }
    return 0;
}

int cmd_bench(const Opts& o) {
    if (!o.has("kernel") || !o.has("periodicity")) throw Usage("--kernel and --periodicity are required");
    if (o.has("in")) throw Usage("bench generates its systems (--n0, --doublings)");
    const Kernel kind = parse_kernel(o.get("kernel"));
    const int d = (int)o.integer("periodicity", 3);
    if (d < 0 || d > 3) throw Usage("--periodicity must be 0..3");
    const long n0 = o.integer("n0", 12500);
    const int J = (int)o.integer("doublings", 4);
    const int reps = (int)o.integer("reps", 3);
    if (n0 < 1 || J < 0 || reps < 1) throw Usage("--n0, --doublings, --reps must be positive");
    const double nrc = o.has("nrc") ? o.num("nrc", 0) : default_nrc(kind, d);
    std::ofstream file;
    std::ostream& out = *open_out(o, file);
    out << "N,xi,M,P,wall_s,s_per_point\n";
    for (int j = 0; j <= J; ++j) {
        Opts oj = o;
        oj.kv["n"] = std::to_string(n0 << j);
        oj.kv["nrc"] = fmt17(nrc);
        oj.kv.erase("xi");
        Setup s = setup(oj, true);
        const ParameterSelection ps = select(s, s.tol.value);
        const TargetSet t = TargetSet::from_sources(s.sys);
        full_potential(s.sys, t, ps.params);  // warm: plans, D = 0 table (excluded, §5.2)
        double best = 1e300;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            full_potential(s.sys, t, ps.params);
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        out << s.sys.size() << ',' << fmt17(s.xi) << ',' << ps.params.grid.M[0] << ',' << ps.params.window.P << ','
            << fmt17(best) << ',' << fmt17(best / (double)s.sys.size()) << '\n';
        out.flush();
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Opts o = parse(argc, argv);
        if (o.cmd == "params") return cmd_params(o);
        if (o.cmd == "gen") return cmd_gen(o);
        if (o.cmd == "compute") return cmd_compute(o);
        if (o.cmd == "validate") return cmd_validate(o);
        if (o.cmd == "sweep") return cmd_sweep(o);
        if (o.cmd == "bench") return cmd_bench(o);
        if (o.cmd == "-h" || o.cmd == "--help" || o.cmd == "help") {
            std::cout << kUsage;
            return 0;
        }
        throw Usage("unknown subcommand '" + o.cmd + "'");
    } catch (const Usage& e) {
        std::cerr << "sewald-cli: " << e.what() << '\n' << kUsage;
        return 2;
    } catch (const Infeasible& e) {
        std::cerr << "sewald-cli: infeasible parameters: " << e.what() << '\n';
        return 4;
    } catch (const std::invalid_argument& e) {
        std::cerr << "sewald-cli: invalid input: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "sewald-cli: " << e.what() << '\n';
        return 1;
    }
}
