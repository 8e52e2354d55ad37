// cli.cpp — `pdb200`, the reference CLI's compute subcommands (proj/tools/main.cpp) on the GPU:
//
//   pdb200 decompose --in PATH [--out PATH] [--format text|binary] [--eps E] [--threads T]
//                    [--serial] [--path gray|wht]
//   pdb200 recompose --in CSV [--out PATH] [--format text|binary]
//   pdb200 coeff LABEL --in PATH [--format text|binary]
//   pdb200 bench [--n-min N] [--n-max N] [--reps R] [--seed S] [--threads T] [--out PATH]
//
// `bench` writes the benchmark CSV of proj/docs/formats.md ("Benchmark CSV") for the three paths
// named there — fast (decompose_parallel), slow (coeff_slow for every string) and
// serial-quaternary — run on the GPU through the reference API, with the seeded generator
// (matrix_seed / random_matrix) and the exact multiplication counts of proj/README.md:113-120.
// bench.py is this repository's measurement; `bench` exists so that callers of the reference CLI
// (and its acceptance criterion 9) find the same subcommand and schema.
//
// Paths may be "-" (stdin/stdout). Exit codes follow main.cpp:140-158: 0 success, 1 usage or
// format error, 2 resource or internal error. `decompose` prints "N=… nonzero=… seconds=…" to
// stderr like main.cpp:42-43 (seconds = read + GPU decomposition + selection + write).
#include <chrono>
#include <cmath>
#include <fstream>
#include <cstring>
#include <iostream>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "paulidecomp_b200/bench.hpp"
#include "paulidecomp_b200/decompose.hpp"
#include "paulidecomp_b200/io.hpp"

using namespace paulidecomp;

namespace {

struct Args {
    std::string cmd, in = "-", out = "-", format = "text", label, path = "gray";
    double eps = 0.0;
    unsigned threads = 1;
    bool serial = false, have_in = false;
    unsigned n_min = 1, n_max = 5, reps = 20;  // bench
    std::uint64_t seed = 1;
};

constexpr unsigned kBenchMaxQubits = 8;

// "--opt value" as an unsigned number; zero rejected unless allowed
std::uint64_t number_arg(const std::string& opt, const std::string& v, bool allow_zero) {
    std::uint64_t x = 0;
    std::size_t used = 0;
    try {
        x = std::stoull(v, &used);
    } catch (...) {
        used = 0;
    }
    if (used == 0 || used != v.size() || v[0] == '-') throw std::invalid_argument(opt + " needs a whole number");
    if (!allow_zero && x == 0) throw std::invalid_argument(opt + " must be positive");
    return x;
}

[[noreturn]] void usage(const std::string& why) { throw std::invalid_argument(why); }

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) usage("a subcommand is required: decompose, recompose, coeff or bench");
    a.cmd = argv[1];
    if (a.cmd != "decompose" && a.cmd != "recompose" && a.cmd != "coeff" && a.cmd != "bench")
        usage("unknown subcommand \"" + a.cmd + "\"");
    for (int k = 2; k < argc; ++k) {
        const std::string s = argv[k];
        auto value = [&]() -> std::string {
            if (k + 1 >= argc) usage("option " + s + " needs a value");
            return argv[++k];
        };
        if (s == "--in") { a.in = value(); a.have_in = true; }
        else if (s == "--out" && a.cmd != "coeff") a.out = value();
        else if (s == "--format") {
            a.format = value();
            if (a.format != "text" && a.format != "binary") usage("--format must be text or binary");
        } else if (s == "--eps" && a.cmd == "decompose") {
            const std::string v = value();
            std::size_t used = 0;
            try { a.eps = std::stod(v, &used); } catch (...) { usage("--eps needs a number"); }
            if (used != v.size() || !(a.eps >= 0.0)) usage("--eps must be a non-negative number");
        } else if (a.cmd == "bench" && (s == "--n-min" || s == "--n-max" || s == "--reps")) {
            const auto v = static_cast<unsigned>(number_arg(s, value(), false));
            (s == "--n-min" ? a.n_min : s == "--n-max" ? a.n_max : a.reps) = v;
        } else if (a.cmd == "bench" && s == "--seed") {
            a.seed = number_arg(s, value(), true);
        } else if (a.cmd == "bench" && s == "--threads") {
            a.threads = static_cast<unsigned>(number_arg(s, value(), false));
        } else if (s == "--threads" && a.cmd == "decompose") {
            const std::string v = value();
            try { a.threads = static_cast<unsigned>(std::stoul(v)); } catch (...) { usage("--threads needs a number"); }
            if (a.threads == 0) usage("--threads must be positive");
        } else if (s == "--serial" && a.cmd == "decompose") a.serial = true;
        else if (s == "--path" && a.cmd == "decompose") {
            a.path = value();
            if (a.path != "gray" && a.path != "wht") usage("--path must be gray or wht");
        } else if (a.cmd == "coeff" && a.label.empty() && !s.empty() && s[0] != '-') a.label = s;
        else usage("unexpected argument \"" + s + "\"");
    }
    if (a.cmd == "bench") {
        if (a.n_min > a.n_max) usage("--n-min must not exceed --n-max");
        if (a.n_max > kBenchMaxQubits) usage("--n-max is capped at 8");
        return a;
    }
    if (!a.have_in) usage("--in is required");
    if (a.cmd == "coeff" && a.label.empty()) usage("coeff needs an operator label");
    return a;
}

MatrixFormat fmt(const Args& a) { return a.format == "binary" ? MatrixFormat::binary : MatrixFormat::text; }

// formats.md "Benchmark CSV": per (N, path) the repetitions, then the rep = -1 summary row
// (master seed, mean seconds, sample standard deviation)
int run_bench(const Args& a, std::ostream& csv) {
    struct BenchPath {
        const char* name;
        std::uint64_t (*mults)(unsigned N);  // proj/README.md:115-120
        PauliDecomposition (*run)(const DenseMatrix&, unsigned threads);
    };
    static const BenchPath paths[] = {
        {"fast", [](unsigned N) { return (std::uint64_t{1} << (2 * N)) * (N + 2 * (std::uint64_t{1} << N) - 1); },
         [](const DenseMatrix& g, unsigned t) { return decompose_parallel(g, t); }},
        {"slow", [](unsigned N) { return (std::uint64_t{1} << (2 * N)) * (N + 1) * (std::uint64_t{1} << N); },
         [](const DenseMatrix& g, unsigned) {
             PauliDecomposition d{g.num_qubits(), std::vector<Complex>(g.element_count())};
             for (std::uint64_t n = 0; n < g.element_count(); ++n) d.coefficients[n] = coeff_slow(g, n);
             return d;
         }},
        {"serial-quaternary",
         [](unsigned N) {
             const std::uint64_t s = std::uint64_t{1} << (2 * N);
             return N + s * (2 * (std::uint64_t{1} << N) - 1) + (s - 1);
         },
         [](const DenseMatrix& g, unsigned) { return decompose_serial_quaternary(g); }},
    };
    csv << "N,path,threads,rep,seed,seconds,mult_count,seconds_stddev\n";
    for (unsigned N = a.n_min; N <= a.n_max; ++N) {
        std::vector<DenseMatrix> mats;
        std::vector<std::uint64_t> seeds;
        for (unsigned r = 0; r < a.reps; ++r) {
            seeds.push_back(matrix_seed(a.seed, N, r));
            mats.push_back(random_matrix(N, seeds.back()));
        }
        std::vector<PauliDecomposition> first(a.reps);
        for (const BenchPath& bp : paths) {
            std::vector<double> secs;
            for (unsigned r = 0; r < a.reps; ++r) {
                const auto t0 = std::chrono::steady_clock::now();
                PauliDecomposition d = bp.run(mats[r], a.threads);
                secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
                if (&bp == &paths[0]) first[r] = std::move(d);
                else if (!(d == first[r]))
                    throw std::runtime_error(std::string("path ") + bp.name + " disagrees with fast at N=" +
                                             std::to_string(N));
                csv << N << ',' << bp.name << ',' << a.threads << ',' << r << ',' << seeds[r] << ','
                    << format_double(secs.back()) << ',' << bp.mults(N) << ",\n";
            }
            double mean = 0.0, var = 0.0;
            for (double x : secs) mean += x / secs.size();
            for (double x : secs) var += (x - mean) * (x - mean);
            const double sd = secs.size() > 1 ? std::sqrt(var / (secs.size() - 1)) : 0.0;
            csv << N << ',' << bp.name << ',' << a.threads << ",-1," << a.seed << ',' << format_double(mean) << ','
                << bp.mults(N) << ',' << format_double(sd) << '\n';
        }
    }
    return 0;
}

int run(const Args& a) {
    if (a.cmd == "bench") {
        if (a.out == "-") return run_bench(a, std::cout);
        std::ofstream f(a.out);
        if (!f) throw FormatError("cannot open \"" + a.out + "\" for writing");
        return run_bench(a, f);
    }
    if (a.cmd == "decompose") {
        const auto t0 = std::chrono::steady_clock::now();
        unsigned N = 0;
        const std::size_t written = decompose_file(a.in, fmt(a), a.out, a.eps,
                                                   a.path == "wht" ? Path::Wht : Path::Gray, &N);
        const auto t1 = std::chrono::steady_clock::now();
        std::cerr << "N=" << N << " nonzero=" << written << " seconds="
                  << format_double(std::chrono::duration<double>(t1 - t0).count()) << '\n';
        return 0;
    }
    if (a.cmd == "recompose") {
        write_matrix(recompose(read_coefficients(a.in)), a.out, fmt(a));
        return 0;
    }
    const DenseMatrix g = read_matrix(a.in, fmt(a));
    const Complex c = coeff_fast(g, string_to_index(a.label, g.num_qubits()));
    std::cout << format_double(c.real()) << ',' << format_double(c.imag()) << '\n';
    return 0;
}

}  // namespace

constexpr const char* kUsage =
    "usage: pdb200 decompose --in PATH [--out PATH] [--format text|binary] [--eps E] [--threads T]\n"
    "                        [--serial] [--path gray|wht]\n"
    "       pdb200 recompose --in CSV [--out PATH] [--format text|binary]\n"
    "       pdb200 coeff LABEL --in PATH [--format text|binary]\n"
    "       pdb200 bench [--n-min N] [--n-max N] [--reps R] [--seed S] [--threads T] [--out PATH]\n";

int main(int argc, char** argv) {
    if (argc == 2 && (std::strcmp(argv[1], "--help") == 0 || std::strcmp(argv[1], "-h") == 0)) {
        std::cout << kUsage;
        return 0;
    }
    try {
        return run(parse(argc, argv));
    } catch (const FormatError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::bad_alloc&) {
        std::cerr << "error: out of memory for this problem size\n";
        return 2;
    } catch (const std::length_error& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << '\n';
        return 2;
    }
}
