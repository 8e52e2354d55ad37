// cli.cpp — `pdb200`, the reference CLI's compute subcommands (proj/tools/main.cpp) on the GPU:
//
//   pdb200 decompose --in PATH [--out PATH] [--format text|binary] [--eps E] [--threads T]
//                    [--serial] [--path gray|wht]
//   pdb200 recompose --in CSV [--out PATH] [--format text|binary]
//   pdb200 coeff LABEL --in PATH [--format text|binary]
//
// Paths may be "-" (stdin/stdout). Exit codes follow main.cpp:140-158: 0 success, 1 usage or
// format error, 2 resource or internal error. `decompose` prints "N=… nonzero=… seconds=…" to
// stderr like main.cpp:42-43 (seconds = read + GPU decomposition + selection + write).
#include <chrono>
#include <fstream>
#include <cstring>
#include <iostream>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "paulidecomp_b200/decompose.hpp"
#include "paulidecomp_b200/io.hpp"

using namespace paulidecomp;

namespace {

struct Args {
    std::string cmd, in = "-", out = "-", format = "text", label, path = "gray";
    double eps = 0.0;
    unsigned threads = 1;
    bool serial = false, have_in = false;
};

[[noreturn]] void usage(const std::string& why) { throw std::invalid_argument(why); }

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) usage("a subcommand is required: decompose, recompose or coeff");
    a.cmd = argv[1];
    if (a.cmd != "decompose" && a.cmd != "recompose" && a.cmd != "coeff")
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
    if (!a.have_in) usage("--in is required");
    if (a.cmd == "coeff" && a.label.empty()) usage("coeff needs an operator label");
    return a;
}

MatrixFormat fmt(const Args& a) { return a.format == "binary" ? MatrixFormat::binary : MatrixFormat::text; }

int run(const Args& a) {
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
    "       pdb200 coeff LABEL --in PATH [--format text|binary]\n";

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
