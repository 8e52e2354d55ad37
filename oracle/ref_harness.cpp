// ref_harness.cpp — C-ABI shim over the UNMODIFIED reference library
// (proj/src/*.cpp compiled from /root/reference by oracle/Makefile into
// oracle/_ref/libpdref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ to pin the oracle and by
// bench.py's cpu_baseline and --impl reference legs to time the reference's own
// CPU path. Nothing in paper_2401_16378_b200/ links or loads it.
//
// Every entry point forwards to the reference's public C++ API
// (proj/include/paulidecomp/decompose.hpp:33-56, bench.hpp, matrix.hpp) and maps
// its exceptions to status codes: -1 invalid_argument, -2 length_error,
// -4 FormatError, -3 anything else (message in pdref_last_error()).
#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "paulidecomp/bench.hpp"
#include "paulidecomp/decompose.hpp"
#include "paulidecomp/io.hpp"
#include "paulidecomp/matrix.hpp"

using namespace paulidecomp;

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return -1;
    } catch (const std::length_error& e) {
        g_error = e.what();
        return -2;
    } catch (const FormatError& e) {
        g_error = e.what();
        return -4;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -3;
    }
}

void copy_out(const std::vector<Complex>& v, double* out) {
    std::memcpy(out, v.data(), v.size() * sizeof(Complex));
}

}  // namespace

extern "C" {

const char* pdref_last_error() { return g_error.c_str(); }

unsigned pdref_hardware_concurrency() { return std::max(1u, std::thread::hardware_concurrency()); }

void* pdref_matrix_new(unsigned n_qubits, const double* interleaved) {
    DenseMatrix* m = nullptr;
    int rc = guarded([&] {
        m = new DenseMatrix(n_qubits);
        std::memcpy(m->data(), interleaved, m->element_count() * sizeof(Complex));
    });
    return rc == 0 ? m : nullptr;
}

// bench.cpp:48-58 random_matrix, generated straight into the handle
void* pdref_matrix_random(unsigned n_qubits, std::uint64_t seed) {
    DenseMatrix* m = nullptr;
    int rc = guarded([&] { m = new DenseMatrix(random_matrix(n_qubits, seed)); });
    return rc == 0 ? m : nullptr;
}

const double* pdref_matrix_data(void* h) {
    return reinterpret_cast<const double*>(static_cast<DenseMatrix*>(h)->data());
}

void pdref_matrix_free(void* h) { delete static_cast<DenseMatrix*>(h); }

std::uint64_t pdref_matrix_seed(std::uint64_t seed, unsigned n_qubits, unsigned rep) {
    return matrix_seed(seed, n_qubits, rep);
}

int pdref_random_matrix(unsigned n_qubits, std::uint64_t seed, double* out) {
    return guarded([&] { copy_out(random_matrix(n_qubits, seed).elements(), out); });
}

int pdref_decompose_parallel(void* h, unsigned threads, double* out) {
    return guarded([&] {
        copy_out(decompose_parallel(*static_cast<DenseMatrix*>(h), threads).coefficients, out);
    });
}

int pdref_decompose_serial(void* h, double* out) {
    return guarded([&] {
        copy_out(decompose_serial_quaternary(*static_cast<DenseMatrix*>(h)).coefficients, out);
    });
}

int pdref_coeff_fast(void* h, std::uint64_t n, double* out) {
    return guarded([&] {
        const Complex c = coeff_fast(*static_cast<DenseMatrix*>(h), n);
        out[0] = c.real();
        out[1] = c.imag();
    });
}

int pdref_coeff_slow(void* h, std::uint64_t n, double* out) {
    return guarded([&] {
        const Complex c = coeff_slow(*static_cast<DenseMatrix*>(h), n);
        out[0] = c.real();
        out[1] = c.imag();
    });
}

int pdref_oracle_kron(void* h, std::uint64_t n, double* out) {
    return guarded([&] {
        const Complex c = oracle_coeff_kron(*static_cast<DenseMatrix*>(h), n);
        out[0] = c.real();
        out[1] = c.imag();
    });
}

// reference coeff_fast over an explicit list of tensor numbers, split into
// contiguous chunks across `threads` std::threads — the same static split the
// reference's decompose_parallel uses (decompose.cpp:103-126)
int pdref_coeff_batch(void* h, const std::uint64_t* ns, std::uint64_t count, double* out,
                      unsigned threads) {
    return guarded([&] {
        if (threads == 0)
            throw std::invalid_argument("thread count must be at least 1");
        const DenseMatrix& g = *static_cast<DenseMatrix*>(h);
        for (std::uint64_t k = 0; k < count; ++k)
            if (!valid_pauli_index(ns[k], g.num_qubits()))
                throw std::invalid_argument("tensor number out of range");
        const std::uint64_t chunk = std::max<std::uint64_t>(1, (count + threads - 1) / threads);
        auto work = [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k) {
                const Complex c = coeff_fast(g, ns[k]);
                out[2 * k] = c.real();
                out[2 * k + 1] = c.imag();
            }
        };
        std::vector<std::thread> pool;
        for (std::uint64_t b = 0; b < count; b += chunk)
            pool.emplace_back(work, b, std::min(count, b + chunk));
        for (auto& t : pool)
            t.join();
    });
}

int pdref_recompose(unsigned n_qubits, const double* coeffs, double* out) {
    return guarded([&] {
        const std::uint64_t total = pow4(n_qubits);
        std::vector<Complex> c(total);
        std::memcpy(c.data(), coeffs, total * sizeof(Complex));
        const DenseMatrix m = recompose(PauliDecomposition{n_qubits, std::move(c)});
        copy_out(m.elements(), out);
    });
}

// ---- file formats (io.hpp): the reference's own readers/writers ----

int pdref_format_double(double v, char* buf, unsigned cap) {
    const std::string s = format_double(v);
    if (s.size() + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

int pdref_write_matrix_file(void* h, const char* path, int binary) {
    return guarded([&] {
        write_matrix(*static_cast<DenseMatrix*>(h), path, binary ? MatrixFormat::binary : MatrixFormat::text);
    });
}

void* pdref_read_matrix_file(const char* path, int binary) {
    DenseMatrix* m = nullptr;
    int rc = guarded([&] {
        m = new DenseMatrix(read_matrix(path, binary ? MatrixFormat::binary : MatrixFormat::text));
    });
    return rc == 0 ? m : nullptr;
}

unsigned pdref_matrix_qubits(void* h) { return static_cast<DenseMatrix*>(h)->num_qubits(); }

long long pdref_write_coefficients_file(unsigned n_qubits, const double* coeffs, const char* path,
                                        double threshold) {
    long long written = -1;
    int rc = guarded([&] {
        std::vector<Complex> c(pow4(n_qubits));
        std::memcpy(c.data(), coeffs, c.size() * sizeof(Complex));
        written = static_cast<long long>(
            write_coefficients(PauliDecomposition{n_qubits, std::move(c)}, path, threshold));
    });
    return rc == 0 ? written : rc;
}

// reads a coefficient CSV; *n_qubits receives N, out (capacity cap entries) the 4^N values
int pdref_read_coefficients_file(const char* path, unsigned* n_qubits, double* out, unsigned long long cap) {
    return guarded([&] {
        const PauliDecomposition d = read_coefficients(path);
        *n_qubits = d.num_qubits;
        if (d.coefficients.size() <= cap)
            std::memcpy(out, d.coefficients.data(), d.coefficients.size() * sizeof(Complex));
    });
}

}  // extern "C"
