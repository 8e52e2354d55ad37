// paulidecomp_b200/decompose.hpp — the reference's C++ decomposition API, served by B200 kernels.
//
// Drop-in for the declarations of proj/include/paulidecomp/{matrix,decompose,pauli_string}.hpp
// (namespace, type and function names, argument meaning and exception contract kept):
//   DenseMatrix / PauliDecomposition  matrix.hpp:14-51
//   coeff_fast / coeff_slow / oracle_coeff_kron   decompose.hpp:33-37
//   decompose_parallel / decompose_serial_quaternary   decompose.hpp:46-56
//   recompose   decompose.hpp:59
//   string_to_index / index_to_string / FormatError   pauli_string.hpp, io.hpp
// Every compute function runs on the GPU through the C ABI of include/pd_api.h; there is
// no CPU path (a missing or non-sm_100 device raises std::runtime_error).
//
// Differences a caller can observe:
//   * `threads` keeps its validation (0 -> std::invalid_argument, decompose.cpp:98-99) but
//     does not choose the parallelism: the GPU launch does.
//   * MultCount overloads add the reference's closed-form multiplication counts
//     (proj/README.md:113-120); the kernels themselves use no multiplications.
//   * results are bit-identical to the reference for finite inputs on the Gray path
//     (same per-coefficient summation order), except possibly the sign of an exact zero.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace paulidecomp {

using Complex = std::complex<double>;

inline constexpr unsigned kMaxQubits = 32;       // bits.hpp:15
inline constexpr unsigned kOracleMaxQubits = 6;  // decompose.hpp:11

// malformed operator labels (io.hpp FormatError; registered as ValueError in Python)
class FormatError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

// row-major 2^N x 2^N complex matrix; element (row j, column i) at offset j*2^N + i
class DenseMatrix {
  public:
    explicit DenseMatrix(unsigned num_qubits);
    DenseMatrix(unsigned num_qubits, std::vector<Complex> elements);
    static DenseMatrix identity(unsigned num_qubits);

    unsigned num_qubits() const { return num_qubits_; }
    std::uint64_t dim() const { return std::uint64_t{1} << num_qubits_; }
    std::uint64_t element_count() const { return std::uint64_t{1} << (2 * num_qubits_); }

    Complex& operator()(std::uint64_t row, std::uint64_t col) { return elements_[row * dim() + col]; }
    Complex operator()(std::uint64_t row, std::uint64_t col) const {
        return elements_[row * dim() + col];
    }
    const Complex* data() const { return elements_.data(); }
    Complex* data() { return elements_.data(); }
    const std::vector<Complex>& elements() const { return elements_; }
    bool operator==(const DenseMatrix&) const = default;

  private:
    unsigned num_qubits_;
    std::vector<Complex> elements_;
};

struct PauliDecomposition {
    unsigned num_qubits = 0;
    std::vector<Complex> coefficients;
    bool operator==(const PauliDecomposition&) const = default;
};

struct MultCount {
    std::uint64_t mults = 0;
};

// which device algorithm serves a full decomposition
enum class Path : int {
    Gray = 0,   // K1 gather + K2 Gray-code FP64 sums: the paper's O(8^N) method (default)
    Wht = 1,    // K1 gather + K4 fast Walsh-Hadamard (separately reported second path)
    Naive = 2,  // K0: one thread per coefficient, reference walk straight from G
};

// ---- reference API (decompose.hpp:33-59) ----
Complex coeff_fast(const DenseMatrix& g, std::uint64_t n);
Complex coeff_fast(const DenseMatrix& g, std::uint64_t n, MultCount& count);
Complex coeff_slow(const DenseMatrix& g, std::uint64_t n);
Complex coeff_slow(const DenseMatrix& g, std::uint64_t n, MultCount& count);
Complex oracle_coeff_kron(const DenseMatrix& g, std::uint64_t n);

PauliDecomposition decompose_parallel(const DenseMatrix& g, unsigned threads = 1);
PauliDecomposition decompose_parallel(const DenseMatrix& g, unsigned threads, MultCount& count);
PauliDecomposition decompose_serial_quaternary(const DenseMatrix& g);
PauliDecomposition decompose_serial_quaternary(const DenseMatrix& g, MultCount& count);

DenseMatrix recompose(const PauliDecomposition& d);

// ---- bits.hpp / pauli.hpp helpers (bits.hpp:17-26, pauli.hpp:16-20) ----
constexpr std::uint64_t pow2(unsigned exponent) { return std::uint64_t{1} << exponent; }
constexpr std::uint64_t pow4(unsigned exponent) { return std::uint64_t{1} << (2 * exponent); }
enum class PauliOp : unsigned { I = 0, X = 1, Y = 2, Z = 3 };
// operator at position t of tensor number n (base-4 digit t, digit 0 rightmost in labels)
constexpr PauliOp pauli_digit(std::uint64_t n, unsigned t) {
    return static_cast<PauliOp>((n >> (2 * t)) & 3u);
}

// ---- pauli_string.hpp (label <-> tensor number) ----
std::uint64_t string_to_index(std::string_view label, unsigned num_qubits);
std::string index_to_string(std::uint64_t n, unsigned num_qubits);
std::uint64_t xy_mask(std::uint64_t n, unsigned num_qubits);
std::uint64_t gray_code(std::uint64_t k);
unsigned flipped_bit_index(std::uint64_t k);

// ---- B200 additions: zero-copy views and batched strings ----

// all 4^N coefficients of the row-major matrix at g into out (4^N entries)
void decompose_into(const Complex* g, unsigned num_qubits, Complex* out, Path path = Path::Gray);
// the same over several GPUs of this host (pd_ctx_create_multi: X-masks split across the
// devices, each uploading only the 1/P of G it needs); a device may be listed more than once
void decompose_into(const Complex* g, unsigned num_qubits, Complex* out, Path path,
                    const std::vector<int>& devices);
PauliDecomposition decompose(const DenseMatrix& g, Path path = Path::Gray);

// the matrix of the 4^N coefficients at c into g_out (2^N x 2^N, row-major): recompose without
// the by-value containers
void recompose_into(const Complex* c, unsigned num_qubits, Complex* g_out);

// out[k] = c_{ns[k]}
void coeff_batch_into(const Complex* g, unsigned num_qubits, const std::uint64_t* ns,
                      std::uint64_t count, Complex* out);
std::vector<Complex> coeff_batch(const DenseMatrix& g, const std::vector<std::uint64_t>& ns);

Complex coeff_view(const Complex* g, unsigned num_qubits, std::uint64_t n, bool slow);
Complex oracle_coeff_view(const Complex* g, unsigned num_qubits, std::uint64_t n);

// validated qubit count of a square power-of-two dimension (module.cpp:23-33 rules)
unsigned qubits_for_dim(std::uint64_t rows, std::uint64_t cols);

// select the GPU used by this thread's subsequent calls (default 0)
void set_device(int device);

}  // namespace paulidecomp
