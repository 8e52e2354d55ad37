// paulidecomp.cpp — the reference's C++ API (include/paulidecomp_b200/decompose.hpp) over the
// C ABI of include/pd_api.h. Host logic only: validation, exception mapping, label algebra.
// All arithmetic on matrices and coefficients happens in the CUDA kernels.
#include "paulidecomp_b200/bench.hpp"
#include "paulidecomp_b200/decompose.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <bit>
#include <memory>
#include <thread>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <utility>

#include "pd_api.h"

namespace paulidecomp {

namespace {

// pd_status -> the reference's exception types (decompose.cpp:14-19, matrix.cpp:10-19)
void raise(int rc) {
    if (rc == PD_OK) return;  // no message string on the success path (fixed memory)
    const std::string msg = pd_last_error();
    switch (rc) {
        case PD_OK: return;
        case PD_EINVAL: throw std::invalid_argument(msg);
        case PD_ELENGTH: throw std::length_error(msg);
        case PD_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

// one lazily created context per device; calls on a context are serialised
struct Device {
    std::mutex mu;
    pd_ctx* ctx = nullptr;
};

std::mutex g_devices_mu;
std::unordered_map<int, std::unique_ptr<Device>> g_devices;
thread_local int t_device = 0;

struct Lease {
    std::unique_lock<std::mutex> lock;
    pd_ctx* ctx;
};

Lease lease() {
    Device* d;
    {
        std::lock_guard<std::mutex> g(g_devices_mu);
        auto& slot = g_devices[t_device];
        if (!slot) slot = std::make_unique<Device>();
        d = slot.get();
    }
    std::unique_lock<std::mutex> lock(d->mu);
    if (!d->ctx) raise(pd_ctx_create(t_device, &d->ctx));
    return Lease{std::move(lock), d->ctx};
}

const double* as_doubles(const Complex* p) { return reinterpret_cast<const double*>(p); }
double* as_doubles(Complex* p) { return reinterpret_cast<double*>(p); }

void check_qubit_count(unsigned num_qubits) {  // matrix.cpp:10-19
    if (num_qubits == 0) throw std::invalid_argument("a matrix needs at least one qubit (2x2)");
    if (num_qubits > kMaxQubits)
        throw std::invalid_argument("qubit count " + std::to_string(num_qubits) +
                                    " exceeds the word-size bound of 32");
    if (num_qubits >= 32)
        throw std::length_error("dense storage for 32 qubits exceeds the address space");
}

void check_index(unsigned num_qubits, std::uint64_t n) {  // decompose.cpp:14-19
    if (num_qubits < 32 && n >= (std::uint64_t{1} << (2 * num_qubits)))
        throw std::invalid_argument("tensor number " + std::to_string(n) + " out of range for " +
                                    std::to_string(num_qubits) + " qubits");
}

// closed-form multiplication counts of the reference kernels (proj/README.md:113-120)
std::uint64_t fast_mults(unsigned N) { return N + 2 * (std::uint64_t{1} << N) - 1; }

}  // namespace

namespace {

// The reference API returns its coefficients (and matrices) by value in value-initialised
// std::vectors. Its
// zero fill first-touches 4 GiB at N=14 on one thread (~1.3 s of page faults and zeroing, four
// times the GPU call); the pages are populated on helper threads first (MADV_HUGEPAGE where the
// box runs THP in madvise mode, then MADV_POPULATE_WRITE: allocated and zeroed by the kernel),
// so the fill that follows runs over resident pages.
std::vector<Complex> result_vector(std::uint64_t n) {
    std::vector<Complex> v;
    const std::uint64_t bytes = n * sizeof(Complex);
    if (bytes >= (std::uint64_t{64} << 20)) {
        v.reserve(n);
        const uintptr_t page = 4096, huge = uintptr_t{2} << 20;
        const uintptr_t lo = reinterpret_cast<uintptr_t>(v.data()), hi = lo + bytes;
        const uintptr_t hlo = (lo + huge - 1) & ~(huge - 1), hhi = hi & ~(huge - 1);
        if (hhi > hlo) madvise(reinterpret_cast<void*>(hlo), hhi - hlo, MADV_HUGEPAGE);
#ifdef MADV_POPULATE_WRITE
        const uintptr_t b = (lo + page - 1) & ~(page - 1), e = hi & ~(page - 1);
        std::atomic<uintptr_t> next{b};
        std::vector<std::thread> pool;
        for (int k = 0; k < 8; ++k)
            pool.emplace_back([&] {
                constexpr uintptr_t kPiece = uintptr_t{32} << 20;
                for (uintptr_t at; (at = next.fetch_add(kPiece)) < e;)
                    if (madvise(reinterpret_cast<void*>(at), std::min(kPiece, e - at), MADV_POPULATE_WRITE)) return;
            });
        for (auto& t : pool) t.join();
#endif
    }
    v.resize(n);
    return v;
}

}  // namespace

// ---------------- DenseMatrix (matrix.hpp:14-43 semantics) ----------------

DenseMatrix::DenseMatrix(unsigned num_qubits) : num_qubits_(num_qubits) {
    check_qubit_count(num_qubits);
    elements_ = result_vector(std::uint64_t{1} << (2 * num_qubits));
}

DenseMatrix::DenseMatrix(unsigned num_qubits, std::vector<Complex> elements)
    : num_qubits_(num_qubits), elements_(std::move(elements)) {
    check_qubit_count(num_qubits);
    const std::uint64_t want = std::uint64_t{1} << (2 * num_qubits);
    if (elements_.size() != want)
        throw std::invalid_argument("element buffer holds " + std::to_string(elements_.size()) +
                                    " entries, expected " + std::to_string(want));
}

DenseMatrix DenseMatrix::identity(unsigned num_qubits) {
    DenseMatrix m(num_qubits);
    for (std::uint64_t i = 0; i < m.dim(); ++i) m(i, i) = Complex{1.0, 0.0};
    return m;
}

// ---------------- views ----------------

void set_device(int device) { t_device = device; }

unsigned qubits_for_dim(std::uint64_t rows, std::uint64_t cols) {  // module.cpp:24-30
    if (rows != cols || rows < 2 || !std::has_single_bit(rows))
        throw std::invalid_argument("matrix must be square with power-of-two dimension >= 2");
    return static_cast<unsigned>(std::countr_zero(rows));
}

void decompose_into(const Complex* g, unsigned num_qubits, Complex* out, Path path) {
    check_qubit_count(num_qubits);
    Lease l = lease();
    raise(pd_decompose(l.ctx, num_qubits, as_doubles(g), as_doubles(out),
                       static_cast<pd_path>(static_cast<int>(path))));
}

void decompose_into(const Complex* g, unsigned num_qubits, Complex* out, Path path,
                    const std::vector<int>& devices) {
    check_qubit_count(num_qubits);
    if (devices.empty()) {
        decompose_into(g, num_qubits, out, path);
        return;
    }
    // one multi-device context per device list, serialised like the single-device ones
    static std::mutex mu;
    static std::map<std::vector<int>, std::unique_ptr<Device>> contexts;
    Device* d;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = contexts[devices];
        if (!slot) slot = std::make_unique<Device>();
        d = slot.get();
    }
    std::lock_guard<std::mutex> lk(d->mu);
    if (!d->ctx)
        raise(pd_ctx_create_multi(devices.data(), static_cast<int>(devices.size()), &d->ctx));
    raise(pd_decompose(d->ctx, num_qubits, as_doubles(g), as_doubles(out),
                       static_cast<pd_path>(static_cast<int>(path))));
}

void coeff_batch_into(const Complex* g, unsigned num_qubits, const std::uint64_t* ns,
                      std::uint64_t count, Complex* out) {
    check_qubit_count(num_qubits);
    for (std::uint64_t k = 0; k < count; ++k) check_index(num_qubits, ns[k]);
    Lease l = lease();
    raise(pd_coeff_batch(l.ctx, num_qubits, as_doubles(g), ns, count, as_doubles(out)));
}

Complex coeff_view(const Complex* g, unsigned num_qubits, std::uint64_t n, bool slow) {
    check_qubit_count(num_qubits);
    check_index(num_qubits, n);
    double out[2];
    Lease l = lease();
    raise(pd_coeff(l.ctx, num_qubits, as_doubles(g), n, slow ? 1 : 0, out));
    return Complex{out[0], out[1]};
}

Complex oracle_coeff_view(const Complex* g, unsigned num_qubits, std::uint64_t n) {
    check_qubit_count(num_qubits);
    check_index(num_qubits, n);
    if (num_qubits > kOracleMaxQubits)
        throw std::invalid_argument("reference path is capped at " +
                                    std::to_string(kOracleMaxQubits) + " qubits");
    double out[2];
    Lease l = lease();
    raise(pd_oracle_coeff(l.ctx, num_qubits, as_doubles(g), n, out));
    return Complex{out[0], out[1]};
}

// ---------------- reference API ----------------

Complex coeff_fast(const DenseMatrix& g, std::uint64_t n) {
    return coeff_view(g.data(), g.num_qubits(), n, false);
}

Complex coeff_fast(const DenseMatrix& g, std::uint64_t n, MultCount& count) {
    const Complex c = coeff_fast(g, n);
    count.mults += fast_mults(g.num_qubits());
    return c;
}

Complex coeff_slow(const DenseMatrix& g, std::uint64_t n) {
    return coeff_view(g.data(), g.num_qubits(), n, true);
}

Complex coeff_slow(const DenseMatrix& g, std::uint64_t n, MultCount& count) {
    const Complex c = coeff_slow(g, n);
    count.mults += (g.num_qubits() + 1) * g.dim();
    return c;
}

Complex oracle_coeff_kron(const DenseMatrix& g, std::uint64_t n) {
    return oracle_coeff_view(g.data(), g.num_qubits(), n);
}

// bench.cpp:42-46: the per-(N, rep) seed is one splitmix64 output of the mixed master seed
std::uint64_t matrix_seed(std::uint64_t seed, unsigned num_qubits, unsigned rep) {
    std::uint64_t z = (seed ^ (std::uint64_t{num_qubits} * 0xD6E8FEB86659FD93ull) ^
                       (std::uint64_t{rep} * 0xCA5A826395121157ull)) + 0x9E3779B97F4A7C15ull;
    for (const auto& [shift, mul] : {std::pair{30, 0xBF58476D1CE4E5B9ull}, std::pair{27, 0x94D049BB133111EBull}})
        z = (z ^ (z >> shift)) * mul;
    return z ^ (z >> 31);
}

void random_matrix_into(unsigned num_qubits, std::uint64_t seed, Complex* out) {
    check_qubit_count(num_qubits);
    Lease l = lease();
    raise(pd_random_matrix(l.ctx, num_qubits, seed, as_doubles(out)));
}

DenseMatrix random_matrix(unsigned num_qubits, std::uint64_t seed) {  // bench.cpp:48-58, on the GPU
    DenseMatrix m(num_qubits);
    Lease l = lease();
    raise(pd_random_matrix(l.ctx, num_qubits, seed, as_doubles(m.data())));
    return m;
}

PauliDecomposition decompose(const DenseMatrix& g, Path path) {
    PauliDecomposition d{g.num_qubits(), result_vector(g.element_count())};
    decompose_into(g.data(), g.num_qubits(), d.coefficients.data(), path);
    return d;
}

PauliDecomposition decompose_parallel(const DenseMatrix& g, unsigned threads) {
    if (threads == 0) throw std::invalid_argument("thread count must be at least 1");
    return decompose(g, Path::Gray);
}

PauliDecomposition decompose_parallel(const DenseMatrix& g, unsigned threads, MultCount& count) {
    PauliDecomposition d = decompose_parallel(g, threads);
    count.mults += g.element_count() * fast_mults(g.num_qubits());
    return d;
}

PauliDecomposition decompose_serial_quaternary(const DenseMatrix& g) {
    // same coefficients (the reference's quaternary walk is bit-identical to its parallel one)
    return decompose(g, Path::Gray);
}

PauliDecomposition decompose_serial_quaternary(const DenseMatrix& g, MultCount& count) {
    PauliDecomposition d = decompose_serial_quaternary(g);
    const std::uint64_t strings = g.element_count();
    count.mults += g.num_qubits() + strings * (2 * g.dim() - 1) + (strings - 1);
    return d;
}

std::vector<Complex> coeff_batch(const DenseMatrix& g, const std::vector<std::uint64_t>& ns) {
    std::vector<Complex> out(ns.size());
    coeff_batch_into(g.data(), g.num_qubits(), ns.data(), ns.size(), out.data());
    return out;
}

void recompose_into(const Complex* c, unsigned num_qubits, Complex* g_out) {
    check_qubit_count(num_qubits);
    Lease l = lease();
    raise(pd_recompose(l.ctx, num_qubits, as_doubles(c), as_doubles(g_out)));
}

DenseMatrix recompose(const PauliDecomposition& d) {  // decompose.cpp:221-230 validation
    if (d.num_qubits == 0 || d.num_qubits > kMaxQubits)
        throw std::invalid_argument("qubit count must be in [1, 32]");
    if (d.num_qubits == kMaxQubits)
        throw std::length_error("a dense matrix for N=32 exceeds the address space");
    const std::uint64_t want = std::uint64_t{1} << (2 * d.num_qubits);
    if (d.coefficients.size() != want)
        throw std::invalid_argument("coefficient array holds " +
                                    std::to_string(d.coefficients.size()) + " entries, expected " +
                                    std::to_string(want));
    DenseMatrix out(d.num_qubits);
    Lease l = lease();
    raise(pd_recompose(l.ctx, d.num_qubits, as_doubles(d.coefficients.data()), as_doubles(out.data())));
    return out;
}

// ---------------- labels and bit utilities (pauli_string.cpp:25-54, bits.hpp, pauli.hpp) ----

std::uint64_t string_to_index(std::string_view label, unsigned num_qubits) {
    if (num_qubits == 0 || num_qubits > kMaxQubits)
        throw FormatError("operator count must be in [1, 32], got " + std::to_string(num_qubits));
    if (label.size() != num_qubits)
        throw FormatError("label \"" + std::string(label) + "\" has " +
                          std::to_string(label.size()) + " characters, expected " +
                          std::to_string(num_qubits));
    std::uint64_t n = 0;
    for (unsigned t = 0; t < num_qubits; ++t) {  // digit 0 is the rightmost character
        unsigned code;
        switch (label[num_qubits - 1 - t]) {
            case 'I': code = 0; break;
            case 'X': code = 1; break;
            case 'Y': code = 2; break;
            case 'Z': code = 3; break;
            default:
                throw FormatError("label \"" + std::string(label) +
                                  "\" contains a character outside IXYZ");
        }
        n |= std::uint64_t{code} << (2 * t);
    }
    return n;
}

std::string index_to_string(std::uint64_t n, unsigned num_qubits) {
    if (num_qubits == 0 || num_qubits > kMaxQubits)
        throw std::invalid_argument("operator count must be in [1, 32]");
    check_index(num_qubits, n);
    static constexpr char kOps[4] = {'I', 'X', 'Y', 'Z'};
    std::string label(num_qubits, 'I');
    for (unsigned t = 0; t < num_qubits; ++t) label[num_qubits - 1 - t] = kOps[(n >> (2 * t)) & 3u];
    return label;
}

std::uint64_t xy_mask(std::uint64_t n, unsigned num_qubits) {
    std::uint64_t mask = 0;
    for (unsigned t = 0; t < num_qubits && t < kMaxQubits; ++t) {
        const unsigned d = (n >> (2 * t)) & 3u;
        mask |= std::uint64_t{(d ^ (d >> 1)) & 1u} << t;
    }
    return mask;
}

std::uint64_t gray_code(std::uint64_t k) { return k ^ (k >> 1); }

unsigned flipped_bit_index(std::uint64_t k) { return static_cast<unsigned>(std::countr_zero(k + 1)); }

}  // namespace paulidecomp
