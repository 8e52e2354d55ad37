// module.cpp — pybind11 module `_paulidecomp`: the reference's Python surface
// (proj/bindings/module.cpp:87-121, same function names, arguments and exception mapping)
// served by the B200 kernels, plus device-pointer entry points for the sharding layer
// and the benchmark (submodule `device`).
//
// Unlike the reference binding (which copies the numpy buffer into a std::vector,
// module.cpp:31, and copies results back, :37,42), C-contiguous complex128 inputs are
// read in place and results are written straight into the returned array.
#include <pybind11/complex.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "paulidecomp_b200/bench.hpp"
#include "paulidecomp_b200/decompose.hpp"
#include "paulidecomp_b200/io.hpp"
#include "pd_api.h"

namespace py = pybind11;
using namespace paulidecomp;

namespace {

using ComplexArray = py::array_t<Complex, py::array::c_style | py::array::forcecast>;

unsigned matrix_qubits(const ComplexArray& a) {
    if (a.ndim() != 2) throw std::invalid_argument("matrix must be a 2-d array");
    return qubits_for_dim(static_cast<std::uint64_t>(a.shape(0)),
                          static_cast<std::uint64_t>(a.shape(1)));
}

// A fresh result array. Above 64 MiB it is its own mapping with transparent huge pages
// requested (MADV_HUGEPAGE; the box runs THP in "madvise" mode): the GPU path writes every byte
// of it from the staging threads (csrc/pd_stage.cu), and first-touching 4 GiB in 4 KiB pages
// cost more than the whole decomposition (N=14: 605 ms per call against 370 ms into an array
// that was already touched).
py::array_t<Complex> new_result(py::ssize_t count) {
    if (count < 0 || static_cast<size_t>(count) > (size_t{1} << 58)) throw std::bad_alloc();
    const size_t bytes = static_cast<size_t>(count) * sizeof(Complex);
    constexpr size_t kHuge = size_t{2} << 20;
    static const char* thp = std::getenv("PD_RESULT_THP");  // "0": a plain numpy array (A/B)
    if (bytes < (size_t{64} << 20) || (thp && thp[0] == '0')) return py::array_t<Complex>(count);
    const size_t span = ((bytes + kHuge - 1) & ~(kHuge - 1)) + kHuge;
    void* base = mmap(nullptr, span, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (base == MAP_FAILED) return py::array_t<Complex>(count);
    char* data = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~(kHuge - 1));
    madvise(data, span - static_cast<size_t>(data - static_cast<char*>(base)), MADV_HUGEPAGE);
    struct Mapping {
        void* base;
        size_t span;
    };
    auto* m = new Mapping{base, span};
    py::capsule owner(m, [](void* q) {
        auto* mm = static_cast<Mapping*>(q);
        munmap(mm->base, mm->span);
        delete mm;
    });
    return py::array_t<Complex>({count}, {static_cast<py::ssize_t>(sizeof(Complex))},
                                reinterpret_cast<Complex*>(data), owner);
}

// Populates (allocates and zeroes, content untouched) the pages of a fresh result array on
// helper threads while the decomposition runs: MADV_POPULATE_WRITE leaves pages that are
// already present alone, so it cannot race with the staging threads' writes. Without it the
// first touch of 4 GiB happened inside the staging scatter, behind the GPU.
class Prefault {
public:
    Prefault(void* data, size_t bytes, unsigned threads) {
#ifdef MADV_POPULATE_WRITE
        constexpr uintptr_t kPage = 4096;
        const uintptr_t b = (reinterpret_cast<uintptr_t>(data) + kPage - 1) & ~(kPage - 1);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(data) + bytes) & ~(kPage - 1);
        if (e <= b) return;
        begin_ = b;
        end_ = e;
        for (unsigned k = 0; k < threads; ++k)
            pool_.emplace_back([this] {
                constexpr uintptr_t kPiece = uintptr_t{32} << 20;
                for (;;) {
                    const uintptr_t at = begin_ + next_.fetch_add(kPiece);
                    if (at >= end_) return;
                    const uintptr_t len = std::min(kPiece, end_ - at);
                    if (madvise(reinterpret_cast<void*>(at), len, MADV_POPULATE_WRITE) != 0) return;
                }
            });
#else
        (void)data, (void)bytes, (void)threads;
#endif
    }
    ~Prefault() {
        for (auto& t : pool_) t.join();
    }

private:
    uintptr_t begin_ = 0, end_ = 0;
    std::atomic<uintptr_t> next_{0};
    std::vector<std::thread> pool_;
};

// index of the first element with a non-finite part, UINT64_MAX if none (8 threads over slices;
// the smallest hit wins, so the row/column reported is the first in row-major order)
std::uint64_t first_nonfinite(const Complex* v, std::uint64_t n) {
    const unsigned parts = n >= (std::uint64_t{1} << 20) ? 8u : 1u;
    std::vector<std::uint64_t> hit(parts, UINT64_MAX);
    auto scan = [&](unsigned k) {
        const std::uint64_t b = n * k / parts, e = n * (k + 1) / parts;
        for (std::uint64_t i = b; i < e; ++i)
            if (!std::isfinite(v[i].real()) || !std::isfinite(v[i].imag())) {
                hit[k] = i;
                return;
            }
    };
    std::vector<std::thread> pool;
    for (unsigned k = 1; k < parts; ++k) pool.emplace_back(scan, k);
    scan(0);
    for (auto& t : pool) t.join();
    return *std::min_element(hit.begin(), hit.end());
}

Path parse_path(const std::string& s) {
    if (s == "gray") return Path::Gray;
    if (s == "wht") return Path::Wht;
    if (s == "naive") return Path::Naive;
    throw std::invalid_argument("path must be 'gray', 'wht' or 'naive'");
}

py::array_t<Complex> py_decompose(const ComplexArray& g, unsigned threads, bool serial,
                                  const std::string& path, py::object out, py::object devices) {
    const unsigned N = matrix_qubits(g);
    // the serial quaternary driver ignores `threads`; the parallel one rejects 0
    // (module.cpp:56-60 -> decompose.cpp:98-99, 133-152); both yield the same coefficients
    if (!serial && threads == 0) throw std::invalid_argument("thread count must be at least 1");
    const Path p = parse_path(path);
    const py::ssize_t count = static_cast<py::ssize_t>(1) << (2 * N);
    py::array_t<Complex> result;
    if (out.is_none()) {
        result = new_result(count);
    } else {
        result = py::array_t<Complex>::ensure(out);
        if (!result || result.ndim() != 1 || result.shape(0) != count ||
            !(result.flags() & py::array::c_style) || !result.writeable() ||
            result.ptr() != out.ptr())
            throw std::invalid_argument("out must be a writable C-contiguous complex128 array of 4**N");
    }
    const Complex* src = g.data();
    Complex* dst = result.mutable_data();
    std::vector<int> devs;
    if (!devices.is_none()) devs = devices.cast<std::vector<int>>();
    {
        py::gil_scoped_release nogil;
        static const char* pf_env = std::getenv("PD_RESULT_PREFAULT");  // threads; "0" = off
        const unsigned pf = pf_env ? static_cast<unsigned>(std::atoi(pf_env)) : 2u;  // 2-12 threads measured: 2 best (profiles/r02_pageable_probe.txt)
        const size_t nbytes = static_cast<size_t>(count) * sizeof(Complex);
        std::unique_ptr<Prefault> prefault;
        if (out.is_none() && pf && nbytes >= (size_t{64} << 20))
            prefault = std::make_unique<Prefault>(dst, nbytes, pf);
        if (!devs.empty()) decompose_into(src, N, dst, p, devs);
        else decompose_into(src, N, dst, p);
    }
    return result;
}

py::array_t<Complex> py_recompose(const ComplexArray& c) {  // module.cpp:45-54 validation
    if (c.ndim() != 1) throw std::invalid_argument("coefficients must be a 1-d array");
    const auto count = static_cast<std::uint64_t>(c.shape(0));
    if (count < 4 || !std::has_single_bit(count) || (std::countr_zero(count) & 1))
        throw std::invalid_argument("coefficient count must be a power of four >= 4");
    const unsigned N = static_cast<unsigned>(std::countr_zero(count) / 2);
    if (N >= kMaxQubits) throw std::length_error("a dense matrix for N=32 exceeds the address space");
    // the coefficients are read in place and the matrix is written straight into the returned
    // array (the reference binding copies both ways, module.cpp:45-54)
    py::array_t<Complex> result = new_result(static_cast<py::ssize_t>(count));
    const Complex* src = c.data();
    Complex* dst = result.mutable_data();
    {
        py::gil_scoped_release nogil;
        std::unique_ptr<Prefault> prefault;
        if (count * sizeof(Complex) >= (size_t{64} << 20)) prefault = std::make_unique<Prefault>(dst, count * sizeof(Complex), 2);
        recompose_into(src, N, dst);
    }
    const auto dim = static_cast<py::ssize_t>(std::uint64_t{1} << N);
    return result.reshape({dim, dim});
}

Complex py_coefficient_index(const ComplexArray& g, std::uint64_t n, bool slow) {
    const unsigned N = matrix_qubits(g);
    py::gil_scoped_release nogil;
    return coeff_view(g.data(), N, n, slow);
}

Complex py_coefficient_label(const ComplexArray& g, const std::string& label, bool slow) {
    const unsigned N = matrix_qubits(g);
    return py_coefficient_index(g, string_to_index(label, N), slow);
}

Complex py_oracle_index(const ComplexArray& g, std::uint64_t n) {
    const unsigned N = matrix_qubits(g);
    py::gil_scoped_release nogil;
    return oracle_coeff_view(g.data(), N, n);
}

Complex py_oracle_label(const ComplexArray& g, const std::string& label) {
    const unsigned N = matrix_qubits(g);
    return py_oracle_index(g, string_to_index(label, N));
}

py::array_t<Complex> py_coefficients(const ComplexArray& g,
                                     py::array_t<std::uint64_t, py::array::c_style | py::array::forcecast> ns) {
    const unsigned N = matrix_qubits(g);
    if (ns.ndim() != 1) throw std::invalid_argument("ns must be a 1-d array of tensor numbers");
    py::array_t<Complex> out(ns.shape(0));
    const std::uint64_t count = static_cast<std::uint64_t>(ns.shape(0));
    const std::uint64_t* np = ns.data();
    Complex* dst = out.mutable_data();
    {
        py::gil_scoped_release nogil;
        coeff_batch_into(g.data(), N, np, count, dst);
    }
    return out;
}

// ---- device-pointer entry points (pointers are ints, e.g. torch.Tensor.data_ptr()) ----

void check(int rc) {
    if (rc == PD_OK) return;
    const std::string msg = pd_last_error();
    if (rc == PD_EINVAL) throw std::invalid_argument(msg);
    if (rc == PD_ELENGTH) throw std::length_error(msg);
    if (rc == PD_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

template <class T>
T* P(std::uintptr_t p) {
    return reinterpret_cast<T*>(p);
}

pd_path path_of(const std::string& s) { return static_cast<pd_path>(static_cast<int>(parse_path(s))); }

}  // namespace

PYBIND11_MODULE(_paulidecomp, m) {
    m.doc() = "Pauli-string decomposition of dense complex matrices on B200 (sm_100a)";

    py::register_exception<FormatError>(m, "FormatError", PyExc_ValueError);

    m.def("decompose", &py_decompose, py::arg("matrix"), py::arg("threads") = 1,
          py::arg("serial") = false, py::arg("path") = "gray", py::arg("out") = py::none(),
          py::arg("devices") = py::none(),
          "All 4**N expansion coefficients of a 2**N x 2**N matrix, indexed by tensor number. "
          "devices=[d0, d1, ...] (a power-of-two count) splits the X-masks over those GPUs.");
    m.def("recompose", &py_recompose, py::arg("coefficients"),
          "Rebuild the dense matrix from its full coefficient vector.");
    m.def("coefficient", &py_coefficient_index, py::arg("matrix"), py::arg("n"),
          py::arg("slow") = false, "One expansion coefficient by tensor number.");
    m.def("coefficient", &py_coefficient_label, py::arg("matrix"), py::arg("label"),
          py::arg("slow") = false, "One expansion coefficient by operator label, e.g. \"IXZY\".");
    m.def("oracle_coefficient", &py_oracle_index, py::arg("matrix"), py::arg("n"),
          "Brute-force Kronecker-product trace for one coefficient (N <= 6).");
    m.def("oracle_coefficient", &py_oracle_label, py::arg("matrix"), py::arg("label"));
    m.def("coefficients", &py_coefficients, py::arg("matrix"), py::arg("ns"),
          "Coefficients for an array of tensor numbers (batched single-string path).");

    m.def("gray_code", &gray_code, py::arg("k"));
    m.def("flipped_bit_index", &flipped_bit_index, py::arg("k"),
          "Index of the bit that changes between gray_code(k) and gray_code(k + 1).");
    m.def("xy_mask", &xy_mask, py::arg("n"), py::arg("num_qubits"),
          "Bitmask with bit t set when operator t of tensor n is X or Y.");
    m.def("label_to_index", &string_to_index, py::arg("label"), py::arg("num_qubits"));
    m.def("index_to_label", &index_to_string, py::arg("n"), py::arg("num_qubits"));
    m.def("set_device", &set_device, py::arg("device"),
          "GPU used by this thread's subsequent host-buffer calls.");
    m.def("launch_count", &pd_launch_count, "Kernels launched by libpd_b200 in this process.");
    m.def("fp64_add_probe", [](int device) {
        pd_ctx* ctx = nullptr;
        check(pd_ctx_create(device, &ctx));
        double r = 0.0;
        int rc = pd_fp64_add_probe(ctx, &r);
        pd_ctx_destroy(ctx);
        check(rc);
        return r;
    }, py::arg("device") = 0, "Achieved DADD/s of a pure FP64-add kernel on all SMs.");
    m.attr("__version__") = "0.1.0+b200";

    // file formats (proj/docs/formats.md), io.hpp
    auto mfmt = [](const std::string& f) {
        if (f == "text") return MatrixFormat::text;
        if (f == "binary") return MatrixFormat::binary;
        throw std::invalid_argument("format must be 'text' or 'binary'");
    };
    m.def("format_double", &format_double, py::arg("value"),
          "Shortest round-trip decimal text, '.0' appended to integral values.");
    m.def("read_matrix", [mfmt](const std::string& path, const std::string& format) {
        if (mfmt(format) == MatrixFormat::binary && path != "-") {
            // PDMAT-V1 payload straight into the returned array, finiteness checked on threads
            const unsigned N = read_matrix_binary_header(path);
            const py::ssize_t count = static_cast<py::ssize_t>(1) << (2 * N);
            py::array_t<Complex> a = new_result(count);
            Complex* dst = a.mutable_data();
            std::uint64_t first_bad = UINT64_MAX;
            {
                py::gil_scoped_release nogil;
                {
                    std::unique_ptr<Prefault> prefault;
                    if (count * sizeof(Complex) >= (size_t{64} << 20))
                        prefault = std::make_unique<Prefault>(dst, count * sizeof(Complex), 2);
                    read_matrix_binary_into(path, dst, static_cast<std::uint64_t>(count));
                }
                first_bad = first_nonfinite(dst, static_cast<std::uint64_t>(count));
            }
            if (first_bad != UINT64_MAX)
                throw FormatError("non-finite value at row " + std::to_string(first_bad >> N) + ", column " +
                                  std::to_string(first_bad & ((std::uint64_t{1} << N) - 1)));
            const py::ssize_t d = static_cast<py::ssize_t>(1) << N;
            return py::array_t<Complex>(a.reshape({d, d}));
        }
        DenseMatrix g = read_matrix(path, mfmt(format));
        const auto d = static_cast<py::ssize_t>(g.dim());
        return py::array_t<Complex>({d, d}, g.data());
    }, py::arg("path"), py::arg("format") = "text");
    m.def("write_matrix", [mfmt](const ComplexArray& a, const std::string& path, const std::string& format) {
        const unsigned N = matrix_qubits(a);
        const Complex* g = a.data();
        const MatrixFormat f = mfmt(format);
        py::gil_scoped_release nogil;
        write_matrix_view(g, N, path, f);
    }, py::arg("matrix"), py::arg("path"), py::arg("format") = "text");
    m.def("read_coefficients", [](const std::string& path) {
        PauliDecomposition d = read_coefficients(path);
        return py::array_t<Complex>(static_cast<py::ssize_t>(d.coefficients.size()), d.coefficients.data());
    }, py::arg("path"));
    m.def("write_coefficients", [](const ComplexArray& c, const std::string& path, double threshold) {
        if (c.ndim() != 1) throw std::invalid_argument("coefficients must be a 1-d array");
        const auto count = static_cast<std::uint64_t>(c.shape(0));
        if (count < 4 || !std::has_single_bit(count) || (std::countr_zero(count) & 1))
            throw std::invalid_argument("coefficient count must be a power of four >= 4");
        PauliDecomposition d{static_cast<unsigned>(std::countr_zero(count) / 2),
                             std::vector<Complex>(c.data(), c.data() + count)};
        py::gil_scoped_release nogil;
        return write_coefficients(d, path, threshold);
    }, py::arg("coefficients"), py::arg("path"), py::arg("threshold") = 0.0,
          "Write the coefficient CSV; returns the number of records.");
    m.def("decompose_file", [mfmt](const std::string& in, const std::string& out, const std::string& format,
                                   double threshold, const std::string& path) {
        const MatrixFormat f = mfmt(format);
        const Path p = parse_path(path);
        py::gil_scoped_release nogil;
        return decompose_file(in, f, out, threshold, p);
    }, py::arg("in_path"), py::arg("out_path"), py::arg("format") = "binary", py::arg("threshold") = 0.0,
          py::arg("path") = "gray",
          "Matrix file -> GPU decomposition -> threshold selection on the GPU -> coefficient CSV.");

    m.def("matrix_seed", &matrix_seed, py::arg("seed"), py::arg("num_qubits"), py::arg("rep"),
          "The reference benchmark's per-(N, rep) generator seed (bench.cpp:42-46).");
    m.def("random_matrix", [](unsigned N, std::uint64_t seed) {
        if (N == 0 || N >= kMaxQubits) {
            DenseMatrix probe(N);  // the reference's errors (matrix.cpp:10-19)
        }
        // generated on the device straight into the returned array (no DenseMatrix round trip)
        const py::ssize_t count = static_cast<py::ssize_t>(1) << (2 * N);
        py::array_t<Complex> a = new_result(count);
        Complex* dst = a.mutable_data();
        {
            py::gil_scoped_release nogil;
            std::unique_ptr<Prefault> prefault;
            if (count * sizeof(Complex) >= (size_t{64} << 20)) prefault = std::make_unique<Prefault>(dst, count * sizeof(Complex), 2);
            random_matrix_into(N, seed, dst);
        }
        const py::ssize_t dim = static_cast<py::ssize_t>(1) << N;
        return a.reshape({dim, dim});
    }, py::arg("num_qubits"), py::arg("seed"),
          "random_matrix(N, seed) of the reference benchmark (bench.cpp:48-58), generated on the GPU.");
    py::module_ d = m.def_submodule("device", "Stream-ordered entry points on device pointers");
    d.def("scratch_bytes", [](unsigned N, std::uint64_t x_count, const std::string& path) {
        return pd_scratch_bytes(N, x_count, path_of(path));
    }, py::arg("num_qubits"), py::arg("x_count"), py::arg("path") = "gray");
    d.def("run_offset", &pd_run_offset, py::arg("num_qubits"), py::arg("run_bits"),
          py::arg("shard"), py::arg("run"));
    d.def("decompose", [](unsigned N, std::uintptr_t g, std::uintptr_t out, std::uintptr_t scratch,
                          const std::string& path, std::uintptr_t stream) {
        check(pd_decompose_device(N, P<const double>(g), P<double>(out), P<void>(scratch),
                                  path_of(path), P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("g"), py::arg("out"), py::arg("scratch"),
          py::arg("path") = "gray", py::arg("stream") = 0);
    d.def("decompose_blocked", [](unsigned N, std::uintptr_t g, std::uintptr_t out,
                                  std::uintptr_t scratch, std::uint64_t scratch_bytes,
                                  const std::string& path, std::uintptr_t stream) {
        check(pd_decompose_device_blocked(N, P<const double>(g), P<double>(out), P<void>(scratch),
                                          scratch_bytes, path_of(path), P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("g"), py::arg("out"), py::arg("scratch"),
          py::arg("scratch_bytes"), py::arg("path") = "gray", py::arg("stream") = 0,
          "Full decomposition with a bounded scratch buffer (X-mask blocks).");
    d.def("diag_gather", [](unsigned N, std::uintptr_t g, std::uint64_t x0, std::uint64_t x_count,
                            std::uintptr_t diag, std::uintptr_t stream) {
        check(pd_diag_gather_device(N, P<const double>(g), x0, x_count, P<double>(diag),
                                    P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("g"), py::arg("x0"), py::arg("x_count"), py::arg("diag"),
          py::arg("stream") = 0);
    auto layout_of = [](const std::string& l) {
        if (l == "global") return PD_LAYOUT_GLOBAL;
        if (l == "runs") return PD_LAYOUT_RUNS;
        throw std::invalid_argument("layout must be 'global' or 'runs'");
    };
    d.def("xmask_coeffs", [layout_of](unsigned N, std::uintptr_t diag, std::uint64_t x0,
                                      std::uint64_t x_count, unsigned run_bits, std::uintptr_t out,
                                      const std::string& layout, const std::string& path,
                                      std::uintptr_t stream) {
        check(pd_xmask_coeffs_device(N, P<const double>(diag), x0, x_count, run_bits, P<double>(out),
                                     layout_of(layout), path_of(path), P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("diag"), py::arg("x0"), py::arg("x_count"),
          py::arg("run_bits"), py::arg("out"), py::arg("layout") = "global", py::arg("path") = "gray",
          py::arg("stream") = 0);
    d.def("shard_coeffs", [layout_of](unsigned N, std::uintptr_t g, std::uint64_t x0,
                                      std::uint64_t x_count, unsigned run_bits, std::uintptr_t out,
                                      const std::string& layout, std::uintptr_t scratch,
                                      const std::string& path, std::uintptr_t stream) {
        check(pd_shard_coeffs_device(N, P<const double>(g), x0, x_count, run_bits, P<double>(out),
                                     layout_of(layout), P<void>(scratch), path_of(path),
                                     P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("g"), py::arg("x0"), py::arg("x_count"), py::arg("run_bits"),
          py::arg("out"), py::arg("layout") = "global", py::arg("scratch") = 0,
          py::arg("path") = "gray", py::arg("stream") = 0,
          "All coefficients of an X-mask range straight from G (one shard's work).");
    d.def("copy_runs", [](std::uintptr_t src, std::uintptr_t dst, std::uint64_t run_len,
                          std::uintptr_t src_off, std::uintptr_t dst_off, std::uint64_t count,
                          std::uintptr_t stream) {
        check(pd_copy_runs_device(P<const double>(src), P<double>(dst), run_len,
                                  P<const std::uint64_t>(src_off), P<const std::uint64_t>(dst_off),
                                  count, P<void>(stream)));
    }, py::arg("src"), py::arg("dst"), py::arg("run_len"), py::arg("src_off"), py::arg("dst_off"),
          py::arg("count"), py::arg("stream") = 0);
    d.def("ipc_export", [](std::uintptr_t ptr) {
        pd_ipc_handle h{};
        check(pd_ipc_export(P<const void>(ptr), &h));
        return py::make_tuple(py::bytes(reinterpret_cast<const char*>(h.bytes), sizeof(h.bytes)),
                              h.offset);
    }, py::arg("ptr"), "CUDA IPC export of the allocation holding ptr: (handle bytes, offset).");
    d.def("ipc_open", [](const py::bytes& handle, std::uint64_t offset) {
        pd_ipc_handle h{};
        const std::string b = handle;
        if (b.size() != sizeof(h.bytes)) throw std::invalid_argument("IPC handle must be 64 bytes");
        std::memcpy(h.bytes, b.data(), sizeof(h.bytes));
        h.offset = offset;
        void* p = nullptr;
        check(pd_ipc_open(&h, &p));
        return reinterpret_cast<std::uintptr_t>(p);
    }, py::arg("handle"), py::arg("offset"), "Map a peer's exported buffer; returns a device pointer.");
    d.def("ipc_close", [](std::uintptr_t ptr) { check(pd_ipc_close(P<void>(ptr))); }, py::arg("ptr"));
    d.def("coeff_batch", [](unsigned N, std::uintptr_t g, std::uintptr_t ns, std::uint64_t count,
                            bool slow, std::uintptr_t out, std::uintptr_t stream) {
        check(pd_coeff_batch_device(N, P<const double>(g), P<const std::uint64_t>(ns), count,
                                    slow ? 1 : 0, P<double>(out), P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("g"), py::arg("ns"), py::arg("count"), py::arg("slow"),
          py::arg("out"), py::arg("stream") = 0);
    d.def("random_matrix", [](unsigned N, std::uint64_t seed, std::uintptr_t g, std::uintptr_t stream) {
        check(pd_random_matrix_device(N, seed, P<double>(g), P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("seed"), py::arg("g"), py::arg("stream") = 0);
    d.def("recompose", [](unsigned N, std::uintptr_t coeffs, std::uintptr_t g, std::uintptr_t scratch,
                          std::uintptr_t stream) {
        check(pd_recompose_device(N, P<const double>(coeffs), P<double>(g), P<void>(scratch),
                                  P<void>(stream)));
    }, py::arg("num_qubits"), py::arg("coeffs"), py::arg("g"), py::arg("scratch"),
          py::arg("stream") = 0);
}
