// paulidecomp_b200/io.hpp — the reference's file formats (proj/docs/formats.md,
// proj/include/paulidecomp/io.hpp) feeding the B200 path.
//
//   * binary matrix PDMAT-V1 (8-byte magic, uint64-LE N, row-major float64-LE (re, im)) —
//     read straight into a caller-provided (e.g. pinned) buffer; finiteness is checked on the
//     GPU after upload (pd_first_nonfinite_device) when the matrix is decomposed there;
//   * text matrix "PAULIDECOMP-MAT v1 N=<N>" (and the headerless square layout on read);
//   * coefficient CSV "# PAULIDECOMP-COEF v1 N=<N>" / "pauli,re,im", ascending tensor number,
//     records with |c| > threshold (threshold 0 keeps all) — the kept indices are selected on
//     the GPU (pd_select_coeffs_device), the text is formatted on host threads with the
//     reference's shortest-round-trip rule (format_double).
// Errors follow the reference: FormatError for malformed data, std::invalid_argument for a
// negative threshold, std::length_error for N = 32.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "paulidecomp_b200/decompose.hpp"

namespace paulidecomp {

enum class MatrixFormat { text, binary };

// shortest float text that round-trips, ".0" appended to integral values (io.cpp:130-137)
std::string format_double(double value);

// ---- matrices ----
DenseMatrix read_matrix(const std::string& path, MatrixFormat format);
void write_matrix(const DenseMatrix& matrix, const std::string& path, MatrixFormat format);
// view form: the row-major 2^N x 2^N matrix at g (no DenseMatrix copy)
void write_matrix_view(const Complex* g, unsigned num_qubits, const std::string& path, MatrixFormat format);
DenseMatrix read_matrix_text(std::istream& in);
DenseMatrix read_matrix_binary(std::istream& in);
void write_matrix_text(const DenseMatrix& matrix, std::ostream& out);
void write_matrix_binary(const DenseMatrix& matrix, std::ostream& out);

// PDMAT-V1 header of a file: the qubit count (validated magic, N range and exact size)
unsigned read_matrix_binary_header(const std::string& path);
// read the payload of a PDMAT-V1 file into dst (16 * 4^N bytes, e.g. pinned host memory)
// without the finiteness scan (the GPU path checks the device copy instead); returns N
unsigned read_matrix_binary_into(const std::string& path, Complex* dst, std::uint64_t capacity);

// ---- coefficients ----
std::size_t write_coefficients(const PauliDecomposition& d, const std::string& path,
                               double threshold = 0.0);
std::size_t write_coefficients(const PauliDecomposition& d, std::ostream& out,
                               double threshold = 0.0);
// view form: coefficients of num_qubits at c (4^N entries)
std::size_t write_coefficients_view(const Complex* c, unsigned num_qubits, std::ostream& out,
                                    double threshold = 0.0);
PauliDecomposition read_coefficients(const std::string& path);
PauliDecomposition read_coefficients(std::istream& in);

// records (n, c_n) already selected, ascending n: the CSV body of write_coefficients
std::size_t write_coefficient_records(unsigned num_qubits, const std::uint64_t* idx,
                                      const Complex* vals, std::uint64_t count, double threshold,
                                      std::ostream& out);

// ---- end-to-end file path (the CLI's decompose) ----
// read a matrix file, decompose on the GPU, write the coefficient CSV; returns records written
std::size_t decompose_file(const std::string& in_path, MatrixFormat format,
                           const std::string& out_path, double threshold = 0.0,
                           Path path = Path::Gray, unsigned* num_qubits = nullptr);

}  // namespace paulidecomp
