// pd_kernels.h — host launchers of the kernels in pd_kernels.cu / pd_wht.cu (namespace pdb).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "pd_device.cuh"

namespace pdb {

constexpr unsigned kMaxRunBits = 8;  // run bits of the RUNS output layout (shards x sub-blocks)

extern std::atomic<uint64_t> g_launches;

// K1: diag[(x - x0) * 2^N + i] = G[i ^ x][i], x in [x0, x0 + x_count)
cudaError_t launch_diag_gather(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                               double2* diag, cudaStream_t stream);

// K1 restricted to the columns [col0, col0 + cols) (a power-of-two aligned range)
cudaError_t launch_diag_gather_cols(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                    uint64_t col0, uint64_t cols, double2* diag, cudaStream_t stream);
// dst[dst_off[k] + j] = src[src_off[k] + j] for j < run_len, k < count (offsets in elements)
cudaError_t launch_copy_runs(const double2* src, double2* dst, uint64_t run_len,
                             const uint64_t* src_off, const uint64_t* dst_off, uint64_t count,
                             cudaStream_t stream);

// Non-finite elements (pd_nonfinite.cu). After a fast kernel has stored the coefficients of the
// X-masks [x0, x0 + x_count) through `map`, every X-mask whose Z-mask-0 coefficient (the plain
// sum of its diagonal) is not finite gets all its coefficients recomputed with the reference's
// complex products. src: the gathered diagonals (row x - x0), or G itself when from_matrix.
// With `flags` (x_count words) the X-masks are the flagged ones instead (nonfinite_scan).
cudaError_t launch_nonfinite_fixup(const double2* src, bool from_matrix, unsigned N, uint64_t x0,
                                   uint64_t x_count, const OutMap& map, const unsigned* flags,
                                   cudaStream_t stream);
// flags[x - x0] = 1 if D_x (row x - x0 of diag) holds a non-finite element, else 0
cudaError_t launch_nonfinite_scan(const double2* diag, unsigned N, uint64_t x_count, unsigned* flags,
                                  cudaStream_t stream);
// stream-ordered scratch from the library's own memory pool (not the device's default pool)
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t stream);
cudaError_t pool_free(void* p, cudaStream_t stream);

// K2 over the walk chunks [c_begin, c_end) (c_end = 0: to the end), continuing from raw sums
// part_in (null: from zero) and storing raw sums to part_out (null: finished coefficients)
cudaError_t launch_gray_segment(const double2* diag, unsigned N, uint64_t x0, uint64_t x_count,
                                unsigned c_begin, unsigned c_end, const double2* part_in,
                                double2* part_out, unsigned run_bits, double2* out, int layout,
                                cudaStream_t stream, unsigned chunk_log = 0);
unsigned gray_xmask_chunks(unsigned N);  // walk chunks per diagonal (1 for N < 12)
// fewest X-masks per Gray launch for which K2s-c (N >= 13) is used: each of its 16 compile-time
// bodies must span more CTAs than the GPU holds at once (smaller launches take K2s)
uint64_t gray_share_c_min_xmasks(unsigned N);

// K2: Gray-code sums for the X-masks [x0, x0 + x_count); output layout as in pd_api.h
cudaError_t launch_gray_xmask(const double2* diag, unsigned N, uint64_t x0, uint64_t x_count,
                              unsigned run_bits, double2* out, int layout, cudaStream_t stream);
uint64_t gray_xmask_grid(unsigned N, uint64_t x_count);

// K3b: batched strings bucketed by X-mask, one CTA per X-mask over its staged diagonal
// (bit-identical to K3); used by launch_walk when strings_grouped_ok
bool strings_grouped_ok(unsigned N, uint64_t count);
cudaError_t launch_strings_grouped(const double2* G, unsigned N, const uint64_t* ns,
                                   uint64_t count, double2* out, cudaStream_t stream);

// K4: fast Walsh-Hadamard path over the same diagonals (separately reported)
cudaError_t launch_wht_xmask(const double2* diag, unsigned N, uint64_t x0, uint64_t x_count,
                             unsigned run_bits, double2* out, int layout, cudaStream_t stream);

// K4 fused two-pass WHT straight from G for X-masks [x0, x0 + x_count) (N in [8,16],
// x_count >= 32); scratch holds x_count * 2^N complex128 (the half-transformed diagonals)
bool wht_fused_ok(unsigned N, uint64_t x_count);
cudaError_t launch_wht_from_matrix(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                   double2* scratch, unsigned run_bits, double2* out, int layout,
                                   cudaStream_t stream);

// in-place unnormalised Walsh-Hadamard transform of x_count rows of 2^N (N <= 16)
// recompose through the chunked inverse WHT passes (N in [11, 15]); scratch >= 4^N / 4 elements
bool wht_inverse_ok(unsigned N);
cudaError_t launch_wht_inverse(const double2* coeffs, unsigned N, double2* scratch, double2* G,
                               cudaStream_t stream);
cudaError_t launch_wht_inplace(double2* rows, unsigned N, uint64_t x_count, cudaStream_t stream);

// recompose (decompose.cpp:221-250) on the device:
//   gather   E[x][z] = (-i)^{|x&z|} c[n(x,z)]
//   (WHT in place over z)
//   scatter  G[row][col] = E[row ^ col][row]
cudaError_t launch_recompose_gather(const double2* coeffs, unsigned N, double2* rows,
                                    cudaStream_t stream);
cudaError_t launch_recompose_scatter(const double2* rows, unsigned N, double2* G,
                                     cudaStream_t stream);

// K0/K3: one thread per tensor number (ns == nullptr: n = 0..count-1)
// K3 over compact diagonals: string k walks D + slot[k] 2^N (its X-mask's gathered diagonal)
cudaError_t launch_walk_slots(const double2* D, unsigned N, const uint64_t* ns, const uint32_t* slot,
                              uint64_t count, double2* out, cudaStream_t stream);
// K3 for one string over its gathered diagonal D[i] = G[i ^ x][i] (2^N entries)
cudaError_t launch_walk_diag(const double2* D, unsigned N, const uint64_t* n, bool slow, double2* out,
                             cudaStream_t stream);
cudaError_t launch_walk(const double2* G, unsigned N, const uint64_t* ns, uint64_t count, bool slow,
                        double2* out, cudaStream_t stream);

cudaError_t launch_kron_trace(const double2* G, unsigned N, uint64_t n, double2* out,
                              cudaStream_t stream);

// file-path helpers (pd_io.cu)
cudaError_t launch_first_nonfinite(const double2* v, uint64_t count, unsigned long long* result,
                                   cudaStream_t stream);
uint64_t select_tiles(uint64_t count);
cudaError_t launch_select(const double2* c, uint64_t count, double threshold, unsigned* tile_counts,
                          unsigned long long* tile_offsets, uint64_t* idx_out, double2* val_out,
                          cudaStream_t stream);

cudaError_t launch_random_matrix(unsigned N, uint64_t seed, double2* out, cudaStream_t stream);

cudaError_t launch_fp64_probe(unsigned blocks, unsigned iters, double* sink, cudaStream_t stream);

}  // namespace pdb
