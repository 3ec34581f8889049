// bfa_kernels.hpp -- host launchers of the ahead-of-time kernels (bfa_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bfa_k {
// table: n_rows rows of 2^(n-6) u64 words each (n >= 7)
cudaError_t fill_generators(int n, int n_rows, uint64_t* table, cudaStream_t st);
// d = LOP3(a, b, c; imm) over n_words64 u64 words (even)
cudaError_t vec_lut3(uint64_t* d, const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t n_words64,
                     uint32_t imm, cudaStream_t st);
// *count = popcount(v[0..n_words))
cudaError_t popcount(const uint64_t* v, uint64_t n_words, uint64_t* count, cudaStream_t st);
// constant-memory interpreter (engine=1 ablation); synchronous on st
cudaError_t interp(const uint32_t* ops, int n_ops, const uint32_t* consts, int n_consts, int n_slots,
                   uint32_t out_op, int out_neg, uint64_t w_begin, uint64_t w_count, uint32_t mask, uint32_t* out,
                   uint64_t* count, cudaStream_t st, int* block_used);
// ordered compaction: append the set bits of vec[0..n_words) whose index
// (relative to the vector) lies in [lo, hi) as valuations base + index, in
// ascending order, at positions *running.. of mu_out (< cap written);
// *running (device) += their number.  No atomics, no sort.
cudaError_t compact_models(const uint64_t* vec, uint64_t n_words, uint64_t lo, uint64_t hi, uint64_t base,
                           uint64_t* mu_out, uint64_t cap, uint64_t* running, cudaStream_t st);
// out.txt rows: row r = the letters of deposit(mu[r], free_ids) | fixed_values,
// id n_all-1 first, as '0'/'1', then '\n' (n_all + 1 bytes per row)
cudaError_t rows(const uint64_t* mu, uint64_t count, int n_free, const int* free_ids, int n_all,
                 uint64_t fixed_values, char* out, cudaStream_t st);
// *dst += *src on the device
cudaError_t add_u64(uint64_t* dst, const uint64_t* src, cudaStream_t st);
// op 0: lop3.b32, 1: mad.lo.u32, 2: both 1:1 -- 256 ops per thread per iteration
cudaError_t peak_int(int op, int blocks, int threads, int iters, uint32_t* sink, cudaStream_t st);
}  // namespace bfa_k
