// Reference-exact binary16 GEMM with tcgen05-generated rounded products
// (gemm_f16x.cu). Same operand / epilogue contract as gemm_f16ref
// (gemm_f16ref.cuh), bit-identical results; additionally A must be finite and
// args.zfix must point at f16x_zfix_words(M, N) + 2 zeroed words, args.hash_a
// at M and args.hash_b at N unsigned 64-bit words.
#pragma once

#include "gemm_f16ref.cuh"

namespace kp {
long f16x_zfix_words(int M, int N);
// Row sign hashes of a K-major operand (see gemm_f16x.cu); precompute
// args.hash_a once for a fixed A and set args.hash_a_ready.
void f16x_row_hash(const F16Operand& X, int rows, int K, unsigned long long* out);
unsigned long long f16x_hash_sum(int K);
int gemm_f16x_num_ctas(int M, int N);  // = output tiles (one partial slot each)
int gemm_f16x_partials_per_image(int M, int n_img);  // batched products (F16Epilogue::part_img)
void gemm_f16x(const F16GemmArgs& a, int kernel_class);
}  // namespace kp
