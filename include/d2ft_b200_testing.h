/* d2ft_b200 self-test hooks (not part of the reference-facing boundary).
 * They run the library's tcgen05 GEMM core on the three operand shapes the
 * D2FT step uses, so tests can check the kernel against a plain fp32
 * reference in isolation.  Host buffers in, host buffers out; bf16 passed as
 * raw uint16 bit patterns. */
#ifndef D2FT_B200_TESTING_H
#define D2FT_B200_TESTING_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* D[m][n] = sum_k A[m][k] B[n][k]; bn selects the tile width (160, 208, 256; -208 / -160 = CTA pair with multicast B). */
int d2ft_test_gemm_dense(const uint16_t* A, const uint16_t* B, int M, int N, int K, int bn, float* D);
/* MN-major B: D[m][n] = sum_k A[m][k] BT[k][n] (BT row-major K x N); bn 208 / 64, negative = CTA pair. */
int d2ft_test_gemm_mn(const uint16_t* A, const uint16_t* BT, int M, int N, int K, int bn, float* D);
/* Both MN-major: D[m][n] = sum_k AT[k][m] BT[k][n] (CTA pair, BN 208). */
int d2ft_test_gemm_mn_ab(const uint16_t* AT, const uint16_t* BT, int M, int N, int K, float* D);
/* Tokens as N: D[p][m][t] = sum_k A[m][k] X[p][t][k] for t < T (T-row planes). */
int d2ft_test_gemm_planes(const uint16_t* A, const uint16_t* X, int M, int T, int K, int P, float* D);
/* Tokens as K: D[m][n] = sum_p sum_{t<T} XT[p][m][t] YT[p][n][t]; pitch TP >= T. */
int d2ft_test_gemm_tokenk(const uint16_t* XT, const uint16_t* YT, int M, int N, int T, int TP, int P, float* D);
/* ms per launch of a dense M x N x K GEMM (BN = 256), CUDA-event timed. */
int d2ft_test_gemm_bench_pair(int M, int K, int variant, int iters, double* ms_per);
int d2ft_test_gemm_bench(int M, int N, int K, int iters, double* ms_per);

#ifdef __cplusplus
}
#endif
#endif
