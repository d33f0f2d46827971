// GEMM self-test hooks (include/d2ft_b200_testing.h): the library's tcgen05
// GEMM core on the operand shapes the D2FT step uses, host buffers in and
// out, so tests/test_gemm_gpu.py checks the kernel against a plain fp32
// reference in isolation.  Test infrastructure: built into
// libd2ft_b200_testing.so, linked against the product library.
#include <cuda.h>

#include <mutex>
#include <vector>

#include "../../../include/d2ft_b200_testing.h"
#include "../common.cuh"
#include "../gemm_sm100.cuh"

namespace d2ft_b200 {

namespace {

// D[m][n] = sum_k A[m][k] B[n][k]; A, B 2-D row-major bf16 (K contiguous).
template <int BN>
struct DenseProb {
  int M, N, K;
  float* D;
  struct Tile {
    int nkb, mt, nt;
  };
  struct Row {};
  __device__ int ntn() const { return (N + BN - 1) / BN; }
  __device__ int ntiles() const { return ((M + 127) / 128) * ntn(); }
  __device__ void tile(int t, int, Tile& c) const {
    c.mt = t / ntn();
    c.nt = t % ntn();
    c.nkb = (K + 63) / 64;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, 0, kb * 64, c.nt * BN, 0};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int m = c.mt * 128 + row;
    if (m >= M) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c.nt * BN + col0 + i;
      if (n < N) D[(size_t)m * N + n] = v[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// Tokens as N: D[p][m][t] = sum_k A[m][k] X[p][t][k], t < T (box of BN rows, OOB zero).
template <int BN>
struct PlanesProb {
  int M, T, K, P;
  float* D;
  struct Tile {
    int nkb, mt, p;
  };
  struct Row {};
  __device__ int ntiles() const { return ((M + 127) / 128) * P; }
  __device__ void tile(int t, int, Tile& c) const {
    c.p = t / ((M + 127) / 128);
    c.mt = t % ((M + 127) / 128);
    c.nkb = (K + 63) / 64;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, 0, kb * 64, 0, c.p};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int m = c.mt * 128 + row;
    if (m >= M) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int t = col0 + i;
      if (t < T) D[((size_t)c.p * M + m) * T + t] = v[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// K = tokens of P planes: D[m][n] = sum_p sum_t XT[p][m][t] YT[p][n][t]
// (token-innermost buffers with pitch TP; the tensor maps stop at T, so the
// 64-token block that straddles T reads zeros).
template <int BN>
struct TokenKProb {
  int M, N, T, P;
  float* D;
  struct Tile {
    int nkb, mt, nt;
  };
  struct Row {};
  __device__ int ntn() const { return (N + BN - 1) / BN; }
  __device__ int ntiles() const { return ((M + 127) / 128) * ntn(); }
  __device__ void tile(int t, int, Tile& c) const {
    c.mt = t / ntn();
    c.nt = t % ntn();
    c.nkb = P * ((T + 63) / 64);
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    const int tb = (T + 63) / 64;
    const int p = kb / tb, t0 = (kb % tb) * 64;
    return KCoord{t0, c.mt * 128, c.mt * 128 + 64, p, t0, c.nt * BN, p};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    const int m = c.mt * 128 + row;
    if (m >= M) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c.nt * BN + col0 + i;
      if (n < N) D[(size_t)m * N + n] = v[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// CTA-pair variant of DenseProb: the two CTAs of a cluster take m-tiles 2p and
// 2p+1 of the same n-tile and share (multicast) its B rows.
template <int BN>
struct DensePairProb {
  int M, N, K;
  float* D;
  struct Tile {
    int nkb, mt, nt;
  };
  struct Row {};
  __device__ int ntn() const { return (N + BN - 1) / BN; }
  __device__ int ntiles() const { return (((M + 127) / 128 + 1) / 2) * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.mt = 2 * (t / ntn()) + rank;
    c.nt = t % ntn();
    c.nkb = (K + 63) / 64;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, 0, kb * 64, c.nt * BN, 0};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    if (!D) return;  // throughput runs: accumulator drained, nothing stored
    const int m = c.mt * 128 + row;
    if (m >= M) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c.nt * BN + col0 + i;
      if (n < N) D[(size_t)m * N + n] = v[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

// MN-major B: D[m][n] = sum_k A[m][k] BT[k][n]; BT row-major [K][N] (N contiguous).
template <int BN>
struct DenseMNProb {
  int M, N, K, pair;
  float* D;
  struct Tile {
    int nkb, mt, nt;
  };
  struct Row {};
  __device__ int ntn() const { return (N + BN - 1) / BN; }
  __device__ int mts() const { return pair ? (((M + 127) / 128 + 1) / 2) : (M + 127) / 128; }
  __device__ int ntiles() const { return mts() * ntn(); }
  __device__ void tile(int t, int rank, Tile& c) const {
    c.mt = pair ? 2 * (t / ntn()) + rank : t / ntn();
    c.nt = t % ntn();
    c.nkb = (K + 63) / 64;
  }
  __device__ KCoord kcoord(const Tile& c, int kb) const {
    return KCoord{kb * 64, c.mt * 128, c.mt * 128 + 64, 0, c.nt * BN, kb * 64, 0};
  }
  __device__ void row_begin(const Tile&, int, Row&) const {}
  __device__ void chunk(const Tile& c, int row, int col0, const float (&v)[16], Row&) const {
    if (!D) return;
    const int m = c.mt * 128 + row;
    if (m >= M) return;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c.nt * BN + col0 + i;
      if (n < N) D[(size_t)m * N + n] = v[i];
    }
  }
  __device__ void row_end(const Tile&, int, int, Row&) const {}
};

template <typename T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) { D2FT_CUDA(cudaMalloc(&p, n * sizeof(T) + 256)); }
  ~Dev() { cudaFree(p); }
};

}  // namespace
}  // namespace d2ft_b200

using namespace d2ft_b200;

extern "C" {

int d2ft_test_gemm_dense(const uint16_t* A, const uint16_t* B, int M, int N, int K, int bn, float* D) {
  return guarded([&] {
    D2FT_REQUIRE(K % 8 == 0, kInput, "K must be a multiple of 8");
    Dev<uint16_t> dA((size_t)M * K), dB((size_t)N * K);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemcpy(dA.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(dB.p, B, (size_t)N * K * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemset(dD.p, 0, (size_t)M * N * 4));
    if (bn == -2208) {  // CTA pair, pair UMMA (cta_group::2, B split)
      using S = GemmShape<208, 6, 1, 4, 2, 0, 0, 1>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 104);
      launch_gemm<DensePairProb<208>, S>(a, b, DensePairProb<208>{M, N, K, dD.p}, 0, nullptr);
    } else if (bn == -208) {  // CTA pair, B multicast
      using S = GemmShape<208, 5, 1, 4, 2>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 104);
      launch_gemm<DensePairProb<208>, S>(a, b, DensePairProb<208>{M, N, K, dD.p}, 0, nullptr);
    } else if (bn == -160) {
      using S = GemmShape<160, 6, 1, 4, 2>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 80);
      launch_gemm<DensePairProb<160>, S>(a, b, DensePairProb<160>{M, N, K, dD.p}, 0, nullptr);
    } else if (bn == 256) {
      using S = GemmShape<256, 4, 1>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 256);
      launch_gemm<DenseProb<256>, S>(a, b, DenseProb<256>{M, N, K, dD.p}, 0, nullptr);
    } else if (bn == 208) {
      using S = GemmShape<208, 5, 1>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 208);
      launch_gemm<DenseProb<208>, S>(a, b, DenseProb<208>{M, N, K, dD.p}, 0, nullptr);
    } else {
      using S = GemmShape<160, 6, 1>;
      CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
      CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 160);
      launch_gemm<DenseProb<160>, S>(a, b, DenseProb<160>{M, N, K, dD.p}, 0, nullptr);
    }
    D2FT_CUDA(cudaDeviceSynchronize());
    D2FT_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

int d2ft_test_gemm_mn(const uint16_t* A, const uint16_t* BT, int M, int N, int K, int bn, float* D) {
  return guarded([&] {
    D2FT_REQUIRE(K % 8 == 0 && N % 8 == 0, kInput, "K and N must be multiples of 8");
    Dev<uint16_t> dA((size_t)M * K), dB((size_t)K * N);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemcpy(dA.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(dB.p, BT, (size_t)K * N * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemset(dD.p, 0, (size_t)M * N * 4));
    CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dB.p, N, K, 1, (uint64_t)N * 2, (uint64_t)K * N * 2, 64);
    if (bn == -2208) {  // pair UMMA, MN-major B split across the pair
      launch_gemm<DenseMNProb<208>, GemmShape<208, 6, 1, 4, 2, 1, 0, 1>>(a, b, DenseMNProb<208>{M, N, K, 1, dD.p}, 0,
                                                                          nullptr);
    } else if (bn == -208) {
      launch_gemm<DenseMNProb<208>, GemmShape<208, 4, 1, 4, 2, 1>>(a, b, DenseMNProb<208>{M, N, K, 1, dD.p}, 0,
                                                                    nullptr);
    } else if (bn == 64) {
      launch_gemm<DenseMNProb<64>, GemmShape<64, 8, 1, 4, 1, 1>>(a, b, DenseMNProb<64>{M, N, K, 0, dD.p}, 0, nullptr);
    } else if (bn == -64) {
      launch_gemm<DenseMNProb<64>, GemmShape<64, 8, 1, 4, 2, 1>>(a, b, DenseMNProb<64>{M, N, K, 1, dD.p}, 0, nullptr);
    } else {
      launch_gemm<DenseMNProb<208>, GemmShape<208, 4, 1, 4, 1, 1>>(a, b, DenseMNProb<208>{M, N, K, 0, dD.p}, 0,
                                                                    nullptr);
    }
    D2FT_CUDA(cudaDeviceSynchronize());
    D2FT_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

int d2ft_test_gemm_mn_ab(const uint16_t* AT, const uint16_t* BT, int M, int N, int K, float* D) {
  return guarded([&] {
    D2FT_REQUIRE(K % 8 == 0 && N % 8 == 0 && M % 8 == 0, kInput, "M, N and K must be multiples of 8");
    Dev<uint16_t> dA((size_t)K * M), dB((size_t)K * N);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemcpy(dA.p, AT, (size_t)K * M * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(dB.p, BT, (size_t)K * N * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemset(dD.p, 0, (size_t)M * N * 4));
    CUtensorMap a = make_tmap_bf16_3d(dA.p, M, K, 1, (uint64_t)M * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dB.p, N, K, 1, (uint64_t)N * 2, (uint64_t)K * N * 2, 64);
    launch_gemm<DenseMNProb<208>, GemmShape<208, 4, 1, 4, 2, 1, 1>>(a, b, DenseMNProb<208>{M, N, K, 1, dD.p}, 0,
                                                                     nullptr);
    D2FT_CUDA(cudaDeviceSynchronize());
    D2FT_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

int d2ft_test_gemm_planes(const uint16_t* A, const uint16_t* X, int M, int T, int K, int P, float* D) {
  return guarded([&] {
    Dev<uint16_t> dA((size_t)M * K), dX((size_t)P * T * K + 256 * K);
    Dev<float> dD((size_t)P * M * T);
    D2FT_CUDA(cudaMemcpy(dA.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(dX.p, X, (size_t)P * T * K * 2, cudaMemcpyHostToDevice));
    using S = GemmShape<208, 5, 1>;
    CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dX.p, K, T, P, (uint64_t)K * 2, (uint64_t)K * T * 2, 208);
    launch_gemm<PlanesProb<208>, S>(a, b, PlanesProb<208>{M, T, K, P, dD.p}, 0, nullptr);
    D2FT_CUDA(cudaDeviceSynchronize());
    D2FT_CUDA(cudaMemcpy(D, dD.p, (size_t)P * M * T * 4, cudaMemcpyDeviceToHost));
  });
}

int d2ft_test_gemm_tokenk(const uint16_t* XT, const uint16_t* YT, int M, int N, int T, int TP, int P, float* D) {
  return guarded([&] {
    Dev<uint16_t> dX((size_t)P * M * TP), dY((size_t)P * N * TP);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemcpy(dX.p, XT, (size_t)P * M * TP * 2, cudaMemcpyHostToDevice));
    D2FT_CUDA(cudaMemcpy(dY.p, YT, (size_t)P * N * TP * 2, cudaMemcpyHostToDevice));
    using S = GemmShape<256, 4, 1>;
    CUtensorMap a = make_tmap_bf16_3d(dX.p, T, M, P, (uint64_t)TP * 2, (uint64_t)TP * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dY.p, T, N, P, (uint64_t)TP * 2, (uint64_t)TP * N * 2, 256);
    launch_gemm<TokenKProb<256>, S>(a, b, TokenKProb<256>{M, N, T, P, dD.p}, 0, nullptr);
    D2FT_CUDA(cudaDeviceSynchronize());
    D2FT_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

// Times `iters` launches of a dense M x N x K GEMM shaped like the step's
// tokens-as-N GEMMs (N = 208, K-major A and B, CTA pairs): variant 0 = B
// multicast (G1's config), 1 = pair UMMA (cta_group::2); ms per launch.
int d2ft_test_gemm_bench_pair(int M, int K, int variant, int iters, double* ms_per) {
  return guarded([&] {
    const int N = 208;
    Dev<uint16_t> dA((size_t)M * K), dB((size_t)N * K);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemset(dA.p, 0x3c, (size_t)M * K * 2));
    D2FT_CUDA(cudaMemset(dB.p, 0x3c, (size_t)N * K * 2));
    CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 104);
    DensePairProb<208> prob{M, N, K, (variant >= 2) ? nullptr : dD.p};
    // 4: A MN-major ([K][M]), 5: B MN-major ([K][N]), both pair UMMA, no stores
    CUtensorMap amn = make_tmap_bf16_3d(dA.p, M, K, 1, (uint64_t)M * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap bmn = make_tmap_bf16_3d(dB.p, N, K, 1, (uint64_t)N * 2, (uint64_t)K * N * 2, 64);
    DenseMNProb<208> mnp{M, N, K, 1, nullptr};
    // 6 / 7: MN-major B with N = 256 / 128 (whole 64-token blocks per CTA); 8: MN-major B multicast
    Dev<uint16_t> dB2((size_t)256 * K);
    D2FT_CUDA(cudaMemset(dB2.p, 0x3c, (size_t)256 * K * 2));
    CUtensorMap bmn256 = make_tmap_bf16_3d(dB2.p, 256, K, 1, (uint64_t)256 * 2, (uint64_t)K * 256 * 2, 64);
    DenseMNProb<256> mnp256{M, 256, K, 1, nullptr};
    DenseMNProb<128> mnp128{M, 128, K, 1, nullptr};
    const int v = variant;
    auto run = [&]() {
      if (v == 4) launch_gemm<DensePairProb<208>, GemmShape<208, 6, 1, 4, 2, 0, 1, 1>>(amn, b, prob, 0, nullptr);
      else if (v == 5) launch_gemm<DenseMNProb<208>, GemmShape<208, 6, 1, 4, 2, 1, 0, 1>>(a, bmn, mnp, 0, nullptr);
      else if (v == 6) launch_gemm<DenseMNProb<256>, GemmShape<256, 6, 1, 4, 2, 1, 0, 1>>(a, bmn256, mnp256, 0, nullptr);
      else if (v == 7) launch_gemm<DenseMNProb<128>, GemmShape<128, 8, 1, 4, 2, 1, 0, 1>>(a, bmn256, mnp128, 0, nullptr);
      else if (v == 8) launch_gemm<DenseMNProb<208>, GemmShape<208, 4, 1, 4, 2, 1, 0, 0>>(a, bmn, mnp, 0, nullptr);
      else if (v == 1 || v == 3) launch_gemm<DensePairProb<208>, GemmShape<208, 6, 1, 4, 2, 0, 0, 1>>(a, b, prob, 0, nullptr);
      else launch_gemm<DensePairProb<208>, GemmShape<208, 5, 1, 4, 2>>(a, b, prob, 0, nullptr);
    };
    for (int i = 0; i < 3; ++i) run();
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    D2FT_CUDA(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) run();
    D2FT_CUDA(cudaEventRecord(e1));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// Times `iters` launches of a dense M x N x K GEMM (device-resident random
// data) with CUDA events; returns ms per launch.
int d2ft_test_gemm_bench(int M, int N, int K, int iters, double* ms_per) {
  return guarded([&] {
    Dev<uint16_t> dA((size_t)M * K), dB((size_t)N * K);
    Dev<float> dD((size_t)M * N);
    D2FT_CUDA(cudaMemset(dA.p, 0x3c, (size_t)M * K * 2));
    D2FT_CUDA(cudaMemset(dB.p, 0x3c, (size_t)N * K * 2));
    using S = GemmShape<256, 4, 1>;
    CUtensorMap a = make_tmap_bf16_3d(dA.p, K, M, 1, (uint64_t)K * 2, (uint64_t)K * M * 2, 64);
    CUtensorMap b = make_tmap_bf16_3d(dB.p, K, N, 1, (uint64_t)K * 2, (uint64_t)K * N * 2, 256);
    DenseProb<256> prob{M, N, K, dD.p};
    for (int i = 0; i < 3; ++i) launch_gemm<DenseProb<256>, S>(a, b, prob, 0, nullptr);
    cudaEvent_t e0, e1;
    D2FT_CUDA(cudaEventCreate(&e0));
    D2FT_CUDA(cudaEventCreate(&e1));
    D2FT_CUDA(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) launch_gemm<DenseProb<256>, S>(a, b, prob, 0, nullptr);
    D2FT_CUDA(cudaEventRecord(e1));
    D2FT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    D2FT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
