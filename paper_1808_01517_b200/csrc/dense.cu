// Small dense float64 products of the stacked-LSC path (ops.ChainStackFunction / ChainMseFunction).
//
// Stacked LSC layers fold into one operator L = L_n ... L_1 with bias d_n (d_k = L_k d_{k-1} + bvec_k), and each
// layer's gradient comes from the one float64 Gram of the fused backward: dL_k = A_k G C_{k-1}^T + (A_k s) d_{k-1}^T
// with A_k = L_{k+1}^T ... L_n^T, C_{k-1} = L_{k-1} ... L_1 (per layer), then
// dW_k[o,s,k'] = <P_k', dL_k[o,:,s,:]>, db_k = beta . (A_k s).  The matrices are at most a few hundred square
// (S * R), so one tiled SIMT kernel does every product; nothing here goes through cuBLAS.
#include "common.cuh"
#include "kernels.cuh"

namespace dl {
namespace {

constexpr int kT = 16;   // 16 x 16 output tile per block, 16-deep k slices through shared memory

// C = alpha * op(A) op(B) + beta * C, column-major-free row-major indexing: op(A) is m x k (A[i * lda + p], or
// A[p * lda + i] when ta), op(B) is k x n (B[p * ldb + j], or B[j * ldb + p] when tb).
__global__ void gemm_f64_k(int m, int n, int k, const double* __restrict__ A, int lda, int ta,
                           const double* __restrict__ B, int ldb, int tb, double* __restrict__ C, int ldc,
                           double alpha, double beta) {
  __shared__ double As[kT][kT + 1], Bs[kT][kT + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.y * kT + ty, j = blockIdx.x * kT + tx;
  double acc = 0.0;
  for (int p0 = 0; p0 < k; p0 += kT) {
    const int pa = p0 + tx, pb = p0 + ty;
    As[ty][tx] = (i < m && pa < k) ? (ta ? A[(int64_t)pa * lda + i] : A[(int64_t)i * lda + pa]) : 0.0;
    Bs[ty][tx] = (pb < k && j < n) ? (tb ? B[(int64_t)j * ldb + pb] : B[(int64_t)pb * ldb + j]) : 0.0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kT; ++q) acc = fma(As[ty][q], Bs[q][tx], acc);
    __syncthreads();
  }
  if (i < m && j < n) {
    double* c = C + (int64_t)i * ldc + j;
    *c = beta == 0.0 ? alpha * acc : fma(alpha, acc, beta * *c);
  }
}

// dW[o, s, k'] = sum_{r, t} P[k', r, t] dL[(o, r), (s, t)]; one block per output, fixed-order reduction.
__global__ void lsc_dw_k(const double* __restrict__ dL, const float* __restrict__ P, float* __restrict__ dW, int s_out,
                         int s_in, int K, int r_out, int r_in) {
  __shared__ double red[32];
  const int id = blockIdx.x;
  const int o = id / (s_in * K), s = (id / K) % s_in, kk = id % K;
  const int cols = s_in * r_in;
  double acc = 0.0;
  for (int e = threadIdx.x; e < r_out * r_in; e += blockDim.x) {
    const int r = e / r_in, t = e - r * r_in;
    acc = fma((double)__ldg(P + ((int64_t)kk * r_out + r) * r_in + t), dL[(int64_t)(o * r_out + r) * cols + s * r_in + t],
              acc);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) dW[id] = (float)v;
  }
}

}  // namespace
}  // namespace dl

extern "C" {

int dl_gemm_f64(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, int ta, const double* B, int64_t ldb,
                int tb, double* C, int64_t ldc, double alpha, double beta, void* stream) {
  using namespace dl;
  begin_call();
  DL_TRY(device_check(nullptr));
  DL_REQUIRE(m >= 0 && n >= 0 && k >= 0 && m < (1 << 20) && n < (1 << 20) && k < (1 << 20), "gemm_f64: bad sizes");
  if (m == 0 || n == 0) return DL_OK;
  DL_REQUIRE(A && B && C, "gemm_f64: null pointer");
  const dim3 grid((unsigned)ceil_div<int64_t>(n, kT), (unsigned)ceil_div<int64_t>(m, kT));
  gemm_f64_k<<<grid, dim3(kT, kT), 0, as_stream(stream)>>>((int)m, (int)n, (int)k, A, (int)lda, ta, B, (int)ldb, tb, C,
                                                           (int)ldc, alpha, beta);
  return after_launch("gemm_f64");
}

int dl_lsc_dw_from_dl_f64(const double* dL, const float* P, float* dW, int64_t s_out, int64_t s_in, int64_t K,
                          int64_t r_out, int64_t r_in, void* stream) {
  using namespace dl;
  begin_call();
  DL_TRY(device_check(nullptr));
  DL_REQUIRE(dL && P && dW && s_out >= 1 && s_in >= 1 && K >= 1 && r_out >= 1 && r_in >= 1,
             "lsc_dw_from_dl: bad arguments");
  lsc_dw_k<<<(unsigned)(s_out * s_in * K), 256, 0, as_stream(stream)>>>(dL, P, dW, (int)s_out, (int)s_in, (int)K,
                                                                        (int)r_out, (int)r_in);
  return after_launch("lsc_dw_from_dl");
}

}  // extern "C"
