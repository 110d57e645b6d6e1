// LSC operator build and weight/bias gradient (SIMT fp32 with fp64 finalize).
//
// Reference forward (per voxel, /root/reference/pkg/src/sphdwi/_kernels.py:91-104 then the
// refit at lsc.py:197):  u[o,i] = bias[o] + sum_{s,k} w[o,s,k] Rs[iK+k].c[s];  c_out[o] = F u[o].
// Folded: c_out[o] = sum_s L_{o,s} c[s] + bias[o] beta with
// P_k = F Rs[k::K], L_{o,s} = sum_k w[o,s,k] P_k, beta = F 1.  The forward is then a
// chan_contract with W = L (one group spanning all shells) and bias = bvec.
// The reference has no backward; the gradient here is the adjoint of the
// folded map: dW[o,s,k] = <P_k, sum_v g[o] c[s]^T>, db[o] = beta . sum_v g[o].
#include "common.cuh"
#include "kernels.cuh"

namespace dl {
namespace {

__global__ void build_operator_k(const float* __restrict__ P, const float* __restrict__ beta,
                                 const float* __restrict__ w, const float* __restrict__ bias,
                                 float* __restrict__ L, float* __restrict__ Lt, float* __restrict__ bvec,
                                 int s_out, int s_in, int K, int r_out, int r_in) {
  const int rows = s_out * r_out, cols = s_in * r_in;
  const int64_t n = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / cols), col = (int)(e - (int64_t)row * cols);
    const int o = row / r_out, r = row - o * r_out, s = col / r_in, t = col - s * r_in;
    float acc = 0.f;
    for (int k = 0; k < K; ++k)
      acc = fmaf(__ldg(w + ((int64_t)o * s_in + s) * K + k), __ldg(P + ((int64_t)k * r_out + r) * r_in + t), acc);
    if (L) L[e] = acc;
    if (Lt) Lt[(int64_t)col * rows + row] = acc;
    if (bvec && col == 0) bvec[row] = bias ? __ldg(bias + o) * __ldg(beta + r) : 0.f;
  }
}

// ---- Gram partials: partial[p][row][col] = sum over this CTA's voxel tiles of g[row] * c_aug[col]
// where c_aug = [c; 1] (the ones column yields sum_v g for the bias gradient).
// Output tile edge GT = 16 thread groups x GPER rows / cols per thread: 144 (9 x 9 per thread) for 3-shell
// operators, 48 (3 x 3) when rows and cols + 1 fit one 48 tile (a single-shell order-8 LSC: 45 x 46), so a
// small Gram does not pay for a 144 x 144 tile.
constexpr int kGVK = 32;     // voxels per shared-memory stage
constexpr int kMaxParts = 512;

template <int kGT, int kGPer>
__global__ void __launch_bounds__(256, 2)
gram_k(const float* __restrict__ g, const float* __restrict__ c, float* __restrict__ partials, int rows,
       int cols, int64_t nvox, int64_t g_bs, int64_t c_bs, int64_t nbatch, int64_t tiles_per_b) {
  __shared__ float gs[kGT][kGVK + 1];
  __shared__ float cs[kGT][kGVK + 1];
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
  const int row0 = blockIdx.y * kGT, col0 = blockIdx.z * kGT;
  const int ccols = cols + 1;
  float acc[kGPer][kGPer];
#pragma unroll
  for (int i = 0; i < kGPer; ++i)
#pragma unroll
    for (int j = 0; j < kGPer; ++j) acc[i][j] = 0.f;

  const int64_t ntiles = nbatch * tiles_per_b;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const int64_t v0 = (t - b * tiles_per_b) * kGVK;
    const float* gb = g + b * g_bs;
    const float* cbp = c + b * c_bs;
    for (int idx = threadIdx.x; idx < kGT * kGVK; idx += 256) {
      const int r = idx / kGVK, k = idx - r * kGVK;
      const int64_t v = v0 + k;
      const bool inv = v < nvox;
      const int gr = row0 + r, cc = col0 + r;
      gs[r][k] = (inv && gr < rows) ? __ldg(gb + (int64_t)gr * nvox + v) : 0.f;
      cs[r][k] = (inv && cc < cols) ? __ldg(cbp + (int64_t)cc * nvox + v) : ((inv && cc == cols) ? 1.f : 0.f);
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kGVK; ++k) {
      float a[kGPer], bb[kGPer];
#pragma unroll
      for (int i = 0; i < kGPer; ++i) a[i] = gs[tr * kGPer + i][k];
#pragma unroll
      for (int j = 0; j < kGPer; ++j) bb[j] = cs[tc * kGPer + j][k];
#pragma unroll
      for (int i = 0; i < kGPer; ++i)
#pragma unroll
        for (int j = 0; j < kGPer; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* pp = partials + (int64_t)blockIdx.x * rows * ccols;
#pragma unroll
  for (int i = 0; i < kGPer; ++i) {
    const int r = row0 + tr * kGPer + i;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < kGPer; ++j) {
      const int cc = col0 + tc * kGPer + j;
      if (cc < ccols) pp[(int64_t)r * ccols + cc] = acc[i][j];
    }
  }
}

// Fixed-order float64 sum of the partials.  Block (32, 8): lane x takes one element, row y a contiguous chunk
// of parts (loads of eight parts in flight); the chunk sums are added in chunk order (deterministic).
__global__ void __launch_bounds__(256) reduce_parts_k(const float* __restrict__ partials, double* __restrict__ G,
                                                      int nparts, int64_t n) {
  __shared__ double red[8][33];
  const int64_t e = blockIdx.x * 32LL + threadIdx.x;
  const int per = (nparts + 7) / 8;
  const int q0 = threadIdx.y * per, q1 = q0 + per < nparts ? q0 + per : nparts;
  double s = 0.0;
  if (e < n) {
    int q = q0;
    for (; q + 8 <= q1; q += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(partials + (int64_t)(q + j) * n + e);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += (double)v[j];
    }
    for (; q < q1; ++q) s += (double)__ldg(partials + (int64_t)q * n + e);
  }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && e < n) {
    double t = red[0][threadIdx.x];
#pragma unroll
    for (int c = 1; c < 8; ++c) t += red[c][threadIdx.x];
    G[e] = t;
  }
}

// One block per output: dW[o,s,k] = <P_k, G_{o,s}>, then db[o] = beta . G[o rows, ones col].
__global__ void finalize_k(const double* __restrict__ G, const float* __restrict__ P,
                           const float* __restrict__ beta, float* __restrict__ dW, float* __restrict__ db,
                           int s_out, int s_in, int K, int r_out, int r_in) {
  __shared__ double red[32];
  const int ccols = s_in * r_in + 1;
  const int nw = s_out * s_in * K;
  const int id = blockIdx.x;
  double acc = 0.0;
  if (id < nw) {
    const int o = id / (s_in * K), s = (id / K) % s_in, k = id % K;
    for (int e = threadIdx.x; e < r_out * r_in; e += blockDim.x) {
      const int r = e / r_in, t = e - r * r_in;
      acc += (double)__ldg(P + ((int64_t)k * r_out + r) * r_in + t) * G[(int64_t)(o * r_out + r) * ccols + s * r_in + t];
    }
  } else {
    const int o = id - nw;
    for (int r = threadIdx.x; r < r_out; r += blockDim.x)
      acc += (double)__ldg(beta + r) * G[(int64_t)(o * r_out + r) * ccols + (ccols - 1)];
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) {
      if (id < nw) { if (dW) dW[id] = (float)v; }
      else if (db) db[id - nw] = (float)v;
    }
  }
}

}  // namespace

int lsc_build_operator(const float* P, const float* beta, const float* w, const float* bias, float* L,
                       float* Lt, float* bvec, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
                       int64_t r_in, cudaStream_t st) {
  DL_TRY(device_check(nullptr));
  DL_REQUIRE(s_out >= 1 && s_in >= 1 && K >= 1 && r_out >= 1 && r_in >= 1, "lsc_build_operator: bad sizes");
  DL_REQUIRE(P && w && (L || Lt || bvec), "lsc_build_operator: null pointer");
  DL_REQUIRE(!bvec || beta, "lsc_build_operator: bvec needs beta");
  const int64_t n = s_out * r_out * s_in * r_in;
  const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  build_operator_k<<<blocks, 256, 0, st>>>(P, beta, w, bias, L, Lt, bvec, (int)s_out, (int)s_in, (int)K,
                                          (int)r_out, (int)r_in);
  return after_launch("lsc_build_operator");
}

size_t lsc_wgrad_workspace_bytes(int64_t s_out, int64_t s_in, int64_t r_out, int64_t r_in) {
  const size_t n = (size_t)(s_out * r_out) * (size_t)(s_in * r_in + 1);
  return (size_t)kMaxParts * n * sizeof(float) + n * sizeof(double) + 256;
}

int lsc_wgrad(const float* g, const float* c, const float* P, const float* beta, float* dW, float* db,
              void* workspace, int64_t nbatch, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
              int64_t r_in, int64_t nvox, int64_t g_bs, int64_t c_bs, cudaStream_t st) {
  int sm = 0;
  DL_TRY(device_check(&sm));
  DL_REQUIRE(s_out >= 1 && s_in >= 1 && K >= 1 && r_out >= 1 && r_in >= 1 && nbatch >= 0 && nvox >= 0,
             "lsc_wgrad: bad sizes");
  DL_REQUIRE(P && beta && workspace && (dW || db), "lsc_wgrad: null pointer");
  const int rows = (int)(s_out * r_out), cols = (int)(s_in * r_in);
  const int64_t n = (int64_t)rows * (cols + 1);
  float* partials = reinterpret_cast<float*>(workspace);
  double* G = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(partials + (int64_t)kMaxParts * n) + 255) & ~uintptr_t(255));
  const int64_t tiles_per_b = ceil_div<int64_t>(nvox, kGVK);
  const int64_t ntiles = nbatch * tiles_per_b;
  const bool small = rows <= 48 && cols + 1 <= 48;
  const int gt = small ? 48 : 144;
  const int rt = ceil_div(rows, gt), ct = ceil_div(cols + 1, gt);
  int64_t parts = (int64_t)sm * 2 / (rt * ct);
  if (parts < 1) parts = 1;
  if (parts > kMaxParts) parts = kMaxParts;
  if (parts > ntiles) parts = ntiles > 0 ? ntiles : 1;
  if (ntiles > 0) {
    DL_REQUIRE(g && c, "lsc_wgrad: null g/c");
    if (small)
      gram_k<48, 3><<<dim3((unsigned)parts, rt, ct), 256, 0, st>>>(g, c, partials, rows, cols, nvox, g_bs, c_bs,
                                                                  nbatch, tiles_per_b);
    else
      gram_k<144, 9><<<dim3((unsigned)parts, rt, ct), 256, 0, st>>>(g, c, partials, rows, cols, nvox, g_bs, c_bs,
                                                                   nbatch, tiles_per_b);
    DL_TRY(after_launch("lsc_gram"));
  } else {
    DL_CUDA(cudaMemsetAsync(partials, 0, n * sizeof(float), st));
  }
  reduce_parts_k<<<(unsigned)((n + 31) / 32), dim3(32, 8), 0, st>>>(partials, G, (int)parts, n);
  DL_TRY(after_launch("lsc_reduce_parts"));
  finalize_k<<<(unsigned)(s_out * s_in * K + s_out), 256, 0, st>>>(G, P, beta, dW, db, (int)s_out, (int)s_in,
                                                                   (int)K, (int)r_out, (int)r_in);
  return after_launch("lsc_wgrad_finalize");
}

}  // namespace dl

extern "C" {

int dl_lsc_build_operator_f32(const float* P, const float* beta, const float* w, const float* bias, float* L,
                              float* Lt, float* bvec, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
                              int64_t r_in, void* stream) {
  dl::begin_call();
  return dl::lsc_build_operator(P, beta, w, bias, L, Lt, bvec, s_out, s_in, K, r_out, r_in,
                                dl::as_stream(stream));
}

size_t dl_lsc_wgrad_workspace_bytes(int64_t s_out, int64_t s_in, int64_t r_out, int64_t r_in) {
  return dl::lsc_wgrad_workspace_bytes(s_out, s_in, r_out, r_in);
}

int dl_lsc_wgrad_f32(const float* g, const float* c, const float* P, const float* beta, float* dW, float* db,
                     void* workspace, int64_t nbatch, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
                     int64_t r_in, int64_t nvox, int64_t g_bs, int64_t c_bs, void* stream) {
  dl::begin_call();
  return dl::lsc_wgrad(g, c, P, beta, dW, db, workspace, nbatch, s_out, s_in, K, r_out, r_in, nvox, g_bs,
                       c_bs, dl::as_stream(stream));
}

}  // extern "C"
