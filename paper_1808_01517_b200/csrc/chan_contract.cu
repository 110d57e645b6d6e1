// K1 chan_contract: per-voxel channel contraction out = W . in (+ bias), SIMT fp32.
// (Operators with more than 144 output rows are split into 48-row slices, each streaming the input.)
//
// Replaces fitting._apply_channel_matrix (/root/reference/pkg/src/sphdwi/fitting.py:155-188),
// which runs a (C_out x C_in) . (C_in x 1024) dgemm per zero-padded voxel block.
// Here one persistent CTA owns a TM-row slice of W (staged once in shared memory,
// transposed so a row j of inputs meets TM contiguous weights) and streams voxel
// tiles: each thread holds TM x 2 accumulators for 2 adjacent voxels, reads its
// inputs straight from HBM with 8-byte coalesced loads (double-buffered in
// registers), broadcasts W from shared memory, and writes TM x 2 outputs with
// coalesced 8-byte stores.  No intermediate ever touches HBM.
#include "common.cuh"
#include "kernels.cuh"

namespace dl {
namespace {

constexpr int kThreads = 256;
constexpr int kTile = 2 * kThreads;   // voxels per CTA iteration
constexpr int kUnroll = 8;            // input rows in flight per thread

template <bool VEC2>
__device__ __forceinline__ float2 load_x(const float* __restrict__ p, bool full, bool any) {
  if (VEC2) {
    if (full) return __ldg(reinterpret_cast<const float2*>(p));
    return make_float2(any ? __ldg(p) : 0.f, 0.f);
  }
  return make_float2(any ? __ldg(p) : 0.f, full ? __ldg(p + 1) : 0.f);
}

template <int TM, bool VEC2>
__global__ void __launch_bounds__(kThreads, 1)
chan_contract_k(const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ W,
                const float* __restrict__ bias, int c_in, int c_out, int64_t nvox, int64_t in_bs,
                int64_t out_bs, int64_t nbatch, int w_per_group, int64_t tiles_per_b) {
  extern __shared__ __align__(16) float Ws[];  // [c_in][TM]
  const int cb = blockIdx.y, g = blockIdx.z, i0 = cb * TM;
  const float* Wg = W + (w_per_group ? (int64_t)g * c_out * c_in : 0);
  for (int idx = threadIdx.x; idx < c_in * TM; idx += kThreads) {
    const int j = idx / TM, i = idx - j * TM;
    Ws[idx] = (i0 + i < c_out) ? __ldg(Wg + (int64_t)(i0 + i) * c_in + j) : 0.f;
  }
  const float* bg = bias ? bias + (w_per_group ? (int64_t)g * c_out : 0) + i0 : nullptr;
  __syncthreads();

  const int64_t ntiles = nbatch * tiles_per_b;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const int64_t v = (t - b * tiles_per_b) * kTile + 2 * threadIdx.x;
    const bool any = v < nvox, full = v + 1 < nvox;
    const float* src = in + b * in_bs + (int64_t)g * c_in * nvox + v;

    float acc[TM][2];
#pragma unroll
    for (int i = 0; i < TM; ++i) acc[i][0] = acc[i][1] = 0.f;

    float2 buf[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      buf[u] = (u < c_in) ? load_x<VEC2>(src + (int64_t)u * nvox, full, any) : make_float2(0.f, 0.f);

    for (int j0 = 0; j0 < c_in; j0 += kUnroll) {
      float2 cur[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) cur[u] = buf[u];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int j = j0 + kUnroll + u;
        buf[u] = (j < c_in) ? load_x<VEC2>(src + (int64_t)j * nvox, full, any) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (j0 + u < c_in) {
          const float4* wr = reinterpret_cast<const float4*>(Ws + (j0 + u) * TM);
#pragma unroll
          for (int q = 0; q < TM / 4; ++q) {
            const float4 w = wr[q];
            acc[4 * q + 0][0] = fmaf(w.x, cur[u].x, acc[4 * q + 0][0]);
            acc[4 * q + 0][1] = fmaf(w.x, cur[u].y, acc[4 * q + 0][1]);
            acc[4 * q + 1][0] = fmaf(w.y, cur[u].x, acc[4 * q + 1][0]);
            acc[4 * q + 1][1] = fmaf(w.y, cur[u].y, acc[4 * q + 1][1]);
            acc[4 * q + 2][0] = fmaf(w.z, cur[u].x, acc[4 * q + 2][0]);
            acc[4 * q + 2][1] = fmaf(w.z, cur[u].y, acc[4 * q + 2][1]);
            acc[4 * q + 3][0] = fmaf(w.w, cur[u].x, acc[4 * q + 3][0]);
            acc[4 * q + 3][1] = fmaf(w.w, cur[u].y, acc[4 * q + 3][1]);
          }
        }
      }
    }

    if (any) {
      float* dst = out + b * out_bs + ((int64_t)g * c_out + i0) * nvox + v;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        if (i0 + i < c_out) {
          const float bi = bg ? __ldg(bg + i) : 0.f;
          float* p = dst + (int64_t)i * nvox;
          if (VEC2 && full) {
            *reinterpret_cast<float2*>(p) = make_float2(acc[i][0] + bi, acc[i][1] + bi);
          } else {
            p[0] = acc[i][0] + bi;
            if (full) p[1] = acc[i][1] + bi;
          }
        }
      }
    }
  }
}

// One voxel per thread, all TM (<= 144) output rows per CTA: every input row is read once (no per-slice
// re-streaming) -- SH2Signal (90 rows), a 3-shell LSC operator (135), and small volumes, where a tile of 256
// voxels gives twice the CTAs of the two-voxel kernel.
template <int TM>
__global__ void __launch_bounds__(kThreads, 1)
chan_contract1_k(const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ W,
                 const float* __restrict__ bias, int c_in, int c_out, int64_t nvox, int64_t in_bs,
                 int64_t out_bs, int64_t nbatch, int w_per_group, int64_t tiles_per_b) {
  extern __shared__ __align__(16) float Ws[];  // [c_in][TM]
  const int g = blockIdx.z;
  const float* Wg = W + (w_per_group ? (int64_t)g * c_out * c_in : 0);
  for (int idx = threadIdx.x; idx < c_in * TM; idx += kThreads) {
    const int j = idx / TM, i = idx - j * TM;
    Ws[idx] = (i < c_out) ? __ldg(Wg + (int64_t)i * c_in + j) : 0.f;
  }
  const float* bg = bias ? bias + (w_per_group ? (int64_t)g * c_out : 0) : nullptr;
  __syncthreads();

  const int64_t ntiles = nbatch * tiles_per_b;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const int64_t v = (t - b * tiles_per_b) * kThreads + threadIdx.x;
    const bool any = v < nvox;
    const float* src = in + b * in_bs + (int64_t)g * c_in * nvox + (any ? v : 0);
    float acc[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) acc[i] = 0.f;
    constexpr int kU = kUnroll;   // input rows in flight per thread
    float buf[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) buf[u] = (u < c_in && any) ? __ldg(src + (int64_t)u * nvox) : 0.f;
    for (int j0 = 0; j0 < c_in; j0 += kU) {
      float cur[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cur[u] = buf[u];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = j0 + kU + u;
        buf[u] = (j < c_in && any) ? __ldg(src + (int64_t)j * nvox) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (j0 + u < c_in) {
          const float4* wr = reinterpret_cast<const float4*>(Ws + (j0 + u) * TM);
#pragma unroll
          for (int q = 0; q < TM / 4; ++q) {
            const float4 w = wr[q];
            acc[4 * q + 0] = fmaf(w.x, cur[u], acc[4 * q + 0]);
            acc[4 * q + 1] = fmaf(w.y, cur[u], acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(w.z, cur[u], acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(w.w, cur[u], acc[4 * q + 3]);
          }
        }
      }
    }
    if (any) {
      float* dst = out + b * out_bs + (int64_t)g * c_out * nvox + v;
#pragma unroll
      for (int i = 0; i < TM; ++i)
        if (i < c_out) dst[(int64_t)i * nvox] = acc[i] + (bg ? __ldg(bg + i) : 0.f);
    }
  }
}

template <int TM>
int launch_tm1(const float* in, float* out, const float* W, const float* bias, int64_t nbatch, int64_t groups,
               int64_t c_in, int64_t c_out, int64_t nvox, int64_t in_bs, int64_t out_bs, int w_per_group,
               cudaStream_t st, int sm_count) {
  auto kern = chan_contract1_k<TM>;
  const size_t smem = (size_t)c_in * TM * sizeof(float);
  DL_REQUIRE(smem <= 227 * 1024, "chan_contract: c_in=%lld too large for shared memory", (long long)c_in);
  DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  DL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
  if (occ < 1) occ = 1;
  const int64_t tiles_per_b = ceil_div<int64_t>(nvox, kThreads);
  const int64_t ntiles = nbatch * tiles_per_b;
  int64_t p = ((int64_t)sm_count * occ) / groups;
  if (p < 1) p = 1;
  if (p > ntiles) p = ntiles;
  dim3 grid((unsigned)p, 1u, (unsigned)groups);
  kern<<<grid, kThreads, smem, st>>>(in, out, W, bias, (int)c_in, (int)c_out, nvox, in_bs, out_bs, nbatch,
                                     w_per_group, tiles_per_b);
  return after_launch("chan_contract");
}

template <int TM, bool VEC2>
int launch_tm(const float* in, float* out, const float* W, const float* bias, int64_t nbatch,
              int64_t groups, int64_t c_in, int64_t c_out, int64_t nvox, int64_t in_bs,
              int64_t out_bs, int w_per_group, cudaStream_t st, int sm_count) {
  auto kern = chan_contract_k<TM, VEC2>;
  const size_t smem = (size_t)c_in * TM * sizeof(float);
  DL_REQUIRE(smem <= 227 * 1024, "chan_contract: c_in=%lld too large for shared memory", (long long)c_in);
  DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  DL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
  if (occ < 1) occ = 1;
  const int64_t ncb = ceil_div<int64_t>(c_out, TM);
  const int64_t tiles_per_b = ceil_div<int64_t>(nvox, kTile);
  const int64_t ntiles = nbatch * tiles_per_b;
  int64_t p = ((int64_t)sm_count * occ) / (ncb * groups);
  if (p < 1) p = 1;
  if (p > ntiles) p = ntiles;
  dim3 grid((unsigned)p, (unsigned)ncb, (unsigned)groups);
  kern<<<grid, kThreads, smem, st>>>(in, out, W, bias, (int)c_in, (int)c_out, nvox, in_bs, out_bs,
                                     nbatch, w_per_group, tiles_per_b);
  return after_launch("chan_contract");
}

}  // namespace

int chan_contract(const float* in, float* out, const float* W, const float* bias, int64_t nbatch,
                  int64_t groups, int64_t c_in, int64_t c_out, int64_t nvox, int64_t in_bs,
                  int64_t out_bs, int w_per_group, cudaStream_t st) {
  int sm = 0;
  DL_TRY(device_check(&sm));
  DL_REQUIRE(nbatch >= 0 && groups >= 1 && c_in >= 1 && c_out >= 1 && nvox >= 0,
             "chan_contract: bad sizes (nbatch=%lld groups=%lld c_in=%lld c_out=%lld nvox=%lld)",
             (long long)nbatch, (long long)groups, (long long)c_in, (long long)c_out, (long long)nvox);
  DL_REQUIRE(groups <= 65535, "chan_contract: too many groups");
  if (nbatch == 0 || nvox == 0) return DL_OK;
  DL_REQUIRE(in && out && W, "chan_contract: null pointer");
  DL_REQUIRE(in_bs >= groups * c_in * nvox && out_bs >= groups * c_out * nvox,
             "chan_contract: subject stride smaller than one subject");
  const bool vec2 = (nvox % 2 == 0) && (in_bs % 2 == 0) && (out_bs % 2 == 0) &&
                    ((uintptr_t)in % 8 == 0) && ((uintptr_t)out % 8 == 0);
#define DL_CC(TM)                                                                                  \
  return vec2 ? launch_tm<TM, true>(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs,   \
                                    out_bs, w_per_group, st, sm)                                  \
              : launch_tm<TM, false>(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs,  \
                                     out_bs, w_per_group, st, sm)
  // one voxel per thread and every output row in one CTA when the rows fit in registers (no input re-streaming),
  // or when the two-voxel tiles would leave most SMs idle (small volumes)
  const int64_t tiles2 = nbatch * ceil_div<int64_t>(nvox, kTile) * groups;
  if (c_out > 48 && c_out <= 96)
    return launch_tm1<96>(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs, out_bs, w_per_group, st, sm);
  if (c_out > 96 && c_out <= 144)
    return launch_tm1<144>(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs, out_bs, w_per_group, st, sm);
  if (c_out <= 48 && tiles2 < 2 * sm)
    return launch_tm1<48>(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs, out_bs, w_per_group, st, sm);
  if (c_out <= 16) DL_CC(16);
  if (c_out <= 32) DL_CC(32);
  DL_CC(48);
#undef DL_CC
}

}  // namespace dl

extern "C" int dl_chan_contract_f32(const float* in, float* out, const float* W, const float* bias,
                                    int64_t nbatch, int64_t groups, int64_t c_in, int64_t c_out,
                                    int64_t nvox, int64_t in_bs, int64_t out_bs, int w_per_group,
                                    void* stream) {
  dl::begin_call();
  return dl::chan_contract(in, out, W, bias, nbatch, groups, c_in, c_out, nvox, in_bs, out_bs,
                           w_per_group, dl::as_stream(stream));
}
