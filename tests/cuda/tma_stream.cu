// Test-only microbenchmark: HBM read bandwidth of the channel-pair TMA streaming pattern used by the
// chain / Gram kernels (boxes of W voxels x 8 channel pairs, NS-stage ring, one consumer warp).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../paper_1808_01517_b200/csrc/umma.cuh"

using namespace dl::umma;

struct P {
  CUtensorMap tm;
  int64_t nvox, tiles;
  int rows, W, NS, consumers;
};

__global__ void __launch_bounds__(256, 1) stream_k(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 32;
  uint8_t* ring = smem + 1024;
  const int warp = threadIdx.x >> 5;
  const uint32_t stage = (uint32_t)(16 * (p.W + 4) * 4);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], p.consumers); }
    mbar_fence_init();
  }
  __syncthreads();
  const int per_tile = p.rows / 16;
  const int sh = (int)(p.nvox & 3);
  if (warp == 0) {
    uint32_t s = 0, round = 0;
    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int v0 = (int)(t * p.W);
      for (int r = 0; r < per_tile; ++r) {
        if (round > 0) mbar_wait_warp(&empty[s], (round - 1) & 1);
        if (elect_one()) {
          mbar_arrive_tx(&full[s], stage);
          tma_load_3d(ring + s * stage, &p.tm, v0, 8 * r, 0, &full[s]);
          tma_load_3d(ring + s * stage + stage / 2, &p.tm, (int)p.nvox + v0 - sh, 8 * r, 0, &full[s]);
        }
        __syncwarp();
        if (++s == (uint32_t)p.NS) { s = 0; ++round; }
      }
    }
  } else if (warp <= p.consumers) {
    uint32_t s = 0, round = 0;
    float acc = 0.f;
    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x)
      for (int r = 0; r < per_tile; ++r) {
        mbar_wait_warp(&full[s], round & 1);
        acc += reinterpret_cast<const float*>(ring + s * stage)[threadIdx.x & 31];
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        if (++s == (uint32_t)p.NS) { s = 0; ++round; }
      }
    if (acc == 12345.f) printf("x");
  }
}

// Read + write: 4 consumer warps (one per 32-voxel quarter of the 128-voxel tile) read each 16-channel stage
// and store it to `out` with the chain kernel's OUT pattern (thread = voxel, one 128-byte row segment per
// warp store); `wrows` of every 16 rows are stored (the rest only read).
__global__ void __launch_bounds__(160, 1) stream_rw_k(const __grid_constant__ P p, float* out, int wrows) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 32;
  uint8_t* ring = smem + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t stage = (uint32_t)(16 * (p.W + 4) * 4);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    mbar_fence_init();
  }
  __syncthreads();
  const int per_tile = p.rows / 16;
  const int sh = (int)(p.nvox & 3);
  if (warp == 0) {
    uint32_t s = 0, round = 0;
    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int v0 = (int)(t * p.W);
      for (int r = 0; r < per_tile; ++r) {
        if (round > 0) mbar_wait_warp(&empty[s], (round - 1) & 1);
        if (elect_one()) {
          mbar_arrive_tx(&full[s], stage);
          tma_load_3d(ring + s * stage, &p.tm, v0, 8 * r, 0, &full[s]);
          tma_load_3d(ring + s * stage + stage / 2, &p.tm, (int)p.nvox + v0 - sh, 8 * r, 0, &full[s]);
        }
        __syncwarp();
        if (++s == (uint32_t)p.NS) { s = 0; ++round; }
      }
    }
  } else {
    const int q = warp - 1;
    const int odd0 = 8 * (p.W + 4) + sh;
    uint32_t s = 0, round = 0;
    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int64_t v = t * p.W + 32 * q + lane;
      for (int r = 0; r < per_tile; ++r) {
        mbar_wait_warp(&full[s], round & 1);
        const float* rp = reinterpret_cast<const float*>(ring + s * stage) + 32 * q + lane;
        float vals[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) vals[j] = rp[(j & 1) * odd0 + (j >> 1) * (p.W + 4)];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (v < p.nvox) {
          float* d = out + (int64_t)(16 * r) * p.nvox + v;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < wrows) __stcs(d + (int64_t)j * p.nvox, vals[j]);
        }
        if (++s == (uint32_t)p.NS) { s = 0; ++round; }
      }
    }
  }
}

extern "C" int tma_stream_rw(const float* base, float* out, int64_t nvox, int rows, int NS, int wrows, float* ms_out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int W = 128;
  P p{};
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * nvox), (cuuint64_t)(rows / 2), 1};
  const cuuint64_t strides[2] = {(cuuint64_t)(8 * nvox), (cuuint64_t)(4 * rows * nvox)};
  const cuuint32_t box[3] = {(cuuint32_t)(W + 4), 8u, 1u};
  const cuuint32_t es[3] = {1, 1, 1};
  if (encode(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  p.nvox = nvox;
  p.tiles = (nvox + W - 1) / W;
  p.rows = rows;
  p.W = W;
  p.NS = NS;
  const int smem = 1024 + NS * 16 * (W + 4) * 4;
  cudaFuncSetAttribute(stream_rw_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  stream_rw_k<<<148, 160, smem>>>(p, out, wrows);
  cudaEventRecord(a);
  stream_rw_k<<<148, 160, smem>>>(p, out, wrows);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  cudaEventElapsedTime(ms_out, a, b);
  return (int)e;
}

extern "C" int tma_stream(const float* base, int64_t nvox, int rows, int W, int NS, int consumers, float* ms_out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  P p{};
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * nvox), (cuuint64_t)(rows / 2), 1};
  const cuuint64_t strides[2] = {(cuuint64_t)(8 * nvox), (cuuint64_t)(4 * rows * nvox)};
  const cuuint32_t box[3] = {(cuuint32_t)(W + 4), 8u, 1u};
  const cuuint32_t es[3] = {1, 1, 1};
  if (encode(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  p.nvox = nvox;
  p.tiles = (nvox + W - 1) / W;
  p.rows = rows;
  p.W = W;
  p.NS = NS;
  p.consumers = consumers;
  const int smem = 1024 + NS * 16 * (W + 4) * 4;
  cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  stream_k<<<148, 256, smem>>>(p);
  cudaEventRecord(a);
  stream_k<<<148, 256, smem>>>(p);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  cudaEventElapsedTime(ms_out, a, b);
  return (int)e;
}
