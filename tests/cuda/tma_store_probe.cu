// Test-only probe: does a TMA tensor store / load accept a box whose global start is only 8-byte aligned?
// The chain kernels view (rows, nvox) fp32 as channel pairs (2*nvox, rows/2); with nvox % 4 == 2 every odd
// channel row starts 8 bytes off a 16-byte boundary.  Stores box [32 voxels x 8 pairs] at (u0, 0) and
// loads the same box back; the host checks values and that nothing outside the box was written.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../paper_1808_01517_b200/csrc/umma.cuh"

using namespace dl::umma;

__global__ void probe_k(const __grid_constant__ CUtensorMap tm, int u0, float* back) {
  __shared__ __align__(128) float box[8][32];
  __shared__ __align__(128) float box2[8][32];
  __shared__ uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 256; i += blockDim.x) box[i / 32][i % 32] = 1000.f + i;
  if (t == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (t == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(&tm), "r"(u0),
                 "r"(0), "r"(smem_u32(&box[0][0]))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    mbar_arrive_tx(&bar, 1024);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(&box2[0][0])),
        "l"(&tm), "r"(u0), "r"(0), "r"(smem_u32(&bar))
        : "memory");
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = t; i < 256; i += blockDim.x) back[i] = box2[i / 32][i % 32];
}

extern "C" int tma_store_probe(int64_t nvox, int u0, float* host_out, float* host_back) {
  const int rows = 16;
  float* g;
  float* back;
  cudaMalloc(&g, rows * nvox * 4);
  cudaMalloc(&back, 256 * 4);
  cudaMemset(g, 0xFF, rows * nvox * 4);   // NaN pattern
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * nvox), (cuuint64_t)(rows / 2)};
  const cuuint64_t strides[1] = {(cuuint64_t)(8 * nvox)};
  const cuuint32_t boxd[2] = {32u, 8u};
  const cuuint32_t es[2] = {1u, 1u};
  int r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != 0) return 1000 + r;
  probe_k<<<1, 128>>>(tm, u0, back);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host_out, g, rows * nvox * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(host_back, back, 256 * 4, cudaMemcpyDeviceToHost);
  cudaFree(g);
  cudaFree(back);
  return (int)e;
}
