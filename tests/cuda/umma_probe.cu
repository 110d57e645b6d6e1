// Test-only probe: validates the tcgen05 descriptor / TMEM conventions in csrc/umma.cuh
// against host-built operand images (tests/test_gpu_umma.py).  Not part of the product.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_1808_01517_b200/csrc/umma.cuh"

using namespace dl::umma;

// mode 0: A from smem (a_img, descriptor a_lbo/a_sbo/a_swz, per-kstep offsets a_off[])
// mode 1: A from TMEM, rows of packed bf16 pairs a_words[128][K/2]
__global__ void probe_k(int mode, const uint8_t* a_img, int a_bytes, const uint8_t* b_img, int b_bytes,
                        const uint32_t* a_words, float* d_out, int N, int K, uint32_t a_lbo, uint32_t a_sbo,
                        int a_swz, int a_mn, const uint32_t* a_off, uint32_t b_lbo, uint32_t b_sbo, int b_swz,
                        int b_mn, const uint32_t* b_off, int M) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase_s;
  uint8_t* sa = smem;
  uint8_t* sb = smem + ((a_bytes + 1023) / 1024) * 1024;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < a_bytes; i += blockDim.x) sa[i] = a_img[i];
  for (int i = tid; i < b_bytes; i += blockDim.x) sb[i] = b_img[i];
  if (warp == 0) tmem_alloc(&tbase_s, 512);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_fence_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase_s;
  const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
  if (mode == 1) {
    const int row = 32 * (warp & 3) + lane;
    for (int j = 0; j < K / 2; j += 4) {
      uint32_t w[4] = {a_words[row * (K / 2) + j], a_words[row * (K / 2) + j + 1], a_words[row * (K / 2) + j + 2],
                       a_words[row * (K / 2) + j + 3]};
      tmem_st<4>(tb + lane_off + 256 + j, w);
    }
    tmem_wait_st();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn, b_mn);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint32_t bs = smem_u32(sb) + b_off[kk];
      const uint64_t bd = b_swz ? desc_sw128_k(bs, b_sbo) : desc_noswz(bs, b_lbo, b_sbo);
      if (mode == 0) {
        const uint32_t as = smem_u32(sa) + a_off[kk];
        const uint64_t ad = a_swz ? desc_sw128_k(as, a_sbo) : desc_noswz(as, a_lbo, a_sbo);
        mma_ss(tb, ad, bd, idesc, kk > 0);
      } else {
        mma_ts(tb, tb + 256 + 8 * kk, bd, idesc, kk > 0);
      }
    }
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after();
  if (warp < 4) {
    const int row = 32 * warp + lane;
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      tmem_ld<16>(tb + lane_off + c, r);
      tmem_wait_ld();
      for (int i = 0; i < 16; ++i) d_out[row * N + c + i] = __uint_as_float(r[i]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int umma_probe(int mode, const uint8_t* a_img, int a_bytes, const uint8_t* b_img, int b_bytes,
                          const uint32_t* a_words, float* d_out, int N, int K, uint32_t a_lbo, uint32_t a_sbo,
                          int a_swz, int a_mn, const uint32_t* a_off, uint32_t b_lbo, uint32_t b_sbo, int b_swz,
                          int b_mn, const uint32_t* b_off, int M) {
  const int smem = ((a_bytes + 1023) / 1024) * 1024 + b_bytes + 1024;
  cudaFuncSetAttribute(probe_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_k<<<1, 128, smem>>>(mode, a_img, a_bytes, b_img, b_bytes, a_words, d_out, N, K, a_lbo, a_sbo, a_swz, a_mn,
                            a_off, b_lbo, b_sbo, b_swz, b_mn, b_off, M);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
