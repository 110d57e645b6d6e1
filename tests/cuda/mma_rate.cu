// Test-only microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, cta_group::1) for SS/TS and N.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../paper_1808_01517_b200/csrc/umma.cuh"

using namespace dl::umma;

__global__ void rate_k(int mode, int N, int iters, long long* out, int dcol, int acol) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (mode >= 70 ? 200 : 64) * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tb_s, 512);
  if (threadIdx.x == 0) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tb_s;
  if (mode >= 80) {
    // TMEM load throughput without MMAs: warps 1..(blockDim/32-1) load for `iters` cycles.
    // mode 80: 32x32b.x8, 81: x16, 82: x32, 83: x16 with distinct columns per warp, 84: x32 two in flight
    long long t0 = clock64();
    if (warp == 0 && mode >= 85) {
      // mode 85: TS MMAs (N, D at col 0, A at col 256) back to back; 86: SS; 87: TMEM stores (x16) by warp 0
      const uint32_t sbb = smem_u32(smem + 32768);
      const uint64_t bd = desc_noswz(sbb, 128, 256), ad = desc_noswz(smem_u32(smem), 128, 256);
      const uint32_t id = idesc_bf16(128, N, 0, 0);
      long long k = 0;
      while (clock64() - t0 < (long long)iters) {
        if (mode == 87) {
          uint32_t q[16];
          for (int i = 0; i < 16; ++i) q[i] = i;
          tmem_st<16>(tb + 256u, q);
          tmem_wait_st();
        } else {
          for (int j = 0; j < 16; ++j) {
            if (elect_one()) {
              if (mode == 85) mma_ts(tb, tb + 256u, bd, id, 1);
              else mma_ss(tb, ad, bd, id, 1);
            }
            __syncwarp();
          }
          if (elect_one()) commit(&mbar);
          __syncwarp();
          mbar_wait(&mbar, (uint32_t)(k & 1));
        }
        ++k;
      }
      if (threadIdx.x == 0) out[0] = k;
    } else if (warp > 0) {
      const uint32_t ta = tb + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)dcol +
                          (mode == 83 || mode == 84 ? (uint32_t)((warp >> 2) * 64) : 0u);
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) r[i] = i;
      long long n = 0;
      while (clock64() - t0 < (long long)iters) {
        if (mode == 80) { uint32_t q[8]; tmem_ld<8>(ta, q); tmem_wait_ld(); r[0] += q[0]; }
        else if (mode == 81 || mode == 83 || mode >= 85) { uint32_t q[16]; tmem_ld<16>(ta, q); tmem_wait_ld(); r[0] += q[0]; }
        else if (mode == 82) { tmem_ld<32>(ta, r); tmem_wait_ld(); }
        else { uint32_t q[16], q2[16]; tmem_ld<16>(ta, q); tmem_ld<16>(ta + 16, q2); tmem_wait_ld(); r[0] += q[0] + q2[0]; }
        ++n;
      }
      if (r[0] == 12345u) out[1] = 0;
      if ((threadIdx.x & 31) == 0 && warp == 1) out[1] = n;
    }
    if (threadIdx.x == 0 && mode < 85) out[0] = iters;
  } else if (mode >= 70) {
    // the chain kernel's stage-2 pattern: B = three 144x144 K-major images (SBO 2304) 41472 bytes apart
    // in a 128 KB region, A alternating between two TMEM slots (cols 72 / 96), D at col 264 (N = 144),
    // 9 K-steps per item, a commit per K-step.  mode 71: the B images one byte-offset 0 apart (same image)
    __shared__ uint64_t mb2;
    if (threadIdx.x == 0) { mbar_init(&mb2, 1); mbar_fence_init(); }
    __syncthreads();
    const uint32_t sb0 = smem_u32(smem);
    const uint32_t id = idesc_bf16(128, 144, 0, 0);
    if (warp == 0) {
      const uint32_t img = mode == 71 ? 0u : 41472u;
      long long t0 = clock64();
      for (int it = 0; it < iters / 54; ++it) {
        for (int jj = 0; jj < 9; ++jj) {
          const uint32_t a0 = tb + ((jj & 1) ? 96u : 72u);
          uint64_t bd[3];
          for (int j = 0; j < 3; ++j) bd[j] = desc_noswz(sb0 + j * img + jj * 256, 128, 2304);
          if (elect_one()) {
            mma_ts(tb + 264, a0 + 16, bd[0], id, jj > 0);
            mma_ts(tb + 264, a0 + 8, bd[1], id, 1);
            mma_ts(tb + 264, a0, bd[2], id, 1);
            mma_ts(tb + 264, a0 + 8, bd[0], id, 1);
            mma_ts(tb + 264, a0, bd[1], id, 1);
            mma_ts(tb + 264, a0, bd[0], id, 1);
            commit(&mb2);
          }
          __syncwarp();
        }
      }
      if (elect_one()) commit(&mbar);
      __syncwarp();
      mbar_wait(&mbar, 0);
      long long t1 = clock64();
      if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; }
    }
  } else if (mode >= 60) {
    // issue cost under contention: warp 0 issues 6-MMA K-steps (N, TS) while warps 1..(blockDim/32-1)
    // run an FMA/shared-memory busy loop.  mode 60: descriptors carried in registers (+= per step);
    // mode 61: descriptors recomputed from the loop index inside the elected block.
    __shared__ volatile int stop2;
    if (threadIdx.x == 0) stop2 = 0;
    __syncthreads();
    const uint32_t sbb = smem_u32(smem + 32768);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    if (warp == 0) {
      const uint64_t b0 = desc_noswz(sbb, 128, 256);
      uint64_t bd[3] = {b0, b0 + 64, b0 + 128};
      long long t0 = clock64();
      for (int k = 0; k < iters / 6; ++k) {
        if (mode == 60) {
          if (elect_one()) {
            mma_ts(tb + dcol, tb + acol + 16, bd[0], id, k > 0);
            mma_ts(tb + dcol, tb + acol + 8, bd[1], id, 1);
            mma_ts(tb + dcol, tb + acol, bd[2], id, 1);
            mma_ts(tb + dcol, tb + acol + 8, bd[0], id, 1);
            mma_ts(tb + dcol, tb + acol, bd[1], id, 1);
            mma_ts(tb + dcol, tb + acol, bd[0], id, 1);
          }
          __syncwarp();
          for (int j = 0; j < 3; ++j) bd[j] += ((k & 7) == 7) ? (uint64_t)-14 : 2;
        } else {
          if (elect_one()) {
            const uint64_t kk = (uint64_t)(2 * (k & 7));
            mma_ts(tb + dcol, tb + acol + 16, b0 + kk, id, k > 0);
            mma_ts(tb + dcol, tb + acol + 8, b0 + 64 + kk, id, 1);
            mma_ts(tb + dcol, tb + acol, b0 + 128 + kk, id, 1);
            mma_ts(tb + dcol, tb + acol + 8, b0 + kk, id, 1);
            mma_ts(tb + dcol, tb + acol, b0 + 64 + kk, id, 1);
            mma_ts(tb + dcol, tb + acol, b0 + kk, id, 1);
          }
          __syncwarp();
        }
      }
      if (elect_one()) commit(&mbar);
      __syncwarp();
      mbar_wait(&mbar, 0);
      long long t1 = clock64();
      if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; stop2 = 1; }
    } else {
      float a = threadIdx.x, b2 = 1.0001f;
      volatile float* sm = reinterpret_cast<volatile float*>(smem);
      long long n = 0;
      while (!stop2) {
        for (int r = 0; r < 32; ++r) a = a * b2 + 0.5f;
        sm[(threadIdx.x * 4 + (int)n) & 4095] = a;
        ++n;
      }
      if (a == 1.234f) out[1] = n;
    }
  } else if (mode >= 50) {
    // kernel-like B operand: K-major core-matrix image of N rows x Kc cols (SBO = Kc/8*128, LBO = 128),
    // 6 split-pair TS MMAs per K-step, K-step advance = 256 bytes; mode 51: MN-major (LBO = Nc/8*128, SBO = 128)
    const uint32_t sbb = smem_u32(smem);
    const uint32_t id = idesc_bf16(128, N, 0, mode == 51 ? 1 : 0);
    const int Kc = 144;
    if (warp == 0) {
      uint64_t bd[3];
      for (int j = 0; j < 3; ++j)
        bd[j] = mode == 51 ? desc_noswz(sbb + j * 9216, (uint32_t)(N / 8) * 128u, 128)
                           : desc_noswz(sbb + j * 9216, 128, (uint32_t)(Kc / 8) * 128u);
      const uint64_t ks = mode == 51 ? (uint64_t)((2u * (uint32_t)(N / 8) * 128u) >> 4) : (uint64_t)(256 >> 4);
      long long t0 = clock64();
      for (int k = 0; k < iters / 6; ++k) {
        if (elect_one()) {
          mma_ts(tb + dcol, tb + acol + 16, bd[0], id, k > 0);
          mma_ts(tb + dcol, tb + acol + 8, bd[1], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[2], id, 1);
          mma_ts(tb + dcol, tb + acol + 8, bd[0], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[1], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[0], id, 1);
        }
        __syncwarp();
        for (int j = 0; j < 3; ++j) bd[j] += ((k & 7) == 7) ? (uint64_t)0 - 7 * ks : ks;
      }
      if (elect_one()) commit(&mbar);
      __syncwarp();
      mbar_wait(&mbar, 0);
      long long t1 = clock64();
      if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; }
    }
  } else if (mode >= 40) {
    // kernel-pattern probe: 6 TS MMAs (3x3 split pairs) per step, plus optional commit / fence / poll
    __shared__ uint64_t mb2, mb3;
    if (threadIdx.x == 0) { mbar_init(&mb2, 1); mbar_init(&mb3, 1); mbar_fence_init(); mbar_arrive(&mb3); }
    __syncthreads();
    const uint32_t sbb = smem_u32(smem + 32768);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    const int v = mode - 40;
    if (warp == 0) {
      uint64_t bd[3];
      for (int j = 0; j < 3; ++j) bd[j] = desc_noswz(sbb + j * 1024, 128, 256);
      long long t0 = clock64();
      for (int k = 0; k < iters / 6; ++k) {
        if (v & 4) { volatile bool r = mbar_test_warp(&mb3, 0); (void)r; }
        if (v & 2) fence_after();
        if (elect_one()) {
          mma_ts(tb + dcol, tb + acol + 16, bd[0], id, k > 0);
          mma_ts(tb + dcol, tb + acol + 8, bd[1], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[2], id, 1);
          mma_ts(tb + dcol, tb + acol + 8, bd[0], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[1], id, 1);
          mma_ts(tb + dcol, tb + acol, bd[0], id, 1);
          if (v & 1) commit(&mb2);
        }
        __syncwarp();
        for (int j = 0; j < 3; ++j) bd[j] += ((k & 7) == 7) ? (uint64_t)-14 : 2;
      }
      long long t1 = clock64();
      if (elect_one()) commit(&mbar);
      __syncwarp();
      mbar_wait(&mbar, 0);
      long long t2 = clock64();
      if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
  } else if (mode >= 30) {
    // warp 0 issues TS MMAs (D at dcol, A at acol); warps 4..7 generate TMEM traffic meanwhile:
    // mode 30 none, 31 tcgen05.ld x16, 32 tcgen05.st x16, 33 both, +4 shared-memory traffic (warps 4..15)
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    const uint32_t sbb = smem_u32(smem + 32768);
    const uint64_t bd = desc_noswz(sbb, 128, 256);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    const uint64_t adss = desc_noswz(smem_u32(smem), 128, 256);
    if (warp == 0) {
      long long t0 = clock64();
      if (dcol & 0x20000) {   // control: no MMA, just wait iters * 24 cycles
        while (clock64() - t0 < (long long)iters * 24) {
        }
      } else if (dcol & 0x10000) {   // A from shared memory
        for (int k = 0; k < iters; ++k) {
          if (elect_one()) mma_ss(tb + (uint32_t)(dcol & 0xFFFF), adss, bd, id, 1);
          __syncwarp();
        }
      } else {
        for (int k = 0; k < iters; ++k) {
          if (elect_one()) mma_ts(tb + (uint32_t)dcol, tb + (uint32_t)acol, bd, id, 1);
          __syncwarp();
        }
      }
      if (elect_one()) commit(&mbar);
      __syncwarp();
      mbar_wait(&mbar, 0);
      long long t1 = clock64();
      if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; stop = 1; }
    } else if (warp >= 4) {
      const uint32_t ta = tb + ((uint32_t)(32 * (warp & 3)) << 16) + 480u;
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) r[i] = i;
      long long n = 0;
      volatile float* sm = reinterpret_cast<volatile float*>(smem);   // first 32 KB: the A image, unused by TS
      float acc = 0.f;
      while (!stop) {
        if (mode & 1) { tmem_ld<16>(ta, r); tmem_wait_ld(); }
        if (mode & 2) { tmem_st<16>(ta + 16, r); tmem_wait_st(); }
        if (mode & 4) {   // shared-memory traffic: 16 x 128-byte warp loads + stores
          for (int k = 0; k < 16; ++k) {
            acc += sm[(k * 1024 + (threadIdx.x & 31) * 4 + (warp & 3) * 128) & 8191];
            sm[((k * 1024 + (threadIdx.x & 31) * 4 + 4096) & 8191)] = acc;
          }
        }
        ++n;
      }
      if (acc == 1.2345f) out[1] = 0;
      if ((threadIdx.x & 31) == 0 && warp == 4) out[1] = n;
    }
  } else if (mode >= 20) {
    // (mode - 20) issuing warps, each its own accumulator, iters/W MMAs each
    const int W = mode - 20;
    const uint32_t sa = smem_u32(smem), sbb = smem_u32(smem + 32768);
    const uint64_t ad = desc_noswz(sa, 128, 256), bd = desc_noswz(sbb, 128, 256);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    __syncthreads();
    long long t0 = clock64();
    if (warp < W) {
      for (int k = 0; k < iters / W; ++k) {
        if (elect_one()) mma_ss(tb + (uint32_t)(warp * N), ad, bd, id, 1);
        __syncwarp();
      }
      if (elect_one()) commit(&mbar);
      __syncwarp();
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t1 - t0; }
  } else if (mode >= 10 && warp == 0) {
    // whole warp converged, one elected lane issues (the CUTLASS idiom)
    const uint32_t sa = smem_u32(smem), sbb = smem_u32(smem + 32768);
    const uint64_t ad = desc_noswz(sa, 128, 256), bd = desc_noswz(sbb, 128, 256);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
      if (elect_one()) {
        if (mode == 10) mma_ss(tb, ad, bd, id, 1);
        else if (mode == 11) mma_ts(tb, tb + 256, bd, id, 1);
        else mma_ss(tb + (uint32_t)((k & 3) * N), ad, bd, id, 1);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (elect_one()) commit(&mbar);
    __syncwarp();
    mbar_wait(&mbar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (mode < 10 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sbb = smem_u32(smem + 32768);
    const uint64_t ad = desc_noswz(sa, 128, 256), bd = desc_noswz(sbb, 128, 256);
    const uint32_t id = idesc_bf16(128, N, 0, 0);
    long long t0 = clock64();
    if (mode < 2) {
      for (int k = 0; k < iters; ++k) {
        if (mode == 0) mma_ss(tb, ad, bd, id, 1);
        else mma_ts(tb, tb + 256, bd, id, 1);
      }
    } else {
      // round-robin over `nacc` independent accumulators of N columns each
      const int nacc = mode - 1;
      for (int k = 0; k < iters; ++k) mma_ss(tb + (uint32_t)((k % nacc) * N), ad, bd, id, 1);
    }
    long long t1 = clock64();
    commit(&mbar);
    mbar_wait(&mbar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int mma_rate(int mode, int N, int iters, long long* out_host, int dcol, int acol) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int nthr = mode >= 80 ? 32 * (1 + acol) : mode >= 60 ? 32 * (1 + (acol >> 16)) : (mode >= 30 && mode < 40 ? 512 : 256);
  rate_k<<<1, nthr, mode >= 70 ? 200 * 1024 : 64 * 1024>>>(mode, N, iters, d, dcol, acol & 0xFFFF);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(out_host, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}
