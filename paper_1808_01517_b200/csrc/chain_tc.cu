// Fused tensor-core (tcgen05) kernels for the Signal2SH -> LSC -> SH2Signal chain.
//
// Reference path (/root/reference/pkg/src/sphdwi/): fitting.signal_to_sh (fitting.py:206-236) ->
// lsc.lsc_forward (lsc.py:158-199, folded as c_out = L c + bias*beta) ->
// fitting.sh_to_signal (fitting.py:239-250); the backward is the adjoint (SPEC.md:12 leaves it out).
//
// One persistent CTA per SM walks voxel tiles of 128 (= the MMA M dimension), warp-specialised:
//   warp 13      loader: TMA tensor copies (cp.async.bulk.tensor) of 16-channel x 128-voxel blocks into
//                a shared-memory ring.  The input is viewed as pairs of channel rows, so one 3-D tensor
//                map serves any even voxel count; each block is two 8-row boxes (even / odd channels).
//                Shapes the map cannot describe (odd voxel or channel counts, unaligned pointers) fall
//                back to per-warp 4-byte cp.async rings run by the IN warps themselves;
//   warps 0-3    IN: thread t owns voxel t; reads its 16 values, splits each fp32 into PARTS bf16
//                terms and writes them into a TMEM A-operand slot (lane = voxel);
//   warp 12      MMA: one elected lane issues tcgen05.mma kind::f16 (A from TMEM, B = weights
//                from shared memory, fp32 accumulate in TMEM) for every term pair i + j < PARTS;
//   warps 4-11   MID: accumulator -> next stage's A operand (split again), the LSC bias, and the
//                final tcgen05.ld -> coalesced global stores.
// chain3: stage1 (per input group) -> stage2 (all groups, one N <= 256 MMA) -> stage3 (per output
// group).  Forward x -> y uses W1 = M, W2 = L, W3 = B' (+ bias); the adjoint dy -> dx uses the same
// shared-memory images through transposed (MN-major) descriptors.  With enough TMEM the next
// tile's stage 1 is interleaved with this tile's stage 3.
// gram: g = B'^T dy and c = M x on the tensor cores, staged as two-term bf16 SWIZZLE_128B tiles,
// G = sum_v g c^T accumulated in TMEM for the whole CTA, then a float64 finalize dW = <P_k, G>.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace dl {
namespace tc {

using namespace dl::umma;

constexpr int kTileV = 128;                 // voxels per tile (MMA M)
constexpr int kIN = 4;                      // input warps (one per TMEM lane quadrant)
constexpr int kMID = 8;                     // accumulator warps (two per quadrant, alternate columns)
constexpr int kWarpMMA = kIN + kMID;        // 12: MMA issuer, also owns the TMEM allocation
constexpr int kWarpLD = kWarpMMA + 1;       // 13: TMA loader
constexpr int kThreads = (kWarpLD + 1) * 32;
constexpr int kBoxV = kTileV + 4;           // TMA box width: 128 voxels + a 16-byte realignment margin
constexpr int kStageBytes = 16 * kBoxV * 4; // one ring stage: 16 channels x 132 voxels fp32
constexpr int kMaxSlots = 6;
constexpr int kMaxStages = 16;
#ifndef DL_SLEEP_NS
#define DL_SLEEP_NS 0
#endif
constexpr uint32_t kSleepNs = DL_SLEEP_NS;   // back-off between polls of non-MMA roles (0 = spin)

// ---------------------------------------------------------------------------- small helpers
template <int P> struct Pairs;
template <> struct Pairs<3> {   // (i, j): activation term i x weight term j, i + j < 3, small first
  static constexpr int n = 6;
  __device__ static constexpr int i(int k) { return k == 0 ? 2 : k == 1 ? 1 : k == 2 ? 0 : k == 3 ? 1 : 0; }
  __device__ static constexpr int j(int k) { return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 0 : k == 4 ? 1 : 0; }
};
template <> struct Pairs<2> {
  static constexpr int n = 3;
  __device__ static constexpr int i(int k) { return k == 0 ? 1 : 0; }
  __device__ static constexpr int j(int k) { return k == 1 ? 1 : 0; }
};

// Weight-image descriptor (rows x cols bf16, core-matrix blocked, umma.cuh) at K-step 0.
//  kmajor: MN = rows, K = cols;  else: K = rows, MN = cols.  mn0: first MN index (multiple of 8).
__device__ __forceinline__ uint64_t wdesc(uint32_t img, int cols, int kmajor, int mn0) {
  if (kmajor) {
    const uint32_t sbo = (uint32_t)(cols / 8) * 128u;
    return desc_noswz(img + (uint32_t)(mn0 / 8) * sbo, 128u, sbo);
  }
  const uint32_t lbo = (uint32_t)(cols / 8) * 128u;
  return desc_noswz(img + (uint32_t)(mn0 / 8) * 128u, lbo, 128u);
}
// Descriptor advance per K-step of 16 (start-address field, 16-byte units).
__device__ __forceinline__ uint64_t wkstep(int cols, int kmajor) {
  return kmajor ? (uint64_t)(256 >> 4) : (uint64_t)((2u * (uint32_t)(cols / 8) * 128u) >> 4);
}

// All term pairs of one K-step: D (+)= A_i (TMEM, part stride a_part cols) . B_j.
template <int P>
__device__ __forceinline__ void kstep_ts(uint32_t d, uint32_t a0, uint32_t a_part, const uint64_t (&b)[P],
                                         uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < Pairs<P>::n; ++k)
    mma_ts(d, a0 + (uint32_t)Pairs<P>::i(k) * a_part, b[Pairs<P>::j(k)], idesc, (first && k == 0) ? 0u : 1u);
}

// 16 fp32 values of one voxel -> PARTS bf16 terms -> TMEM (8 packed columns per term).
template <int PARTS>
__device__ __forceinline__ void split_store16(uint32_t taddr_part0, uint32_t part_stride_cols, const float (&v)[16]) {
  uint32_t w[PARTS][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t pp[PARTS];
    split_pair<PARTS>(v[2 * i], v[2 * i + 1], pp);
#pragma unroll
    for (int q = 0; q < PARTS; ++q) w[q][i] = pp[q];
  }
#pragma unroll
  for (int q = 0; q < PARTS; ++q) tmem_st<8>(taddr_part0 + (uint32_t)q * part_stride_cols, w[q]);
}

// split only (registers), so the TMEM slot can be awaited after the arithmetic.  H: fp16 terms (the caller
// scaled v by the launch's power of two), else bf16 terms.
template <int PARTS, bool H = false>
__device__ __forceinline__ void split16(const float (&v)[16], uint32_t (&w)[PARTS][8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t pp[PARTS];
    if constexpr (H) split_pair_h<PARTS>(v[2 * i], v[2 * i + 1], pp);
    else split_pair<PARTS>(v[2 * i], v[2 * i + 1], pp);
#pragma unroll
    for (int q = 0; q < PARTS; ++q) w[q][i] = pp[q];
  }
}
template <int PARTS>
__device__ __forceinline__ void store_parts(uint32_t taddr_part0, uint32_t part_stride_cols, const uint32_t (&w)[PARTS][8]) {
#pragma unroll
  for (int q = 0; q < PARTS; ++q) tmem_st<8>(taddr_part0 + (uint32_t)q * part_stride_cols, w[q]);
}

// Delayed scaling of the fp16 path: multiply by the launch's power of two and track the largest magnitude
// (checked after the launch; NaN never raises it, inf does).
template <bool H>
__device__ __forceinline__ void scale16(float (&v)[16], float sc, float& amax) {
  if constexpr (H) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] *= sc;
      amax = fmaxf(amax, fabsf(v[i]));
    }
  }
}
template <bool H>
__device__ __forceinline__ void track16(const float (&v)[16], float& amax) {
  if constexpr (H) {
#pragma unroll
    for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(v[i]));
  }
}

__device__ __forceinline__ void ld16f(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tmem_ld<16>(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 channel rows of one voxel -> HBM (row stride `stride` floats), streaming stores
__device__ __forceinline__ void store16(float* d, int64_t stride, const float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    __stcs(d, v[i]);
    d += stride;
  }
}

__device__ __forceinline__ void st_cs_u32(uint16_t* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u16(uint16_t* p, uint32_t v) {
  asm volatile("st.global.cs.u16 [%0], %1;\n" ::"l"(p), "h"((unsigned short)v) : "memory");
}

// 16 D1 rows of one voxel as their first two bf16 split terms (w0 = hi, w1 = next term, packed row pairs)
// -> the two term planes of the mid buffer (`plane` halfs apart, rows `pitch` apart).  Row `ones` (or -1)
// is stored as exactly 1.0: a zero-weight padding row whose Gram column sums g (the bias gradient).
// row `ones` (0..15; anything else: none) of a lane's packed term words becomes the bias column (1.0, 0)
__device__ __forceinline__ void set_ones(uint32_t (&w0)[8], uint32_t (&w1)[8], int ones) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (2 * i == ones) { w0[i] = (w0[i] & 0xFFFF0000u) | 0x3F80u; w1[i] &= 0xFFFF0000u; }
    if (2 * i + 1 == ones) { w0[i] = (w0[i] & 0x0000FFFFu) | 0x3F800000u; w1[i] &= 0x0000FFFFu; }
  }
}

// ONES = false: the caller has applied set_ones already (or the item has no bias row)
template <bool ONES = true>
__device__ __forceinline__ void store_mid(uint16_t* d, int64_t plane, int64_t pitch, const uint32_t (&w0)[8],
                                          const uint32_t (&w1)[8], int ones) {
  // Lanes (2j, 2j+1) hold adjacent voxels: they trade their packed row pairs so that the even lane stores
  // row 2i and the odd lane row 2i+1 of both voxels as one 32-bit word -- half the store instructions of
  // per-voxel 16-bit stores.  Callers are warp-uniform (whole warps inside or outside the mid buffer).
  const uint32_t odd = threadIdx.x & 1u;
  uint16_t* base = d - odd;   // the pair's first voxel (4-byte aligned: tiles are 64 voxels)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t a = w0[i], c = w1[i];
    if (ONES && 2 * i == ones) { a = (a & 0xFFFF0000u) | 0x3F80u; c &= 0xFFFF0000u; }
    if (ONES && 2 * i + 1 == ones) { a = (a & 0x0000FFFFu) | 0x3F800000u; c &= 0x0000FFFFu; }
    const uint32_t pa = __shfl_xor_sync(0xffffffffu, a, 1), pc = __shfl_xor_sync(0xffffffffu, c, 1);
    const uint32_t sel_lo = odd ? 0x7632u : 0x5410u;
    const uint32_t wa = odd ? __byte_perm(pa, a, sel_lo) : __byte_perm(a, pa, sel_lo);
    const uint32_t wc = odd ? __byte_perm(pc, c, sel_lo) : __byte_perm(c, pc, sel_lo);
    uint16_t* r = base + (int64_t)(2 * i + (int)odd) * pitch;
    st_cs_u32(r, wa);
    st_cs_u32(r + plane, wc);
  }
}

__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// Waits of roles off the critical path (IN ahead of the MMA, OUT between drains) can back off so their
// polling does not take issue slots from the MMA warp on the same scheduler (DL_IDLE_NS, 0 = spin).
#ifndef DL_IDLE_NS
#define DL_IDLE_NS 0
#endif
#ifndef DL_IDLE_MASK
#define DL_IDLE_MASK 3   // bit 0: IN waits, bit 1: OUT waits
#endif
#ifndef DL_SUSPEND_NS
#define DL_SUSPEND_NS 0
#endif
template <int ROLE>
__device__ __forceinline__ void idle_wait(uint64_t* bar, uint32_t parity) {
  if (DL_SUSPEND_NS > 0) mbar_wait_suspend(bar, parity, DL_SUSPEND_NS);
  else if (DL_IDLE_NS > 0 && (DL_IDLE_MASK & (1 << ROLE))) mbar_wait_sleep(bar, parity, DL_IDLE_NS);
  else mbar_wait_warp(bar, parity);
}

// wait used by the IN / CONV / OUT / loader roles (the MMA warps keep mbar_wait_warp)
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity) {
  if (DL_SUSPEND_NS > 0) mbar_wait_suspend(bar, parity, DL_SUSPEND_NS);
  else if (kSleepNs) mbar_wait_sleep(bar, parity, kSleepNs);
  else mbar_wait_warp(bar, parity);
}

// byte offset of (row j, voxel k) in a SWIZZLE_128B K-major tile with `rows` rows (K = 128 voxels)
__device__ __forceinline__ uint32_t sw128_off(int j, int k, int rows) {
  return (uint32_t)(k >> 6) * (uint32_t)(rows >> 3) * 1024u + (uint32_t)(j >> 3) * 1024u + (uint32_t)(j & 7) * 128u +
         (uint32_t)((((k & 63) >> 3) ^ (j & 7)) << 4) + (uint32_t)(k & 7) * 2u;
}

// 16 rows (channels) of one voxel via 4-byte cp.async: rows < nval copy, the rest are zero-filled.
__device__ __forceinline__ void stream_chunk(float* dst, const float* src, int64_t stride, int nval,
                                             const float* dummy) {
  if (nval >= 16) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      cp_async4(dst + r * 32, src, 4u);
      src += stride;
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const bool valid = r < nval;
      cp_async4(dst + r * 32, valid ? src : dummy, valid ? 4u : 0u);
      src += stride;
    }
  }
}

// Hands one voxel's 16 values (split into PARTS bf16 terms) to the MMA warp through TMEM A slot
// (aslot, around), then advances the slot cursor by `step` chunks.
template <int PARTS, bool H = false>
__device__ __forceinline__ void put_a(const float (&v)[16], uint32_t tslots, int NA, uint64_t* a_full,
                                      uint64_t* a_empty, uint32_t& aslot, uint32_t& around, int step = 1) {
  uint32_t w[PARTS][8];
  split16<PARTS, H>(v, w);
  if (around > 0) idle_wait<0>(&a_empty[aslot], (around - 1) & 1);
  fence_after();
  store_parts<PARTS>(tslots + aslot * (PARTS * 8), 8, w);
  tmem_wait_st();
  fence_before();
  warp_arrive(&a_full[aslot]);
  aslot += step;
  while (aslot >= (uint32_t)NA) {
    aslot -= NA;
    ++around;
  }
}

// Chunk r of a tile (the geometry functor): which input tensor, its first channel, and how many of
// the 16 rows are real channels of the current group (the rest are zeroed).
struct ChunkGeo {
  int tensor, c0, nval;
};

// Fallback IN role (no tensor map): each warp streams its own 32-voxel segment of its chunks
// q = iw, iw + nIW, ... through a private NS-deep ring with 4-byte cp.async (any alignment).  Every
// thread only reads back what it copied itself, so cp.async.wait_group is the only synchronisation.
template <int PARTS, int NS, typename Geo, bool H = false>
__device__ __forceinline__ void in_role_cpasync(const Geo& geo, int per_tile, int64_t ntiles, int64_t tiles_per_b,
                                                int64_t nvox, const float* const (&base)[2], const int64_t (&bs)[2],
                                                uint32_t tslots, int NA, uint64_t* a_full, uint64_t* a_empty,
                                                float* ring, int iw = 0, int nIW = 1, float sc = 1.f,
                                                float* amax = nullptr) {
  float am = 0.f;
  const int qd = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int64_t nmine = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * per_tile;
  int64_t qp = iw;
  uint32_t pslot = 0, cslot = 0, aslot = (uint32_t)(iw % NA), around = (uint32_t)(iw / NA);
  auto issue = [&]() {
    if (qp < total) {
      const int64_t ti = qp / per_tile;
      const int r = (int)(qp - ti * per_tile);
      const int64_t t = blockIdx.x + ti * gridDim.x, b = t / tiles_per_b;
      const int64_t v = (t - b * tiles_per_b) * kTileV + 32 * qd + lane;
      const ChunkGeo cg = geo(r);
      const bool vok = v < nvox;
      const float* src = base[cg.tensor] + b * bs[cg.tensor] + (int64_t)cg.c0 * nvox + (vok ? v : 0);
      stream_chunk(ring + pslot * 512 + lane, src, nvox, vok ? cg.nval : 0, base[0]);
      qp += nIW;
    }
    cp_async_commit();
    pslot = pslot + 1 == NS ? 0 : pslot + 1;
  };
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) issue();
  for (int64_t q = iw; q < total; q += nIW) {
    issue();
    cp_async_wait<NS - 1>();
    float v[16];
    const float* rp = ring + cslot * 512 + lane;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = rp[r * 32];
    cslot = cslot + 1 == NS ? 0 : cslot + 1;
    scale16<H>(v, sc, am);
    put_a<PARTS, H>(v, tslots, NA, a_full, a_empty, aslot, around, nIW);
  }
  cp_async_wait<0>();
  if (H) *amax = fmaxf(*amax, am);
}

// IN role over a RAW acquisition (b0 normalisation folded into the chain's input):
// channel c of the chain input is stored volume sel[c] of the acquisition (volumes `vstride` elements apart,
// voxels in the acquisition's stored order), in its stored type T (int16 or fp32), and
//   x[c][v] = raw[sel[c]][v] * vox_a[v] + vox_b[v]
// with vox_a = slope / mean_b0, vox_b = inter / mean_b0 (0 for excluded voxels) -- fitting.normalize_b0
// (fitting.py:253-342) applied on the fly, so the normalised volume never exists in HBM.  One warp per lane
// quadrant; each warp streams its 32 voxels of every chunk through a private NS-deep shared-memory ring with
// cp.async (two voxels per lane, two rows per instruction: 16 rows x 32 voxels per stage), NS - 1 chunks ahead.
// Needs an even vstride and T-aligned rows (checked on the host).
template <int PARTS, int NS, typename T, typename Geo, bool H = false>
__device__ __forceinline__ void in_role_raw(const Geo& geo, int per_tile, int64_t ntiles, int64_t tiles_per_b,
                                            int64_t nvox, const T* raw, int64_t vstride, const int* sel,
                                            const float* vox_a, const float* vox_b, uint32_t tslots, int NA,
                                            uint64_t* a_full, uint64_t* a_empty, T* ring, int iw, int nIW,
                                            float sc = 1.f, float* amax = nullptr) {
  constexpr int kV = 2 * (int)sizeof(T);   // bytes per lane per copy (two voxels)
  const int qd = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31, pv = 2 * (lane & 15), half = lane >> 4;
  const int64_t nmine = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * per_tile;
  float am = 0.f;
  int64_t qp = iw;   // this warp's chunks: iw, iw + nIW, ...
  uint32_t pslot = 0, cslot = 0, aslot = (uint32_t)(iw % NA), around = (uint32_t)(iw / NA);
  auto issue = [&]() {
    __syncwarp();   // every lane has read the stage this copy refills (lanes read each other's copies)
    if (qp < total) {
      const int64_t ti = qp / per_tile;
      const int r = (int)(qp - ti * per_tile);
      const int64_t t = blockIdx.x + ti * gridDim.x, b = t / tiles_per_b;
      const int64_t v = (t - b * tiles_per_b) * kTileV + 32 * qd + pv;
      const ChunkGeo cg = geo(r);
      const int nval = cg.nval < 16 ? cg.nval : 16;
      const int vsel = lane < nval ? __ldg(sel + cg.c0 + lane) : 0;   // lane j < 16 holds row j's volume
      const uint32_t nb = v + 1 < nvox ? (uint32_t)kV : v < nvox ? (uint32_t)sizeof(T) : 0u;
      T* dst = ring + pslot * 512 + pv;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = 2 * i + half;
        const int vol = __shfl_sync(0xffffffffu, vsel, row);
        const bool ok = row < nval && nb;
        const T* src = ok ? raw + (int64_t)vol * vstride + v : raw;
        if constexpr (kV == 8) cp_async8(dst + row * 32, src, ok ? nb : 0u);
        else cp_async4(dst + row * 32, src, ok ? nb : 0u);
      }
      qp += nIW;
    }
    cp_async_commit();
    pslot = pslot + 1 == NS ? 0 : pslot + 1;
  };
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) issue();
  int64_t cur_t = -1;
  float a = 0.f, bb = 0.f;
  for (int64_t q = iw; q < total; q += nIW) {
    issue();
    cp_async_wait<NS - 1>();
    __syncwarp();   // the stage holds every lane's copies
    const int64_t ti = q / per_tile;
    const int r = (int)(q - ti * per_tile);
    if (ti != cur_t) {   // this thread's voxel factors for the tile
      cur_t = ti;
      const int64_t t = blockIdx.x + ti * gridDim.x, b = t / tiles_per_b;
      const int64_t v = (t - b * tiles_per_b) * kTileV + 32 * qd + lane;
      a = v < nvox ? __ldg(vox_a + b * nvox + v) : 0.f;
      bb = v < nvox ? __ldg(vox_b + b * nvox + v) : 0.f;
    }
    const int nval = geo(r).nval;
    const T* rp = ring + cslot * 512 + lane;
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = j < nval ? fmaf((float)rp[j * 32], a, bb) : 0.f;
    cslot = cslot + 1 == NS ? 0 : cslot + 1;
    scale16<H>(x, sc, am);
    put_a<PARTS, H>(x, tslots, NA, a_full, a_empty, aslot, around, nIW);
  }
  cp_async_wait<0>();
  if (H) *amax = fmaxf(*amax, am);
}

// TMA loader (one warp, one elected lane issues): chunk (tile, r) -> ring stage, as two 8 x 132 boxes of
// the channel-pair view (even channels first, then odd).  A box must start 16-byte aligned in global
// memory; odd channel rows start at voxel offset nvox, so when nvox % 4 == 2 their box starts 2 voxels
// early (shift) and the readers skip those.
template <int NS, typename Geo>
__device__ __forceinline__ void tma_loader(const Geo& geo, int per_tile, int64_t ntiles, int64_t tiles_per_b,
                                           int64_t nvox, const CUtensorMap* maps, uint8_t* ring, uint64_t* full,
                                           uint64_t* empty) {
  if (elect_one()) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(maps) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(maps + 1) : "memory");
  }
  __syncwarp();
  uint32_t s = 0, round = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const int v0 = (int)((t - b * tiles_per_b) * kTileV);
    for (int r = 0; r < per_tile; ++r) {
      const ChunkGeo cg = geo(r);
      if (round > 0) role_wait(&empty[s], (round - 1) & 1);
      if (elect_one()) {
        uint8_t* dst = ring + s * kStageBytes;
        mbar_arrive_tx(&full[s], kStageBytes);
        tma_load_3d(dst, maps + cg.tensor, v0, cg.c0 >> 1, (int)b, &full[s]);
        tma_load_3d(dst + kStageBytes / 2, maps + cg.tensor, (int)nvox + v0 - (int)(nvox & 3), cg.c0 >> 1, (int)b,
                    &full[s]);
      }
      __syncwarp();
      if (++s == NS) {
        s = 0;
        ++round;
      }
    }
  }
}

// IN role over the TMA ring: thread = voxel; row j of the chunk is channel-pair row j/2 of box j%2.
// This warp takes chunks q = iw, iw + nIW, ... (nIW a power of two).
template <int PARTS, int NS, typename Geo, bool H = false>
__device__ __forceinline__ void in_role_tma(const Geo& geo, int per_tile, int64_t ntiles, int64_t tiles_per_b,
                                            int64_t nvox, uint32_t tslots, int NA, uint64_t* a_full, uint64_t* a_empty,
                                            const float* ring, uint64_t* full, uint64_t* empty, int iw = 0,
                                            int nIW = 1, float sc = 1.f, float* amax = nullptr) {
  float am = 0.f;
  const int qd = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int odd0 = 8 * kBoxV + (int)(nvox & 3);   // first odd-channel value of this thread, minus its voxel
  uint32_t s = 0, round = 0, aslot = (uint32_t)(iw % NA), around = (uint32_t)(iw / NA);
  uint32_t q = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const bool vok = (t - b * tiles_per_b) * kTileV + 32 * qd + lane < nvox;
    for (int r = 0; r < per_tile; ++r, ++q) {
      const uint32_t cs = s;
      const uint32_t cround = round;
      if (++s == NS) {
        s = 0;
        ++round;
      }
      if ((q & (uint32_t)(nIW - 1)) != (uint32_t)iw) continue;
      const ChunkGeo cg = geo(r);
      const int nval = vok ? cg.nval : 0;   // voxels past nvox read neighbouring-row data: zero them
      idle_wait<0>(&full[cs], cround & 1);
      const float* rp = ring + cs * (kStageBytes / 4) + 32 * qd + lane;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = j < nval ? rp[(j & 1) * odd0 + (j >> 1) * kBoxV] : 0.f;
      warp_arrive(&empty[cs]);
      scale16<H>(v, sc, am);
      put_a<PARTS, H>(v, tslots, NA, a_full, a_empty, aslot, around, nIW);
    }
  }
  if (H) *amax = fmaxf(*amax, am);
}

// IN role, two chunks per TMEM item (one handoff per two K-steps): warp iw of a lane quadrant takes
// the chunk pairs p = iw, iw + 2, ...; chunk q lives in ring stage q % NS (NS % 4 == 0: every stage
// keeps one fixed consumer warp).  Pairs never straddle an input group (chunks per group is even).
template <int PARTS, int NS, typename Geo, bool H = false>
__device__ __forceinline__ void in_role_tma2(const Geo& geo, int per_tile, int64_t ntiles, int64_t tiles_per_b,
                                             int64_t nvox, uint32_t tslots, int NA, uint64_t* a_full,
                                             uint64_t* a_empty, const float* ring, uint64_t* full, uint64_t* empty,
                                             int iw, float sc = 1.f, float* amax = nullptr) {
  float am = 0.f;
  static_assert(NS % 4 == 0, "two-chunk IN items need NS % 4 == 0");
  const int qd = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int odd0 = 8 * kBoxV + (int)(nvox & 3);
  uint32_t aslot = (uint32_t)(iw % NA), around = (uint32_t)(iw / NA);
  uint32_t pr = 0;   // CTA-wide pair index
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / tiles_per_b;
    const bool vok = (t - b * tiles_per_b) * kTileV + 32 * qd + lane < nvox;
    for (int r = 0; r < per_tile; r += 2, ++pr) {
      if ((pr & 1u) != (uint32_t)iw) continue;
      const uint32_t q0 = 2 * pr, cs0 = q0 % NS, cs1 = (q0 + 1) % NS;
      const ChunkGeo cg = geo(r);
      const int nval0 = vok ? cg.nval : 0, nval1 = vok ? cg.nval - 16 : 0;
      const uint32_t ta = tslots + aslot * (2 * PARTS * 8);
#if DL_IN_SEQ
      // the two chunks one after the other: 16 values and their terms live at a time (register budget)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t cs = h ? cs1 : cs0;
        const int nv = h ? nval1 : nval0;
        float v[16];
        idle_wait<0>(&full[cs], ((q0 + h) / NS) & 1);
        const float* rp = ring + cs * (kStageBytes / 4) + 32 * qd + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = j < nv ? rp[(j & 1) * odd0 + (j >> 1) * kBoxV] : 0.f;
        warp_arrive(&empty[cs]);
        scale16<H>(v, sc, am);
        uint32_t w[PARTS][8];
        split16<PARTS, H>(v, w);
        if (h == 0) {
          if (around > 0) idle_wait<0>(&a_empty[aslot], (around - 1) & 1);
          fence_after();
        }
        store_parts<PARTS>(ta + (uint32_t)h * PARTS * 8, 8, w);
      }
#else
      float v0[16], v1[16];
      // a full chunk (every row valid) reads without per-row predicates: two row bases, immediate offsets
      auto ld_chunk = [&](float (&v)[16], const float* rp, int nv) {
        if (nv >= 16) {
          const float* re = rp;
          const float* ro = rp + odd0;
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            v[j] = re[(j >> 1) * kBoxV];
            v[j + 1] = ro[(j >> 1) * kBoxV];
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = j < nv ? rp[(j & 1) * odd0 + (j >> 1) * kBoxV] : 0.f;
        }
      };
      idle_wait<0>(&full[cs0], (q0 / NS) & 1);
      ld_chunk(v0, ring + cs0 * (kStageBytes / 4) + 32 * qd + lane, nval0);
      warp_arrive(&empty[cs0]);
      idle_wait<0>(&full[cs1], ((q0 + 1) / NS) & 1);
      ld_chunk(v1, ring + cs1 * (kStageBytes / 4) + 32 * qd + lane, nval1);
      warp_arrive(&empty[cs1]);
      scale16<H>(v0, sc, am);
      scale16<H>(v1, sc, am);
      uint32_t w0[PARTS][8], w1[PARTS][8];
      split16<PARTS, H>(v0, w0);
      split16<PARTS, H>(v1, w1);
      if (around > 0) idle_wait<0>(&a_empty[aslot], (around - 1) & 1);
      fence_after();
      store_parts<PARTS>(ta, 8, w0);
      store_parts<PARTS>(ta + PARTS * 8, 8, w1);
#endif
      tmem_wait_st();
      fence_before();
      warp_arrive(&a_full[aslot]);
      aslot += 2;
      while (aslot >= (uint32_t)NA) {
        aslot -= NA;
        ++around;
      }
    }
  }
  if (H) *amax = fmaxf(*amax, am);
}

// ============================================================================ chain3 kernel
struct Chain3 {
  CUtensorMap tm[2];                  // channel-pair view of `in` (tm[1] unused)
  const float* in;
  float* out;
  uint16_t* mid;                      // optional: stage-1 accumulator D1 -> HBM as two bf16 term planes,
                                      // tiled [b][64-voxel tile][term][row][64] (one contiguous Gram tile)
  int64_t mid_pitch;                  // voxels per mid row (nvox rounded up to 64)
  int mid_ones;                       // D1 row stored as 1.0 (a padding row; the Gram's bias column) or -1
  const float* bias2;                 // real stage-2 bias per (group, channel < C2) or null
  const uint16_t* w1;                 // images, part-major: (q * groups + g) * img_bytes
  const uint16_t* w2;
  const uint16_t* w3;
  int64_t nbatch, nvox, in_bs, out_bs, mid_bs, tiles_per_b;
  int G1, C1, K1, N1;                 // stage 1: groups, real in-ch/group, padded K, padded N
  int G2, C2, N2;                     // stage 2: groups, real out-ch/group, padded N
  int C3, N3;                         // stage 3: real / padded out-ch per group
  int w1_groups, w3_groups;
  int adjoint, overlap, free_at, tma;
  int NA, ns;                         // TMEM A slots (IN items), ring depth
  int cpi;                            // chain3v: input chunks per IN item (1 or 2; a 2-chunk item is one
                                      // handoff for two K-steps)
  int NAc;                            // chain3v: conversion-ring slots
  int t_diag;                         // chain2h: T block-diagonal over shells (round trip, L = I): output shell o
                                      // reads only input group o's A2 items (the 12-stage instantiation; the
                                      // others run the dense T, exact as well)
  uint32_t colC;                      // chain3v: conversion ring (A operands of stages 2 and 3)
  uint32_t w1_img, w2_img, w3_img;    // bytes per image
  uint32_t sm_w1, sm_w2, sm_w3, sm_bias, sm_ring, sm_bar, smem_bytes;
  uint32_t colA, colD1, colA2, colD2, colA3, colD3;
  long long* prof;                    // debug: per-role phase timestamps of CTA 0 (dl_debug_chain_prof)
  int tstream;                        // chain2h: stream each output shell's T image from L2 into two buffers
  const float* target;                // fused MSE: out = out_scale * (y - target), loss[redo] += sum (y - t)^2
  float out_scale;
  double* loss;
  uint32_t* rstate;                   // chain3v delayed-scaling state (kState* words) or null
  int redo;                           // chain3v bf16 pass: check the fp16 pass's ranges, recompute if needed
  dl::KTrace* kt;                     // kernel timer (dl_ktimer_*) or null, and its slot
  int kt_slot;
  uint32_t sm_tring;                  // chain2h fused MSE: per-OUT-warp target rings (2 x 16 x 32 fp32), or 0
  const void* raw;                    // chain3v raw-acquisition input (in_role_raw) or null
  int raw_type;                       // NIfTI datatype code of raw: 4 int16, 16 float32
  int64_t raw_vstride;                // elements between stored volumes
  const int* raw_sel;                 // stored volume of each chain input channel (device)
  const float* vox_a;                 // per-voxel slope / mean_b0 and inter / mean_b0 (stored order)
  const float* vox_b;
};

// Delayed scaling of the fp16 chain (state words, caller-owned, zero-initialised):
//   the fp16 pass multiplies its input by 2^exp, records the largest scaled input magnitude (amax_in) and
//   the largest scaled accumulator it converts (amax_mid); the bf16 pass launched right after checks them:
//   in range -> every CTA exits at once; out of range -> it recomputes everything with 3-term bf16 operands
//   (no range limits).  Its last CTA re-centres exp on the measured magnitudes and clears the words.
enum : int { kStExp = 0, kStAmaxIn, kStAmaxMid, kStArrive, kStRedos, kStChecks, kStLastRedo, kStateWords = 8 };
__device__ __forceinline__ bool range_ok(float ai, float am) {
  // fp16: max 65504, 2^-24 subnormal spacing.  ai >= 2^-2 keeps the absolute rounding floor (2^-25) below
  // 2^-23 of the largest input; <= 2^14 leaves headroom for the split terms and the accumulators.
  return ai >= 0.25f && ai <= 16384.f && am <= 16384.f;
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// the check of the bf16 pass (thread 0 of each CTA); true: the fp16 pass's results stand
__device__ __forceinline__ bool range_check(uint32_t* st) {
  volatile uint32_t* v = st;
  const float ai = __uint_as_float(v[kStAmaxIn]), am = __uint_as_float(v[kStAmaxMid]);
  const bool ok = range_ok(ai, am);
  __threadfence();
  if (atomicAdd(st + kStArrive, 1u) == gridDim.x - 1) {   // last CTA: every CTA has read the verdict
    __threadfence();
    int e = (int)v[kStExp];
    if (ai > 0.f && ai <= 3.0e38f) {   // re-centre: largest input near 2^8, accumulators below 2^12
      int k;
      frexpf(ai, &k);                  // ai in [2^(k-1), 2^k)
      int d = 8 - k;
      if (am > 0.f && am <= 3.0e38f) {
        int km;
        frexpf(am, &km);
        if (km + d > 12) d = 12 - km;
      }
      e += d;
      e = e < -100 ? -100 : e > 100 ? 100 : e;
    }
    v[kStExp] = (uint32_t)e;
    v[kStAmaxIn] = 0u;
    v[kStAmaxMid] = 0u;
    v[kStArrive] = 0u;
    if (!ok) v[kStRedos] = v[kStRedos] + 1u;
    v[kStLastRedo] = ok ? 0u : 1u;   // which pass's results (and loss) stand for this call
    v[kStChecks] = v[kStChecks] + 1u;
    __threadfence();
  }
  return ok;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

// warp sum of the squared residuals -> one float64 atomic per warp (fused MSE)
__device__ __forceinline__ void loss_publish(double* acc, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, v);
}

__device__ __forceinline__ void amax_publish(uint32_t* word, float am) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  if ((threadIdx.x & 31) == 0) atomicMax(word, __float_as_uint(am));
}

// role r < 8 (chain3v: see scripts/prof_chain_phases.py), tile it < 8, event ev < 32
// Phase timestamps are compiled in only with -DDL_PROFILE (scripts/prof_chain_phases.py): the checks cost
// measurable time in the conversion roles.
#ifdef DL_PROFILE
#define DL_PROF(r, ev)                                                                   \
  do {                                                                                   \
    if (p.prof && blockIdx.x == 0 && it < 8 && (threadIdx.x & 31) == 0)                  \
      p.prof[((it)*8 + (r)) * 32 + (ev)] = clock64();                                    \
  } while (0)
#else
#define DL_PROF(r, ev) \
  do {                 \
  } while (0)
#endif

struct Bars3 {
  uint64_t full[kMaxStages], empty[kMaxStages];   // TMA ring
  uint64_t a_full[kMaxSlots], a_empty[kMaxSlots];
  uint64_t d1_full, d1_free, ac_full, u_full, au_full, y_full;
  uint32_t tmem_base;
};

template <int PARTS, int NS>
__global__ void __launch_bounds__(kThreads, 1) chain3_tc(const __grid_constant__ Chain3 p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars3& bars = *reinterpret_cast<Bars3*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kSlotW = PARTS * 8;

  {  // stage weight images + bias once per CTA
    const uint32_t b1 = (uint32_t)PARTS * p.w1_groups * p.w1_img, b2 = (uint32_t)PARTS * p.w2_img,
                   b3 = (uint32_t)PARTS * p.w3_groups * p.w3_img;
    const uint4 *s1 = reinterpret_cast<const uint4*>(p.w1), *s2 = reinterpret_cast<const uint4*>(p.w2),
                *s3 = reinterpret_cast<const uint4*>(p.w3);
    uint4 *d1 = reinterpret_cast<uint4*>(smem + p.sm_w1), *d2 = reinterpret_cast<uint4*>(smem + p.sm_w2),
          *d3 = reinterpret_cast<uint4*>(smem + p.sm_w3);
    for (uint32_t i = threadIdx.x; i < b1 / 16; i += blockDim.x) d1[i] = __ldg(s1 + i);
    for (uint32_t i = threadIdx.x; i < b2 / 16; i += blockDim.x) d2[i] = __ldg(s2 + i);
    for (uint32_t i = threadIdx.x; i < b3 / 16; i += blockDim.x) d3[i] = __ldg(s3 + i);
    float* sb = reinterpret_cast<float*>(smem + p.sm_bias);
    for (int i = threadIdx.x; i < p.G2 * p.N2; i += blockDim.x) {
      const int o = i / p.N2, r = i - o * p.N2;
      sb[i] = (p.bias2 && r < p.C2) ? __ldg(p.bias2 + o * p.C2 + r) : 0.f;
    }
  }
  if (warp == kWarpMMA) tmem_alloc(&bars.tmem_base, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], kIN);
    }
    for (int s = 0; s < p.NA; ++s) {
      mbar_init(&bars.a_full[s], 4);   // one arrival per TMEM lane quadrant
      mbar_init(&bars.a_empty[s], 1);
    }
    mbar_init(&bars.d1_full, 1);
    mbar_init(&bars.d1_free, kMID);
    mbar_init(&bars.ac_full, kMID);
    mbar_init(&bars.u_full, 1);
    mbar_init(&bars.au_full, kMID);
    mbar_init(&bars.y_full, 1);
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;
  const int nk1 = p.K1 / 16;
  const int per_tile = p.G1 * nk1;
  auto geo = [&](int r) {
    const int g = r / nk1, k = r - g * nk1;
    return ChunkGeo{0, g * p.C1 + 16 * k, p.C1 - 16 * k};
  };

  if (warp < kIN) {
    // =========================== IN: ring -> split -> TMEM A slots ===========================
    const uint32_t tslots = tbase + ((uint32_t)(32 * warp) << 16) + p.colA;
    if (p.tma) {
      in_role_tma<PARTS, NS>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, tslots, p.NA, bars.a_full, bars.a_empty,
                             reinterpret_cast<const float*>(smem + p.sm_ring), bars.full, bars.empty);
    } else {
      const float* const base[2] = {p.in, p.in};
      const int64_t bs[2] = {p.in_bs, p.in_bs};
      in_role_cpasync<PARTS, NS>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, base, bs, tslots, p.NA, bars.a_full,
                                 bars.a_empty, reinterpret_cast<float*>(smem + p.sm_ring) + warp * NS * 512);
    }
  } else if (warp < kWarpMMA) {
    // =========================== MID: D1 -> A2, D2 (+bias) -> A3, D3 -> HBM ===========================
    // two warps per TMEM lane quadrant, alternate 16-column chunks
    const int mw = warp - kIN, qd = mw & 3, cg = mw >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int row = 32 * qd + lane;
    const float* sb = reinterpret_cast<const float*>(smem + p.sm_bias);
    const int D1w = p.G1 * p.N1;
    const int64_t stride = p.nvox;
    // stage-3 buffers inside the A2 region: every MID warp must be done reading the last D3 before any
    // warp overwrites A2 with the next tile
    const bool s3_in_a2 = p.colA3 < p.colA2 + (uint32_t)(PARTS * D1w / 2) && p.colD3 + p.N3 > p.colA2;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int64_t b = t / p.tiles_per_b, v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool vok = v < p.nvox;
      if (mw == 0) DL_PROF(1, 0);
      if (it > 0 && s3_in_a2) named_sync(1, kMID * 32);
      mbar_wait_warp(&bars.d1_full, it & 1);
      if (mw == 0) DL_PROF(1, 1);
      fence_after();
      for (int ck = cg; ck < D1w / 16; ck += 2) {
        float vv[16];
        ld16f(tq + p.colD1 + (uint32_t)ck * 16, vv);
        uint32_t w[PARTS][8];
        split16<PARTS>(vv, w);
        if (p.mid && v < p.mid_pitch)
          store_mid(p.mid + ((b * (p.mid_pitch >> 6) + (v >> 6)) * 2 * D1w + 16 * ck) * 64 + (v & 63),
                    (int64_t)D1w * 64, 64, w[0], w[1], vok ? p.mid_ones - 16 * ck : -1);
        store_parts<PARTS>(tq + p.colA2 + (uint32_t)ck * 8, D1w / 2, w);
      }
      tmem_wait_st();
      fence_before();
      warp_arrive(&bars.ac_full);
      if (p.free_at == 0) warp_arrive(&bars.d1_free);
      if (mw == 0) DL_PROF(1, 2);
      mbar_wait_warp(&bars.u_full, it & 1);
      if (mw == 0) DL_PROF(1, 3);
      fence_after();
      for (int o = 0; o < p.G2; ++o) {
        // A3 of group o (the MMA finished reading A3 of group o-1: this warp waited y_full below)
        for (int ck = cg; ck < p.N2 / 16; ck += 2) {
          float vv[16];
          ld16f(tq + p.colD2 + (uint32_t)(o * p.N2 + ck * 16), vv);
#pragma unroll
          for (int i = 0; i < 16; ++i) vv[i] += sb[o * p.N2 + ck * 16 + i];
          split_store16<PARTS>(tq + p.colA3 + (uint32_t)ck * 8, p.N2 / 2, vv);
        }
        tmem_wait_st();
        fence_before();
        warp_arrive(&bars.au_full);   // also: this warp has drained D3 of group o-1
        if (p.free_at == 1 && o == p.G2 - 1) warp_arrive(&bars.d1_free);   // D2 (aliasing D1) fully read
        if (mw == 0) DL_PROF(1, 4 + 3 * o);
        mbar_wait_warp(&bars.y_full, (it * p.G2 + o) & 1);
        if (mw == 0) DL_PROF(1, 5 + 3 * o);
        fence_after();
        for (int ck = cg; ck < p.N3 / 16; ck += 2) {
          float vv[16];
          ld16f(tq + p.colD3 + (uint32_t)ck * 16, vv);
          if (vok && p.out) {   // out == null: a g-only adjoint (no dx)
            float* d = p.out + b * p.out_bs + ((int64_t)o * p.C3 + ck * 16) * stride + v;
            const int nval = p.C3 - ck * 16;
            if (nval >= 16) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                __stcs(d, vv[i]);
                d += stride;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (i < nval) __stcs(d, vv[i]);
                d += stride;
              }
            }
          }
        }
        if (mw == 0) DL_PROF(1, 6 + 3 * o);
      }
      fence_before();
      if (p.free_at == 2) warp_arrive(&bars.d1_free);   // stage-3 buffers (inside D1) fully read
    }
  } else if (warp == kWarpMMA) {
    // =========================== MMA issuer (converged warp, one elected lane issues) ===========
    const uint32_t sw1 = smem_u32(smem + p.sm_w1), sw2 = smem_u32(smem + p.sm_w2), sw3 = smem_u32(smem + p.sm_w3);
    const int km = p.adjoint ? 0 : 1;   // forward: K-major weights; adjoint: MN-major
    const int K2 = p.G1 * p.N1, NT2 = p.G2 * p.N2;
    const bool merge2 = NT2 <= 256;
    const uint32_t id1 = idesc_bf16(128, p.N1, 0, 1 - km);
    const uint32_t id2 = idesc_bf16(128, merge2 ? NT2 : p.N2, 0, 1 - km);
    const uint32_t id3 = idesc_bf16(128, p.N3, 0, 1 - km);
    const int c1 = km ? p.K1 : p.N1, c2 = km ? K2 : NT2, c3 = km ? p.N2 : p.N3;
    const uint64_t ks1 = wkstep(c1, km), ks2 = wkstep(c2, km), ks3 = wkstep(c3, km);
    uint32_t aslot = 0, around = 0, n_au = 0;
    // one stage-1 K-step (chunk k of group g); the caller made sure its A slot is full
    auto s1_chunk = [&](int g, int k) {
      const int wg = p.w1_groups > 1 ? g : 0;
      uint64_t bd[PARTS];
#pragma unroll
      for (int j = 0; j < PARTS; ++j)
        bd[j] = wdesc(sw1 + (uint32_t)(j * p.w1_groups + wg) * p.w1_img, c1, km, 0) + (uint64_t)k * ks1;
      fence_after();
      if (elect_one()) {
        kstep_ts<PARTS>(tbase + p.colD1 + (uint32_t)(g * p.N1), tbase + p.colA + aslot * kSlotW, 8, bd, id1, k == 0);
        commit(&bars.a_empty[aslot]);
        if (k == nk1 - 1 && g == p.G1 - 1) commit(&bars.d1_full);
      }
      __syncwarp();
      if (++aslot == (uint32_t)p.NA) {
        aslot = 0;
        ++around;
      }
    };
    auto s1_all = [&](uint32_t it) {   // blocking stage 1 of tile it
      if (it > 0) {
        mbar_wait_warp(&bars.d1_free, (it - 1) & 1);
        fence_after();
      }
      for (int g = 0; g < p.G1; ++g)
        for (int k = 0; k < nk1; ++k) {
          mbar_wait_warp(&bars.a_full[aslot], around & 1);
          s1_chunk(g, k);
        }
    };
    auto s2 = [&](uint32_t it) {
      DL_PROF(2, 8);
      mbar_wait_warp(&bars.ac_full, it & 1);
      DL_PROF(2, 9);
      fence_after();
      for (int o = 0; o < (merge2 ? 1 : p.G2); ++o) {
        uint64_t bd[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) bd[j] = wdesc(sw2 + (uint32_t)j * p.w2_img, c2, km, o * p.N2);
        const uint32_t d = tbase + p.colD2 + (uint32_t)(o * p.N2);
        for (int kk = 0; kk < K2 / 16; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(d, tbase + p.colA2 + 8u * kk, K2 / 2, bd, id2, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd[j] += ks2;
        }
      }
      if (elect_one()) commit(&bars.u_full);
      __syncwarp();
    };
    // stage 3 of group o; the caller made sure its A operand is ready (au_full, which also means D3 is drained)
    auto s3_issue = [&](uint32_t it, int o) {
      DL_PROF(2, 11 + 2 * o);
      ++n_au;
      const int wg = p.w3_groups > 1 ? o : 0;
      uint64_t bd[PARTS];
#pragma unroll
      for (int j = 0; j < PARTS; ++j) bd[j] = wdesc(sw3 + (uint32_t)(j * p.w3_groups + wg) * p.w3_img, c3, km, 0);
      fence_after();
      for (int kk = 0; kk < p.N2 / 16; ++kk) {
        if (elect_one()) kstep_ts<PARTS>(tbase + p.colD3, tbase + p.colA3 + 8u * kk, p.N2 / 2, bd, id3, kk == 0);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < PARTS; ++j) bd[j] += ks3;
      }
      if (elect_one()) commit(&bars.y_full);
      __syncwarp();
    };
    const uint32_t nmine = ntiles > (int64_t)blockIdx.x ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    if (p.overlap) {
      // stage 3 of tile i and stage 1 of tile i+1 use disjoint TMEM: issue whichever is ready first
      if (nmine > 0) {
        s1_all(0);
        s2(0);
      }
      for (uint32_t it = 0; it < nmine; ++it) {
        const bool next = it + 1 < nmine;
        int g1 = 0, k1 = 0, o3 = 0;
        bool d1ok = !next;   // the next tile's D1 is free once MID has drained this tile's D1
        bool s1_done = !next;
        while (!s1_done || o3 < p.G2) {
          if (o3 < p.G2 && mbar_test(&bars.au_full, n_au & 1)) {
            s3_issue(it, o3++);
            continue;
          }
          if (!s1_done) {
            if (!d1ok) d1ok = mbar_test(&bars.d1_free, it & 1);
            if (d1ok && mbar_test(&bars.a_full[aslot], around & 1)) {
              s1_chunk(g1, k1);
              if (++k1 == nk1) {
                k1 = 0;
                if (++g1 == p.G1) s1_done = true;
              }
            }
          }
        }
        if (next) s2(it + 1);
      }
    } else {
      for (uint32_t it = 0; it < nmine; ++it) {
        s1_all(it);
        s2(it);
        for (int o = 0; o < p.G2; ++o) {
          mbar_wait_warp(&bars.au_full, n_au & 1);
          s3_issue(it, o);
        }
      }
    }
  } else if (p.tma) {
    // =========================== TMA loader ===========================
    tma_loader<NS>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, p.tm, smem + p.sm_ring, bars.full, bars.empty);
  }
  fence_before();
  __syncthreads();
  if (warp == kWarpMMA) tmem_dealloc(tbase, 512);
}

// ============================================================================ chain3v kernel
// Same three stages, but every accumulator stays resident (D1 | D2 | D3) and the A operands of all
// stages stream through two small TMEM rings, so the MMA warp can interleave the next tile's stage 1
// with this tile's stages 2/3 whenever a D3 drain or a conversion is in flight:
//   warps 0-7    IN   (two per lane quadrant, alternate chunks) -> IN ring (colA, NA slots)
//   warps 8-15   CONV D1 chunks -> conversion ring (colC, NAc slots) for stage 2, then D2 (+bias)
//                chunks for stage 3 of every output group (two per quadrant, alternate items)
//   warps 16-23  OUT  D3 -> HBM (two per quadrant, alternate 16-column chunks)
//   warp 24      MMA, warp 25 TMA loader.
// Ordering facts that replace explicit "free" barriers: CONV reads D1(t) only in the stage-2 items of
// tile t and D2(t-1) only before the first stage-2 item of tile t, so the MMA may overwrite D1 once it
// has consumed stage-2 item nk2-1 of tile t, and D2 once it consumes stage-2 item 0 of tile t+1.
#ifndef DL_CV_PER_Q
#define DL_CV_PER_Q 2
#endif
#ifndef DL_OUT_PER_Q
#define DL_OUT_PER_Q 2
#endif
constexpr int kCVQ = DL_CV_PER_Q, kOUTQ = DL_OUT_PER_Q;   // CONV / OUT warps per TMEM lane quadrant
constexpr int kIN3 = 8, kCV3 = 4 * kCVQ, kOUT3 = 4 * kOUTQ;
constexpr int kW3MMA = kIN3 + kCV3 + kOUT3;   // 24: stage-1 MMA issuer (+ TMEM owner)
constexpr int kW3MMA2 = kW3MMA + 1;           // 25: stage-2/3 MMA issuer
constexpr int kW3LD = kW3MMA2 + 1;            // 26
constexpr int kThreads3 = (kW3LD + 1) * 32;

struct Bars3v {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t a_full[kMaxSlots], a_empty[kMaxSlots];
  uint64_t c_full[kMaxSlots], c_empty[kMaxSlots];
  uint64_t d1g_full[2], d1g_free[2];   // stage-1 accumulator, one input group at a time, two buffers
  uint64_t d2_full, d3_full, d3_free;
  uint32_t tmem_base;
};

// H: fp16 two-term operands under delayed scaling (p.rstate), else bf16 PARTS-term operands.
template <int PARTS, int NS, bool H>
__global__ void __launch_bounds__(kThreads3, 1) chain3v_tc(const __grid_constant__ Chain3 p) {
  static_assert(NS % 2 == 0, "two IN warps alternate chunks: each ring stage needs one fixed consumer pair");
  static_assert(!H || PARTS == 2, "the fp16 path uses two terms");
  extern __shared__ __align__(1024) uint8_t smem[];
  if (!H && p.redo) {
    if (__syncthreads_or(threadIdx.x == 0 ? (range_check(p.rstate) ? 1 : 0) : 0)) return;
  }
  Bars3v& bars = *reinterpret_cast<Bars3v*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kSlotW = PARTS * 8;
  int sexp = 0;
  if constexpr (H) {
    sexp = (int)*(volatile const uint32_t*)(p.rstate + kStExp);
    sexp = sexp < -100 ? -100 : sexp > 100 ? 100 : sexp;
  }
  const float sc = pow2f(sexp), isc = pow2f(-sexp);   // 1 on the bf16 path
  float amax = 0.f;                                   // IN: scaled inputs; CONV: scaled accumulators

  {  // stage weight images + bias once per CTA
    const uint32_t b1 = (uint32_t)PARTS * p.w1_groups * p.w1_img, b2 = (uint32_t)PARTS * p.w2_img,
                   b3 = (uint32_t)PARTS * p.w3_groups * p.w3_img;
    const uint4 *s1 = reinterpret_cast<const uint4*>(p.w1), *s2 = reinterpret_cast<const uint4*>(p.w2),
                *s3 = reinterpret_cast<const uint4*>(p.w3);
    uint4 *d1 = reinterpret_cast<uint4*>(smem + p.sm_w1), *d2 = reinterpret_cast<uint4*>(smem + p.sm_w2),
          *d3 = reinterpret_cast<uint4*>(smem + p.sm_w3);
    for (uint32_t i = threadIdx.x; i < b1 / 16; i += blockDim.x) d1[i] = __ldg(s1 + i);
    for (uint32_t i = threadIdx.x; i < b2 / 16; i += blockDim.x) d2[i] = __ldg(s2 + i);
    for (uint32_t i = threadIdx.x; i < b3 / 16; i += blockDim.x) d3[i] = __ldg(s3 + i);
    float* sb = reinterpret_cast<float*>(smem + p.sm_bias);
    for (int i = threadIdx.x; i < p.G2 * p.N2; i += blockDim.x) {
      const int o = i / p.N2, r = i - o * p.N2;
      sb[i] = (p.bias2 && r < p.C2) ? __ldg(p.bias2 + o * p.C2 + r) * sc : 0.f;
    }
  }
  if (warp == kW3MMA) tmem_alloc(&bars.tmem_base, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 4);
    }
    for (int s = 0; s < p.NA; ++s) {
      mbar_init(&bars.a_full[s], 4);
      mbar_init(&bars.a_empty[s], 1);
    }
    for (int s = 0; s < p.NAc; ++s) {
      mbar_init(&bars.c_full[s], 4);   // one CONV warp per quadrant converts each item
      mbar_init(&bars.c_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.d1g_full[b], 1);
      mbar_init(&bars.d1g_free[b], kCV3);   // every CONV warp, once per group
    }
    mbar_init(&bars.d2_full, 1);
    mbar_init(&bars.d3_full, 1);
    mbar_init(&bars.d3_free, kOUT3);
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;
  const int nk1 = p.K1 / 16, per_tile = p.G1 * nk1;
  const int K2 = p.G1 * p.N1, nk2 = K2 / 16, nk3 = p.N2 / 16;
  const float inv_nk1 = 1.f / (float)nk1;   // r / nk1 without an integer division (r < 256: exact)
  auto geo = [&](int r) {
    const int g = (int)(((float)r + 0.5f) * inv_nk1), k = r - g * nk1;
    return ChunkGeo{0, g * p.C1 + 16 * k, p.C1 - 16 * k};
  };

  if (warp < kIN3) {
    // =========================== IN ===========================
    const uint32_t tslots = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + p.colA;
    if (p.raw) {
      // all 8 IN warps (two per quadrant, alternate chunks), each with a private ring: NS stages of 1 KB (int16)
      // or NS / 2 stages of 2 KB (fp32) -- 8 KB per ring stage slot of the plan
      if (p.raw_type == 4)
        in_role_raw<PARTS, NS, int16_t, decltype(geo), H>(
            geo, per_tile, ntiles, p.tiles_per_b, p.nvox, reinterpret_cast<const int16_t*>(p.raw), p.raw_vstride,
            p.raw_sel, p.vox_a, p.vox_b, tslots, p.NA, bars.a_full, bars.a_empty,
            reinterpret_cast<int16_t*>(smem + p.sm_ring) + warp * NS * 512, warp >> 2, 2, sc, &amax);
      else
        in_role_raw<PARTS, NS / 2, float, decltype(geo), H>(
            geo, per_tile, ntiles, p.tiles_per_b, p.nvox, reinterpret_cast<const float*>(p.raw), p.raw_vstride,
            p.raw_sel, p.vox_a, p.vox_b, tslots, p.NA, bars.a_full, bars.a_empty,
            reinterpret_cast<float*>(smem + p.sm_ring) + warp * (NS / 2) * 512, warp >> 2, 2, sc, &amax);
    } else if (p.tma && p.cpi == 2) {
      if constexpr (NS % 4 == 0)
        in_role_tma2<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, tslots, p.NA,
                                                  bars.a_full, bars.a_empty,
                                                  reinterpret_cast<const float*>(smem + p.sm_ring), bars.full,
                                                  bars.empty, warp >> 2, sc, &amax);
    } else if (p.tma) {
      in_role_tma<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, tslots, p.NA,
                                               bars.a_full, bars.a_empty,
                                               reinterpret_cast<const float*>(smem + p.sm_ring), bars.full, bars.empty,
                                               warp >> 2, 2, sc, &amax);
    } else if (warp < 4) {
      const float* const base[2] = {p.in, p.in};
      const int64_t bs[2] = {p.in_bs, p.in_bs};
      in_role_cpasync<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, base, bs, tslots,
                                                   p.NA, bars.a_full, bars.a_empty,
                                                   reinterpret_cast<float*>(smem + p.sm_ring) + warp * NS * 512, 0, 1,
                                                   sc, &amax);
    }
    if (H) amax_publish(p.rstate + kStAmaxIn, amax);
  } else if (warp < kIN3 + kCV3) {
    // =========================== CONV: accumulators -> conversion ring ===========================
    // items per tile: for each input group g, n1c chunks of D1_g (stage-2 A, also stored to the mid
    // buffer), then G2 x nk3 D2 chunks (+bias, stage-3 A).  Item i of the CTA-wide sequence belongs to
    // CONV warp i % kCVQ and uses conversion slot i % NAc.
    const int cw = (warp - kIN3) >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    const float* sb = reinterpret_cast<const float*>(smem + p.sm_bias);
    const int per_c = nk2 + p.G2 * nk3, n1c = p.N1 / 16;
    uint32_t cslot = (uint32_t)(cw % p.NAc), cround = (uint32_t)(cw / p.NAc), it = 0;
    uint32_t base = 0;    // CTA-wide index of the tile's first item
    uint32_t gq = 0;      // CTA-wide input-group counter (D1 buffer gq & 1)
    auto put = [&](const uint32_t (&w)[PARTS][8]) {
      if (cround > 0) role_wait(&bars.c_empty[cslot], (cround - 1) & 1);
      fence_after();
      store_parts<PARTS>(tq + p.colC + cslot * kSlotW, 8, w);
      tmem_wait_st();
      fence_before();
      warp_arrive(&bars.c_full[cslot]);
      cslot += kCVQ;
      while (cslot >= (uint32_t)p.NAc) {
        cslot -= p.NAc;
        ++cround;
      }
    };
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it, base += (uint32_t)per_c) {
      const int64_t b = t / p.tiles_per_b, vx = (t - b * p.tiles_per_b) * kTileV + 32 * (warp & 3) + lane;
      const bool vok = vx < p.nvox;
      uint16_t* mid = (p.mid && vx < p.mid_pitch)
                          ? p.mid + ((b * (p.mid_pitch >> 6) + (vx >> 6)) * 2 * K2) * 64 + (vx & 63)
                          : nullptr;
      if (warp == kIN3) DL_PROF(1, 0);
      for (int g = 0; g < p.G1; ++g, ++gq) {
        const uint32_t nb = p.G1 >= 2 ? 2u : 1u, buf = gq % nb;
        role_wait(&bars.d1g_full[buf], (gq / nb) & 1);
        fence_after();
        for (int c = 0; c < n1c; ++c) {
          const int i = g * n1c + c;
          if ((base + (uint32_t)i) % kCVQ != (uint32_t)cw) continue;
          if ((warp & 3) == 0) DL_PROF(cw ? 6 : 5, i);
          float v[16];
          ld16f(tq + p.colD1 + buf * (uint32_t)p.N1 + (uint32_t)c * 16, v);
          track16<H>(v, amax);
          uint32_t w[PARTS][8];
          split16<PARTS, H>(v, w);
          if (mid) {
            if constexpr (H) {   // the Gram operand is unscaled bf16 (hi, next term)
              float u[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) u[e] = v[e] * isc;
              uint32_t m[2][8];
              split16<2>(u, m);
              store_mid(mid + (int64_t)i * 16 * 64, (int64_t)K2 * 64, 64, m[0], m[1], vok ? p.mid_ones - 16 * i : -1);
            } else {
              store_mid(mid + (int64_t)i * 16 * 64, (int64_t)K2 * 64, 64, w[0], w[1], vok ? p.mid_ones - 16 * i : -1);
            }
          }
          if ((warp & 3) == 0) DL_PROF(cw ? 6 : 5, 10 + i);
          put(w);
          if ((warp & 3) == 0) DL_PROF(cw ? 6 : 5, 20 + i);
        }
        fence_before();
        warp_arrive(&bars.d1g_free[buf]);   // this warp is done reading D1 buffer `buf`
      }
      if (warp == kIN3) DL_PROF(1, 2);
      bool d2_seen = false;
      for (int i = nk2; i < per_c; ++i) {
        if ((base + (uint32_t)i) % kCVQ != (uint32_t)cw) continue;
        if (!d2_seen) {
          role_wait(&bars.d2_full, it & 1);
          if (warp == kIN3) DL_PROF(1, 3);
          fence_after();
          d2_seen = true;
        }
        const int o = (i - nk2) / nk3, j = (i - nk2) - o * nk3;
        if ((warp & 3) == 0) DL_PROF(cw ? 3 : 0, i - nk2);
        float v[16];
        ld16f(tq + p.colD2 + (uint32_t)(o * p.N2 + 16 * j), v);
        const float* bb = sb + o * p.N2 + 16 * j;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] += bb[e];
        track16<H>(v, amax);
        uint32_t w[PARTS][8];
        split16<PARTS, H>(v, w);
        if ((warp & 3) == 0) DL_PROF(cw ? 3 : 0, 10 + i - nk2);
        put(w);
        if ((warp & 3) == 0) DL_PROF(cw ? 3 : 0, 20 + i - nk2);
      }
    }
    if (H) amax_publish(p.rstate + kStAmaxMid, amax);
  } else if (warp < kW3MMA) {
    // =========================== OUT: D3 -> HBM ===========================
    const int ow = warp - kIN3 - kCV3, qd = warp & 3, cg = ow >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int row = 32 * qd + lane;
    const int64_t stride = p.nvox;
    uint32_t n3 = 0, it = 0;
    double lacc = 0.0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int64_t b = t / p.tiles_per_b, v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool vok = v < p.nvox;
      for (int o = 0; o < p.G2; ++o, ++n3) {
        idle_wait<1>(&bars.d3_full, n3 & 1);
        if (ow == 0) DL_PROF(1, 8 + 2 * o);
        fence_after();
        for (int ck = cg; ck < p.N3 / 16; ck += kOUTQ) {
          float vv[16];
          ld16f(tq + p.colD3 + (uint32_t)ck * 16, vv);
          if constexpr (H) {
#pragma unroll
            for (int e = 0; e < 16; ++e) vv[e] *= isc;
          }
          if (vok && p.out) {   // out == null: a g-only adjoint (no dx)
            const int64_t off = b * p.out_bs + ((int64_t)o * p.C3 + ck * 16) * stride + v;
            float* d = p.out + off;
            const int nval = p.C3 - ck * 16;
            if (p.target) {   // fused MSE: d(loss)/dy, and the squared residuals (loads first, see chain2h)
              const float* tg = p.target + off;
              float tv[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) tv[i] = (nval >= 16 || i < nval) ? __ldcs(tg + (int64_t)i * stride) : 0.f;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (nval >= 16 || i < nval) {
                  const float r = vv[i] - tv[i];
                  lacc += (double)r * (double)r;
                  __stcs(d, r * p.out_scale);
                }
                d += stride;
              }
            } else if (nval >= 16) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                __stcs(d, vv[i]);
                d += stride;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (i < nval) __stcs(d, vv[i]);
                d += stride;
              }
            }
          }
        }
        fence_before();
        warp_arrive(&bars.d3_free);
        if (ow == 0) DL_PROF(1, 9 + 2 * o);
      }
    }
    if (p.target) loss_publish(p.loss + (p.redo ? 1 : 0), lacc);
  } else if (warp == kW3MMA || warp == kW3MMA2) {
    // =========================== MMA issuers ===========================
    // Two issuing warps on different schedulers: under contention each tcgen05.mma costs the issuing
    // warp ~100 cycles of issue latency, so stage 1 (fed by IN) and stages 2/3 (fed by CONV) get one
    // warp each and the tensor pipe interleaves them.
    // Lean loop: descriptors advance by additions; stage/group cursors are incremental.
    const uint32_t sw1 = smem_u32(smem + p.sm_w1), sw2 = smem_u32(smem + p.sm_w2), sw3 = smem_u32(smem + p.sm_w3);
    const int km = p.adjoint ? 0 : 1;
    const int NT2 = p.G2 * p.N2;
    const int n2m = NT2 <= 256 ? 1 : p.G2;   // stage-2 MMAs per item (N split when > 256)
    const uint32_t id1 = H ? idesc_f16(128, p.N1, 0, 1 - km) : idesc_bf16(128, p.N1, 0, 1 - km);
    const uint32_t id2 = H ? idesc_f16(128, n2m == 1 ? NT2 : p.N2, 0, 1 - km)
                           : idesc_bf16(128, n2m == 1 ? NT2 : p.N2, 0, 1 - km);
    const uint32_t id3 = H ? idesc_f16(128, p.N3, 0, 1 - km) : idesc_bf16(128, p.N3, 0, 1 - km);
    const int c1 = km ? p.K1 : p.N1, c2 = km ? K2 : NT2, c3 = km ? p.N2 : p.N3;
    const uint64_t ks1 = wkstep(c1, km), ks2 = wkstep(c2, km), ks3 = wkstep(c3, km);
    uint64_t B1[PARTS], B2[PARTS], B3[PARTS];
#pragma unroll
    for (int j = 0; j < PARTS; ++j) {
      B1[j] = wdesc(sw1 + (uint32_t)(j * p.w1_groups) * p.w1_img, c1, km, 0);
      B2[j] = wdesc(sw2 + (uint32_t)j * p.w2_img, c2, km, 0);
      B3[j] = wdesc(sw3 + (uint32_t)(j * p.w3_groups) * p.w3_img, c3, km, 0);
    }
    const uint64_t g1s = p.w1_groups > 1 ? (uint64_t)(p.w1_img >> 4) : 0;   // next group's image
    const uint64_t g3s = p.w3_groups > 1 ? (uint64_t)(p.w3_img >> 4) : 0;
    const uint64_t o2s = wdesc(0, c2, km, p.N2) - wdesc(0, c2, km, 0);      // next N2 block of stage 2
    const uint32_t nmine = ntiles > (int64_t)blockIdx.x ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    const uint32_t tA = tbase + p.colA, tC = tbase + p.colC, tD1 = tbase + p.colD1, tD2 = tbase + p.colD2,
                   tD3 = tbase + p.colD3;
    uint32_t aslot = 0, around = 0, cslot = 0, cround = 0, n3 = 0;
    uint32_t aaddr = tA, caddr = tC;
    const int n1 = p.G1 * nk1;
    if (warp == kW3MMA) {
      // ---- stage 1: input chunks -> D1, one input group at a time into alternating buffers ----
      uint32_t gq = 0;
      for (uint32_t it = 0; it < nmine; ++it) {
        for (int g = 0; g < p.G1; ++g, ++gq) {
          const uint32_t nb = p.G1 >= 2 ? 2u : 1u, buf = gq % nb;
          DL_PROF(4, 3 * g);
          if (gq >= nb) {   // CONV has read (and stored) the group that last used this buffer
            mbar_wait_warp(&bars.d1g_free[buf], ((gq / nb) - 1) & 1);
            fence_after();
          }
          DL_PROF(4, 3 * g + 1);
          const uint32_t d1col = tD1 + buf * (uint32_t)p.N1;
          uint64_t bd[PARTS];
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd[j] = B1[j] + (uint64_t)g * g1s;
          for (int k = 0; k < nk1; k += p.cpi) {   // one IN item = cpi K-steps
            mbar_wait_warp(&bars.a_full[aslot], around & 1);
            DL_PROF(4, 10 + (g * nk1 + k) / p.cpi);
            fence_after();
            if (elect_one()) {
              kstep_ts<PARTS>(d1col, aaddr, 8, bd, id1, k == 0);
              if (p.cpi == 2) {
                uint64_t bn[PARTS];
#pragma unroll
                for (int j = 0; j < PARTS; ++j) bn[j] = bd[j] + ks1;
                kstep_ts<PARTS>(d1col, aaddr + kSlotW, 8, bn, id1, false);
              }
              commit(&bars.a_empty[aslot]);
              if (k + p.cpi >= nk1) commit(&bars.d1g_full[buf]);
            }
            __syncwarp();
            if (++aslot == (uint32_t)p.NA) {
              aslot = 0;
              ++around;
              aaddr = tA;
            } else {
              aaddr += (uint32_t)p.cpi * kSlotW;
            }
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] += (uint64_t)p.cpi * ks1;
          }
        }
      }
    } else {
      // ---- stages 2 and 3: conversion-ring items in CONV order ----
      auto c_take = [&]() {
        mbar_wait_warp(&bars.c_full[cslot], cround & 1);
        fence_after();
      };
      auto c_release = [&](uint64_t* extra) {
        if (elect_one()) {
          commit(&bars.c_empty[cslot]);
          if (extra) commit(extra);
        }
        __syncwarp();
        if (++cslot == (uint32_t)p.NAc) {
          cslot = 0;
          ++cround;
          caddr = tC;
        } else {
          caddr += kSlotW;
        }
      };
      for (uint32_t it = 0; it < nmine; ++it) {
        DL_PROF(2, 0);
        uint64_t bd2[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) bd2[j] = B2[j];
        for (int jj = 0; jj < nk2; ++jj) {
          c_take();
          uint64_t bd[PARTS];
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd[j] = bd2[j];
          for (int oo = 0; oo < n2m; ++oo) {
            if (elect_one()) kstep_ts<PARTS>(tD2 + (uint32_t)(oo * p.N2), caddr, 8, bd, id2, jj == 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] += o2s;
          }
          c_release(jj == nk2 - 1 ? &bars.d2_full : nullptr);
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd2[j] += ks2;
        }
        DL_PROF(2, 1);
        uint64_t bg3[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) bg3[j] = B3[j];
        for (int o = 0; o < p.G2; ++o) {
          if (n3 > 0) mbar_wait_warp(&bars.d3_free, (n3 - 1) & 1);
          DL_PROF(2, 2 + 2 * o);
          uint64_t bd[PARTS];
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd[j] = bg3[j];
          for (int jj = 0; jj < nk3; ++jj) {
            c_take();
            if (elect_one()) kstep_ts<PARTS>(tD3, caddr, 8, bd, id3, jj == 0);
            __syncwarp();
            c_release(jj == nk3 - 1 ? &bars.d3_full : nullptr);
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] += ks3;
          }
          ++n3;
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bg3[j] += g3s;
          DL_PROF(2, 3 + 2 * o);
        }
      }
    }
  } else if (p.tma) {
    tma_loader<NS>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, p.tm, smem + p.sm_ring, bars.full, bars.empty);
  }
  fence_before();
  __syncthreads();
  if (warp == kW3MMA) tmem_dealloc(tbase, 512);
}

// ============================================================================ chain2h kernel
// The fp16 pass with SH2Signal folded into the LSC operator: y_o = T_o c + bias3_o with T_o = B' L_{o,:}
// (forward) or dx_s = T'_s g with T'_s = M_s^T (L^T)_{s,:} (adjoint), so the tile runs two MMA stages:
//   stage 1   D1 = x M^T per input group (issuer 1, as chain3v), into two alternating D1 buffers;
//   CONV      D1 -> A2, the whole tile's stage-2 A operand resident in TMEM (G1 x N1 columns, two fp16
//             terms), plus the c / g term planes for the Gram; A2 of the next tile waits for a2_free;
//   stage 2   D3[o] = A2 T_o^T, one output group at a time into two alternating D3 buffers (issuer 2): group 0
//             streams the A2 items as CONV hands them over, later groups reuse the resident A2;
//   OUT       D3 -> y (x 2^-e + bias3) while the MMA fills the other D3 buffer.
// Against chain3v this drops the D2 accumulator and its conversion pass (half of CONV's TMEM loads, splits
// and handoffs) for ~14% more MMA work; it needs the T images (G2 x N3 x K2 fp16 pairs) in shared memory.
#ifndef DL_IN_SEQ
#define DL_IN_SEQ 0
#endif
#ifndef DL_OB2H
#define DL_OB2H 1
#endif
constexpr int kOB2h = DL_OB2H;   // D3 chunks an OUT warp loads before releasing / storing them
// A2 released item by item as the last output shell's stage-2 MMAs read it (a2_ifree), so CONV converts the
// next tile's items while that shell's MMAs still run; 0: one a2_free for the whole tile (measurement knob)
#ifndef DL_A2_ITEM
#define DL_A2_ITEM 1
#endif
constexpr bool kA2Item = DL_A2_ITEM != 0;
// CONV writes an item's Gram term planes after handing the item to the stage-2 MMA (1) or before (0)
#ifndef DL_MID_LATE
#define DL_MID_LATE 1
#endif
constexpr bool kMidLate = DL_MID_LATE != 0;
// stage 2: shells 0 and 1 of a tile interleaved so that their last kDefer items come after both shells' other
// items (0: shell after shell)
#ifndef DL_DEFER
#define DL_DEFER 1
#endif
constexpr int kDefer = DL_DEFER;
// chain2h keeps its barriers small: with the 12-deep TMA ring the shared-memory plan has < 900 bytes left for
// them (a larger block silently drops the ring to 8 stages)
constexpr int kMaxStages2h = 12;
struct Bars2h {
  uint64_t full[kMaxStages2h], empty[kMaxStages2h];
  uint64_t a_full[kMaxSlots], a_empty[kMaxSlots];
  uint64_t d1g_full[2], d1g_free[2];
  uint64_t a2_full[16], a2_free;
  uint64_t a2_ifree[16];                            // item k of A2 read by the last output shell's MMAs
  uint64_t d3_full[2], d3_free[2];
  uint64_t c_full[kMaxSlots], c_empty[kMaxSlots];   // KOUT: A2 item ring
  uint64_t d3g_free[4];                             // KOUT: output shell o of D3 drained
  uint64_t t_full[2], t_empty[2];                   // tstream: T image buffers
  uint32_t tmem_base;
};
constexpr int kWT = kW3LD + 1;                      // chain2h: T-image loader warp (tstream)
constexpr int kThreads2h = (kWT + 1) * 32;

// KOUT = false: A2 resident, stage 2 one output shell at a time (D3 double-buffered).
// KOUT = true: A2 items stream through a ring (NAc slots) and stage 2 is K-outer over all output shells
//   (D3 holds every shell; OUT releases shell o as soon as it is drained, so the next tile's first K-step
//   into shell o can start), which removes the CONV -> stage 2 -> a2_free -> CONV cycle of the tile.
// GONLY: a g-only adjoint (no dx requested: the first layer of a training step): stage 1 and the Gram term planes
// only -- no A2, no stage 2, no OUT stores, no T images.
template <int NS, bool KOUT, bool DIAG, bool GONLY>
__global__ void __launch_bounds__(kThreads2h, 1) chain2h_tc(const __grid_constant__ Chain3 p) {
  constexpr int PARTS = 2;
  constexpr bool H = true;
  extern __shared__ __align__(1024) uint8_t smem[];
  ktrace_begin(p.kt, p.kt_slot);
  Bars2h& bars = *reinterpret_cast<Bars2h*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kSlotW = PARTS * 8;
  int sexp = (int)*(volatile const uint32_t*)(p.rstate + kStExp);
  sexp = sexp < -100 ? -100 : sexp > 100 ? 100 : sexp;
  const float sc = pow2f(sexp), isc = pow2f(-sexp);
  float amax = 0.f;
  {  // stage weight images + the folded bias once per CTA
    const uint32_t b1 = (uint32_t)PARTS * p.w1_groups * p.w1_img, b2 = p.tstream ? 0u : (uint32_t)PARTS * p.w2_img;
    const uint4 *s1 = reinterpret_cast<const uint4*>(p.w1), *s2 = reinterpret_cast<const uint4*>(p.w2);
    uint4 *d1 = reinterpret_cast<uint4*>(smem + p.sm_w1), *d2 = reinterpret_cast<uint4*>(smem + p.sm_w2);
    for (uint32_t i = threadIdx.x; i < b1 / 16; i += blockDim.x) d1[i] = __ldg(s1 + i);
    for (uint32_t i = threadIdx.x; i < b2 / 16; i += blockDim.x) d2[i] = __ldg(s2 + i);
    float* sb = reinterpret_cast<float*>(smem + p.sm_bias);
    for (int i = threadIdx.x; i < p.G2 * p.N3; i += blockDim.x) {
      const int o = i / p.N3, r = i - o * p.N3;
      sb[i] = (p.bias2 && r < p.C3) ? __ldg(p.bias2 + o * p.C3 + r) : 0.f;
    }
  }
  const int nk1 = p.K1 / 16, per_tile = p.G1 * nk1;
  const int K2 = p.G1 * p.N1, nk2 = K2 / 16;
  if (warp == kW3MMA) tmem_alloc(&bars.tmem_base, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 4);
    }
    for (int s = 0; s < p.NA; ++s) {
      mbar_init(&bars.a_full[s], 4);
      mbar_init(&bars.a_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.d1g_full[b], 1);
      mbar_init(&bars.d1g_free[b], kCV3);
      mbar_init(&bars.d3_full[b], 1);
      mbar_init(&bars.d3_free[b], kOUT3);
    }
    for (int k = 0; k < nk2; ++k) mbar_init(&bars.a2_full[k], 4);   // the quadrant warps converting item k
    mbar_init(&bars.a2_free, 1);
    for (int k = 0; k < 16; ++k) mbar_init(&bars.a2_ifree[k], 1);
    for (int c = 0; c < p.NAc; ++c) {
      mbar_init(&bars.c_full[c], 4);
      mbar_init(&bars.c_empty[c], 1);
    }
    for (int o = 0; o < 4; ++o) mbar_init(&bars.d3g_free[o], kOUT3);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.t_full[b], 1);
      mbar_init(&bars.t_empty[b], 1);
    }
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;
  auto geo = [&](int r) {
    const int g = r / nk1, k = r - g * nk1;
    return ChunkGeo{0, g * p.C1 + 16 * k, p.C1 - 16 * k};
  };

  if (warp < kIN3) {
    // =========================== IN (as chain3v) ===========================
    const uint32_t tslots = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + p.colA;
    if (p.raw) {   // raw acquisition input (in_role_raw, one chunk per IN item)
      if (p.raw_type == 4)
        in_role_raw<PARTS, NS, int16_t, decltype(geo), H>(
            geo, per_tile, ntiles, p.tiles_per_b, p.nvox, reinterpret_cast<const int16_t*>(p.raw), p.raw_vstride,
            p.raw_sel, p.vox_a, p.vox_b, tslots, p.NA, bars.a_full, bars.a_empty,
            reinterpret_cast<int16_t*>(smem + p.sm_ring) + warp * NS * 512, warp >> 2, 2, sc, &amax);
      else
        in_role_raw<PARTS, NS / 2, float, decltype(geo), H>(
            geo, per_tile, ntiles, p.tiles_per_b, p.nvox, reinterpret_cast<const float*>(p.raw), p.raw_vstride,
            p.raw_sel, p.vox_a, p.vox_b, tslots, p.NA, bars.a_full, bars.a_empty,
            reinterpret_cast<float*>(smem + p.sm_ring) + warp * (NS / 2) * 512, warp >> 2, 2, sc, &amax);
    } else if (p.tma && p.cpi == 2) {
      if constexpr (NS % 4 == 0)
        in_role_tma2<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, tslots, p.NA,
                                                  bars.a_full, bars.a_empty,
                                                  reinterpret_cast<const float*>(smem + p.sm_ring), bars.full,
                                                  bars.empty, warp >> 2, sc, &amax);
    } else if (p.tma) {
      in_role_tma<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, tslots, p.NA,
                                               bars.a_full, bars.a_empty,
                                               reinterpret_cast<const float*>(smem + p.sm_ring), bars.full, bars.empty,
                                               warp >> 2, 2, sc, &amax);
    } else if (warp < 4) {
      const float* const base[2] = {p.in, p.in};
      const int64_t bs[2] = {p.in_bs, p.in_bs};
      in_role_cpasync<PARTS, NS, decltype(geo), H>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, base, bs, tslots,
                                                   p.NA, bars.a_full, bars.a_empty,
                                                   reinterpret_cast<float*>(smem + p.sm_ring) + warp * NS * 512, 0, 1,
                                                   sc, &amax);
    }
    amax_publish(p.rstate + kStAmaxIn, amax);
  } else if (warp < kIN3 + kCV3) {
    // =========================== CONV: D1 -> resident A2 (+ the Gram term planes) ===========================
    const int cw = (warp - kIN3) >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    const int n1c = p.N1 / 16;
    const int ones_item = p.mid_ones >= 0 ? p.mid_ones >> 4 : -1;   // the item holding c's bias row
    uint32_t gq = 0, it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int64_t b = t / p.tiles_per_b, vx = (t - b * p.tiles_per_b) * kTileV + 32 * (warp & 3) + lane;
      const bool vok = vx < p.nvox;
      uint16_t* mid = (p.mid && vx < p.mid_pitch)
                          ? p.mid + ((b * (p.mid_pitch >> 6) + (vx >> 6)) * 2 * K2) * 64 + (vx & 63)
                          : nullptr;
      if (!KOUT && !kA2Item && it > 0) {   // the previous tile's stage-2 MMAs have read A2
        role_wait(&bars.a2_free, (it - 1) & 1);
      }
      for (int g = 0; g < p.G1; ++g, ++gq) {
        const uint32_t nb = p.G1 >= 2 ? 2u : 1u, buf = gq % nb;
        role_wait(&bars.d1g_full[buf], (gq / nb) & 1);
        fence_after();
        for (int c = 0; c < n1c; ++c) {
          const int i = g * n1c + c;
          if (i % kCVQ != cw) continue;   // the CONV warps of a quadrant take items round-robin
          float v[16];
          ld16f(tq + p.colD1 + buf * (uint32_t)p.N1 + (uint32_t)c * 16, v);
          track16<H>(v, amax);
          if constexpr (GONLY) {   // the Gram term planes are the only product
            if (mid) {
              float u[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) u[e] = v[e] * isc;
              uint32_t m[2][8];
              split16<2>(u, m);
              if (i == ones_item) set_ones(m[0], m[1], vok ? p.mid_ones - 16 * i : -1);
              store_mid<false>(mid + (int64_t)i * 16 * 64, (int64_t)K2 * 64, 64, m[0], m[1], -1);
            }
            continue;
          }
          uint32_t w[PARTS][8];
          split16<PARTS, H>(v, w);
          if (mid && !kMidLate) {
            float u[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) u[e] = v[e] * isc;
            uint32_t m[2][8];
            split16<2>(u, m);
            store_mid(mid + (int64_t)i * 16 * 64, (int64_t)K2 * 64, 64, m[0], m[1], vok ? p.mid_ones - 16 * i : -1);
          }
          if constexpr (KOUT) {
            const uint32_t ci = it * (uint32_t)nk2 + (uint32_t)i, slot = ci % (uint32_t)p.NAc,
                           round = ci / (uint32_t)p.NAc;
            if (round > 0) role_wait(&bars.c_empty[slot], (round - 1) & 1);
            fence_after();
            store_parts<PARTS>(tq + p.colA2 + slot * kSlotW, 8, w);
            tmem_wait_st();
            fence_before();
            warp_arrive(&bars.c_full[slot]);
          } else {
            // the previous tile's item i was read by its last reader (the last output shell's MMA, or shell i's
            // group alone for a block-diagonal T)
            if (kA2Item && it > 0) {
              role_wait(&bars.a2_ifree[i], (it - 1) & 1);
              fence_after();
            }
            store_parts<PARTS>(tq + p.colA2 + (uint32_t)i * kSlotW, 8, w);
            tmem_wait_st();
            fence_before();
            warp_arrive(&bars.a2_full[i]);
          }
          if (mid && kMidLate) {   // the Gram term planes after the A2 handoff: off the MMA's critical path
            float u[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) u[e] = v[e] * isc;
            uint32_t m[2][8];
            split16<2>(u, m);
            if (i == ones_item) set_ones(m[0], m[1], vok ? p.mid_ones - 16 * i : -1);   // only the bias row's item
            store_mid<false>(mid + (int64_t)i * 16 * 64, (int64_t)K2 * 64, 64, m[0], m[1], -1);
          }
        }
        fence_before();
        warp_arrive(&bars.d1g_free[buf]);
      }
    }
    amax_publish(p.rstate + kStAmaxMid, amax);
  } else if (warp < kW3MMA) {
    if constexpr (!GONLY) {
    // =========================== OUT: D3 -> HBM (x 2^-e + folded bias) ===========================
    const int ow = warp - kIN3 - kCV3, qd = warp & 3, cg = ow >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int row = 32 * qd + lane;
    const int64_t stride = p.nvox;
    const float* sb = reinterpret_cast<const float*>(smem + p.sm_bias);
    const int nck = p.N3 / 16;
    uint32_t n3 = 0;
    double lacc = 0.0;
    // Fused MSE with a target ring (kOB2h == 1): this warp's target chunks (16 channels x its 32 voxels) are
    // copied one chunk ahead by per-thread cp.async into a private 2-stage ring, so the loads overlap the
    // previous chunk's arithmetic and stores instead of stalling them (each thread reads back only what it
    // copied: cp.async.wait_group is the only synchronisation).  Safe when target aliases out: a chunk's
    // target elements are read before that chunk's outputs are written, and chunks never overlap.
    const bool tring = p.target && p.sm_tring && kOB2h == 1 && !KOUT;
    float* tr = reinterpret_cast<float*>(smem + p.sm_tring) + ow * 1024;
    int64_t nt_t = blockIdx.x;   // next target chunk to issue: tile, shell, chunk
    int nt_o = 0, nt_ck = cg;
    uint32_t tq_issue = 0, tq_use = 0;
    // 8-byte copies (two voxels per lane, two rows per instruction) when every row start is 8-byte aligned
    const bool t8 = (p.nvox % 2 == 0) && ((uintptr_t)p.target % 8 == 0) && (p.out_bs % 2 == 0);
    auto t_issue = [&]() {
      __syncwarp();   // every lane has read the stage this copy overwrites (lanes read each other's copies)
      if (nt_t < ntiles) {
        const int64_t bb_ = nt_t / p.tiles_per_b;
        if (t8) {
          const int64_t v0q = (nt_t - bb_ * p.tiles_per_b) * kTileV + 32 * qd;
          const int nrow = p.C3 - nt_ck * 16, pv = 2 * (lane & 15);
          const int64_t vv = v0q + pv;
          const uint32_t nb = vv + 1 < p.nvox ? 8u : vv < p.nvox ? 4u : 0u;
          const float* src = p.target + bb_ * p.out_bs + ((int64_t)nt_o * p.C3 + nt_ck * 16) * stride + (nb ? vv : 0);
          float* dst = tr + (tq_issue & 1) * 512 + pv;
          if (nrow >= 16 && nb == 8u) {   // full chunk, both voxels inside: a 32-bit byte stride per row pair
            const char* sp = reinterpret_cast<const char*>(src + (lane >> 4) * stride);
            const uint32_t rs2 = (uint32_t)stride * 8u;
            float* dp = dst + (lane >> 4) * 32;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              cp_async8(dp + 2 * i * 32, reinterpret_cast<const float*>(sp), 8u);
              sp += rs2;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 2 * i + (lane >> 4);
              const bool ok = r < nrow && nb;
              cp_async8(dst + r * 32, ok ? src + (int64_t)r * stride : p.target, ok ? nb : 0u);
            }
          }
        } else {
          const int64_t vv = (nt_t - bb_ * p.tiles_per_b) * kTileV + row;
          const bool ok = vv < p.nvox;
          const float* src = p.target + bb_ * p.out_bs + ((int64_t)nt_o * p.C3 + nt_ck * 16) * stride + (ok ? vv : 0);
          stream_chunk(tr + (tq_issue & 1) * 512 + lane, src, stride, ok ? p.C3 - nt_ck * 16 : 0, p.target);
        }
        nt_ck += kOUTQ;
        if (nt_ck >= nck) {
          nt_ck = cg;
          if (++nt_o == p.G2) {
            nt_o = 0;
            nt_t += gridDim.x;
          }
        }
      }
      cp_async_commit();
      ++tq_issue;
    };
    if (tring) t_issue();
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t b = t / p.tiles_per_b, v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool vok = v < p.nvox;
      if (KOUT) {
        idle_wait<1>(&bars.d3_full[0], (n3 / (uint32_t)p.G2) & 1);
        fence_after();
      }
      for (int o = 0; o < p.G2; ++o, ++n3) {
        const uint32_t xb = KOUT ? 0u : (n3 & 1);
        if (p.target && vok && !tring) {   // fused MSE: pull this shell's target rows into L2 while the MMA runs
          for (int ck = cg; ck < nck; ck += kOUTQ) {
            const int nval = p.C3 - ck * 16;
            const float* tg = p.target + b * p.out_bs + ((int64_t)o * p.C3 + ck * 16) * stride + v;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (nval >= 16 || e < nval) prefetch_l2(tg + (int64_t)e * stride);
          }
        }
        if (!KOUT) {
          idle_wait<1>(&bars.d3_full[xb], (n3 >> 1) & 1);
          fence_after();
        }
        const uint32_t d3 = tq + p.colD3 + (KOUT ? (uint32_t)(o * p.N3) : xb * (uint32_t)p.N3);
        for (int c0 = cg; c0 < nck; c0 += kOB2h * kOUTQ) {
          uint32_t r[kOB2h][16];
#pragma unroll
          for (int k = 0; k < kOB2h; ++k)
            if (c0 + k * kOUTQ < nck) tmem_ld<16>(d3 + (uint32_t)(c0 + k * kOUTQ) * 16, r[k]);
          tmem_wait_ld();
          if (c0 + kOB2h * kOUTQ >= nck) {
            fence_before();
            warp_arrive(KOUT ? &bars.d3g_free[o] : &bars.d3_free[xb]);
          }
#pragma unroll
          for (int k = 0; k < kOB2h; ++k) {
            const int ck = c0 + k * kOUTQ;
            if (tring && ck < nck) {   // this chunk's target is in ring stage tq_use & 1; start the next copy
              t_issue();
              cp_async_wait<1>();
              __syncwarp();   // the 8-byte path reads values other lanes copied
            }
            if (ck >= nck || !vok || !p.out) {
              if (tring && ck < nck) ++tq_use;
              continue;
            }
            const int64_t off = b * p.out_bs + ((int64_t)o * p.C3 + ck * 16) * stride + v;
            float* d = p.out + off;
            const int nval = p.C3 - ck * 16;
            const float* bb = sb + o * p.N3 + ck * 16;
            if (tring) {   // fused MSE from the target ring: d(loss)/dy and the squared residuals
              const float* tv = tr + (tq_use & 1) * 512 + lane;
              ++tq_use;
              float csum = 0.f;   // 16 squares in fp32, then one float64 add per chunk
              if (nval >= 16) {   // full chunk: as the plain path below
                const uint32_t rs = (uint32_t)stride * 4u;
                char* dc = reinterpret_cast<char*>(d);
#pragma unroll
                for (int h = 0; h < 16; h += 4) {
                  const float4 b4 = *reinterpret_cast<const float4*>(bb + h);
                  const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float res = fmaf(__uint_as_float(r[k][h + e]), isc, bv[e]) - tv[(h + e) * 32];
                    csum = fmaf(res, res, csum);
                    __stcs(reinterpret_cast<float*>(dc), res * p.out_scale);
                    dc += rs;
                  }
                }
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  if (e < nval) {
                    const float res = fmaf(__uint_as_float(r[k][e]), isc, bb[e]) - tv[e * 32];
                    csum = fmaf(res, res, csum);
                    __stcs(d, res * p.out_scale);
                  }
                  d += stride;
                }
              }
              lacc += (double)csum;
            } else if (p.target) {   // fused MSE: d(loss)/dy, and the squared residuals
              // all 16 target loads first: the stores below could alias them, so loads interleaved with
              // stores would each wait out a full memory latency
              const float* tg = p.target + off;
              float csum = 0.f;   // 16 squares in fp32, then one float64 add per chunk
#pragma unroll
              for (int h = 0; h < 16; h += 4) {   // four loads in flight at a time (register budget)
                float tv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  tv[e] = (nval >= 16 || h + e < nval) ? __ldcs(tg + (int64_t)(h + e) * stride) : 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  if (nval >= 16 || h + e < nval) {
                    const float res = fmaf(__uint_as_float(r[k][h + e]), isc, bb[h + e]) - tv[e];
                    csum = fmaf(res, res, csum);
                    __stcs(d, res * p.out_scale);
                  }
                  d += stride;
                }
              }
              lacc += (double)csum;
            } else if (nval >= 16) {
              // full chunk: no per-row predicate, one 128-bit bias load per four rows, and the row pointer
              // bumped by a 32-bit byte stride (the predicated form costs ~8 instructions per row)
              const uint32_t rs = (uint32_t)stride * 4u;
              char* dc = reinterpret_cast<char*>(d);
#pragma unroll
              for (int h = 0; h < 16; h += 4) {
                const float4 b4 = *reinterpret_cast<const float4*>(bb + h);
                const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  __stcs(reinterpret_cast<float*>(dc), fmaf(__uint_as_float(r[k][h + e]), isc, bv[e]));
                  dc += rs;
                }
              }
            } else {   // the shell's last, partial chunk: the same addressing, rows predicated
              const uint32_t rs = (uint32_t)stride * 4u;
              char* dc = reinterpret_cast<char*>(d);
#pragma unroll
              for (int h = 0; h < 16; h += 4) {
                const float4 b4 = *reinterpret_cast<const float4*>(bb + h);   // bias rows are padded to N3
                const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  if (h + e < nval) __stcs(reinterpret_cast<float*>(dc), fmaf(__uint_as_float(r[k][h + e]), isc, bv[e]));
                  dc += rs;
                }
              }
            }
          }
        }
      }
    }
    if (tring) cp_async_wait<0>();
    if (p.target) loss_publish(p.loss, lacc);
    }
  } else if (warp == kW3MMA || warp == kW3MMA2) {
    // =========================== MMA issuers ===========================
    const uint32_t sw1 = smem_u32(smem + p.sm_w1), sw2 = smem_u32(smem + p.sm_w2);
    const int km = p.adjoint ? 0 : 1;   // stage 1 as chain3v; the folded T images are always K-major
    const uint32_t id1 = idesc_f16(128, p.N1, 0, 1 - km);
    const uint32_t id2 = idesc_f16(128, p.N3, 0, 0);
    const int c1 = km ? p.K1 : p.N1;
    const uint64_t ks1 = wkstep(c1, km), ks2 = wkstep(K2, 1);
    const uint32_t nmine = ntiles > (int64_t)blockIdx.x ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    if (warp == kW3MMA) {
      uint64_t B1[PARTS];
#pragma unroll
      for (int j = 0; j < PARTS; ++j) B1[j] = wdesc(sw1 + (uint32_t)(j * p.w1_groups) * p.w1_img, c1, km, 0);
      const uint64_t g1s = p.w1_groups > 1 ? (uint64_t)(p.w1_img >> 4) : 0;
      const uint32_t tA = tbase + p.colA, tD1 = tbase + p.colD1;
      uint32_t aslot = 0, around = 0, aaddr = tA, gq = 0;
      for (uint32_t it = 0; it < nmine; ++it) {
        for (int g = 0; g < p.G1; ++g, ++gq) {
          const uint32_t nb = p.G1 >= 2 ? 2u : 1u, buf = gq % nb;
          if (gq >= nb) {
            mbar_wait_warp(&bars.d1g_free[buf], ((gq / nb) - 1) & 1);
            fence_after();
          }
          const uint32_t d1col = tD1 + buf * (uint32_t)p.N1;
          uint64_t bd[PARTS];
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bd[j] = B1[j] + (uint64_t)g * g1s;
          for (int k = 0; k < nk1; k += p.cpi) {
            mbar_wait_warp(&bars.a_full[aslot], around & 1);
            fence_after();
            if (elect_one()) {
              kstep_ts<PARTS>(d1col, aaddr, 8, bd, id1, k == 0);
              if (p.cpi == 2) {
                uint64_t bn[PARTS];
#pragma unroll
                for (int j = 0; j < PARTS; ++j) bn[j] = bd[j] + ks1;
                kstep_ts<PARTS>(d1col, aaddr + kSlotW, 8, bn, id1, false);
              }
              commit(&bars.a_empty[aslot]);
              if (k + p.cpi >= nk1) commit(&bars.d1g_full[buf]);
            }
            __syncwarp();
            if (++aslot == (uint32_t)p.NA) {
              aslot = 0;
              ++around;
              aaddr = tA;
            } else {
              aaddr += (uint32_t)p.cpi * kSlotW;
            }
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] += (uint64_t)p.cpi * ks1;
          }
        }
      }
    } else if constexpr (!GONLY) {
      // stage 2: T_o images, part-major (term j of group o at j * w2_img, group o rows o * N3 .. of a G2*N3 x K2 image)
      uint64_t B2[PARTS];
#pragma unroll
      for (int j = 0; j < PARTS; ++j) B2[j] = wdesc(sw2 + (uint32_t)j * p.w2_img, K2, 1, 0);
      const uint64_t o2s = wdesc(0, K2, 1, p.N3) - wdesc(0, K2, 1, 0);
      const uint32_t tg = (uint32_t)(p.N3 * K2 * 2);   // one shell's rows of one term image
      const uint32_t tA2 = tbase + p.colA2, tD3 = tbase + p.colD3;
      uint32_t n3 = 0;
      if constexpr (KOUT) {
        uint32_t ci = 0;
        for (uint32_t it = 0; it < nmine; ++it) {
          uint64_t bk[PARTS];
#pragma unroll
          for (int j = 0; j < PARTS; ++j) bk[j] = B2[j];
          for (int k = 0; k < nk2; ++k, ++ci) {
            const uint32_t slot = ci % (uint32_t)p.NAc, round = ci / (uint32_t)p.NAc;
            mbar_wait_warp(&bars.c_full[slot], round & 1);
            fence_after();
            uint64_t bd[PARTS];
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] = bk[j];
            for (int o = 0; o < p.G2; ++o) {
              if (k == 0 && it > 0) {   // OUT has drained shell o of the previous tile
                mbar_wait_warp(&bars.d3g_free[o], (it - 1) & 1);
                fence_after();
              }
              if (elect_one()) kstep_ts<PARTS>(tD3 + (uint32_t)(o * p.N3), tA2 + slot * kSlotW, 8, bd, id2, k == 0);
              __syncwarp();
#pragma unroll
              for (int j = 0; j < PARTS; ++j) bd[j] += o2s;
            }
            if (elect_one()) {
              commit(&bars.c_empty[slot]);
              if (k == nk2 - 1) commit(&bars.d3_full[0]);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bk[j] += ks2;
          }
        }
      } else
      for (uint32_t it = 0; it < nmine; ++it) {
        const uint32_t n3b = it * (uint32_t)p.G2;   // the CTA-wide index of this tile's shell 0
        // shell o: wait for its D3 buffer (and T image), return the buffer; bd = its T descriptors at item 0
        auto shell_begin = [&](int o, uint64_t (&bd)[PARTS]) -> uint32_t {
          const uint32_t n = n3b + (uint32_t)o, xb = n & 1;
          if (n >= 2) {
            mbar_wait_warp(&bars.d3_free[xb], ((n >> 1) - 1) & 1);
            fence_after();
          }
          if (p.tstream) {   // this shell's T image in buffer n & 1 (rows 0.. of the buffer)
            mbar_wait_warp(&bars.t_full[xb], (n >> 1) & 1);
#pragma unroll
            for (int j = 0; j < PARTS; ++j)
              bd[j] = wdesc(sw2 + xb * (uint32_t)PARTS * tg + (uint32_t)j * tg, K2, 1, 0);
          } else {
#pragma unroll
            for (int j = 0; j < PARTS; ++j) bd[j] = B2[j] + (uint64_t)o * o2s;
          }
          return tD3 + xb * (uint32_t)p.N3;
        };
        // items k0..k1-1 of shell o into d3 (k == kfirst overwrites the accumulator)
        auto run_items = [&](int o, uint32_t d3, const uint64_t (&bd)[PARTS], int k0, int k1, int kfirst) {
          for (int k = k0; k < k1; ++k) {
            if (o == 0 || DIAG) {   // the item's first reader in this tile
              mbar_wait_warp(&bars.a2_full[k], it & 1);
              fence_after();
            }
            if (elect_one()) {
              uint64_t bk[PARTS];
#pragma unroll
              for (int j = 0; j < PARTS; ++j) bk[j] = bd[j] + (uint64_t)k * ks2;
              kstep_ts<PARTS>(d3, tA2 + (uint32_t)k * kSlotW, 8, bk, id2, k == kfirst);
              if (kA2Item && (o == p.G2 - 1 || DIAG)) commit(&bars.a2_ifree[k]);   // CONV may overwrite item k
            }
            __syncwarp();
          }
        };
        auto shell_end = [&](int o) {
          const uint32_t xb = (n3b + (uint32_t)o) & 1;
          if (elect_one()) {
            commit(&bars.d3_full[xb]);
            if (p.tstream) commit(&bars.t_empty[xb]);
            if (!kA2Item && o == p.G2 - 1) commit(&bars.a2_free);
          }
          __syncwarp();
        };
        int o = 0;
        if (!DIAG && kDefer > 0 && p.G2 >= 2 && nk2 > kDefer) {
          // shells 0 and 1 interleaved: both run their first nk2 - kDefer items before either reads the last
          // ones, so the items the previous tile's last shell frees last have twice the slack to be refilled
          uint64_t b0[PARTS], b1[PARTS];
          const uint32_t d0 = shell_begin(0, b0);
          run_items(0, d0, b0, 0, nk2 - kDefer, 0);
          const uint32_t d1 = shell_begin(1, b1);
          run_items(1, d1, b1, 0, nk2 - kDefer, 0);
          run_items(0, d0, b0, nk2 - kDefer, nk2, 0);
          shell_end(0);
          run_items(1, d1, b1, nk2 - kDefer, nk2, 0);
          shell_end(1);
          o = 2;
        }
        for (; o < p.G2; ++o) {
          uint64_t bd[PARTS];
          const uint32_t d3 = shell_begin(o, bd);
          // block-diagonal T (round trip): only input group o's items, each read by this shell alone
          // (a compile-time switch: a runtime one in this loop costs the dense chain ~4% of its time)
          const int kb = DIAG ? o * (nk2 / p.G2) : 0, ke = DIAG ? kb + nk2 / p.G2 : nk2;
          run_items(o, d3, bd, kb, ke, kb);
          shell_end(o);
        }
      }
    }
  } else if (warp == kW3LD) {
    if (p.tma)
      tma_loader<NS>(geo, per_tile, ntiles, p.tiles_per_b, p.nvox, p.tm, smem + p.sm_ring, bars.full, bars.empty);
  } else if (!GONLY && p.tstream) {
    // =========================== T-image loader: shell o's rows of both term images, two buffers ===========
    const uint32_t tg = (uint32_t)(p.N3 * K2 * 2);
    const uint32_t nmine = ntiles > (int64_t)blockIdx.x ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    uint32_t n = 0;
    for (uint32_t it = 0; it < nmine; ++it)
      for (int o = 0; o < p.G2; ++o, ++n) {
        const uint32_t b = n & 1;
        if (n >= 2) mbar_wait_warp(&bars.t_empty[b], ((n >> 1) - 1) & 1);
        if (elect_one()) {
          uint8_t* dst = smem + p.sm_w2 + b * 2u * tg;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(p.w2) + (size_t)o * tg;
          mbar_arrive_tx(&bars.t_full[b], 2u * tg);
          bulk_g2s(dst, src, tg, &bars.t_full[b]);
          bulk_g2s(dst + tg, src + p.w2_img, tg, &bars.t_full[b]);
        }
        __syncwarp();
      }
  }
  fence_before();
  __syncthreads();
  if (warp == kW3MMA) tmem_dealloc(tbase, 512);
  ktrace_end(p.kt, p.kt_slot);
}

// ============================================================================ LSC weight Gram
// G[j][i] = sum_v g_v[j] c_v[i] over this CTA's voxels.  c = M x is written by the forward chain kernel
// and g = B'^T dy by the adjoint, both as two-term bf16 planes (hi, next term) with rows padded per shell
// to 16 and voxels padded to 64 (zeros).  Those planes are exactly the operands: a TMA ring streams one
// 64-voxel tile (c hi | c lo | g hi | g lo, SWIZZLE_128B K-major: row = channel, K = voxel) per stage and
// the MMA warp accumulates the three split products in TMEM -- no conversion warps.
// c's first padding row holds 1.0, so G's column `ones` is sum_v g_v: the bias gradient comes out of
// the same MMAs.
// Accuracy: the tensor core's fp32 accumulation is not round-to-nearest, and its error grows with the
// accumulation length (measured at cfg4: dW error 8.6e-5 with one TMEM accumulation per CTA over ~24.7k
// voxels, halving with every halving of the run; scripts/gram_precision.py).  So the MMA accumulates only
// kGGroup tiles into one of two TMEM accumulators, and the 4 epilogue warps drain the finished one into
// round-to-nearest fp32 registers (lane = G row) while the MMA fills the other; the registers are written
// once as the CTA's partial.
constexpr int kGV = 64;                  // voxels per Gram tile (one 128-byte bf16 K atom)
constexpr int kGGroup = 8;               // tiles per TMEM accumulation run (512 voxels)
constexpr int kGEpi = 4;                 // epilogue warps (one per TMEM lane quadrant)
constexpr int kGWarpMMA = kGEpi;
constexpr int kGWarpLD = kGEpi + 1;
constexpr int kGThreads = (kGWarpLD + 1) * 32;
constexpr int kGAccCols = 256;           // one accumulator: block A (<= 144) | block B (16) | block C (16)

struct GramP {
  CUtensorMap tm[2];         // bf16 term planes of g (0) and c (1): dims (pitch, rows, 2 terms, nbatch)
  float* partials;           // [grid][GR*GC]
  int64_t nbatch, tiles_per_b;
  int GR, GC;
  int ns;
  uint32_t cpart, gpart, stage_bytes;   // stage: c hi | c lo | g hi | g lo
  uint32_t sm_ring, sm_bar, smem_bytes;
  uint32_t colGA, colGB, colGC;         // within one accumulator
  dl::KTrace* kt;                       // kernel timer (dl_ktimer_*, slot 2) or null
};

struct BarsG {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

template <int NS>
__global__ void __launch_bounds__(kGThreads, 1) gram_tc(const __grid_constant__ GramP p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  ktrace_begin(p.kt, 2);
  BarsG& bars = *reinterpret_cast<BarsG*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    // g rows GR..127 (block A's M padding) are never loaded: zero them once in every stage
    uint4* z = reinterpret_cast<uint4*>(smem + p.sm_ring);
    for (uint32_t i = threadIdx.x; i < NS * p.stage_bytes / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (warp == kGWarpMMA) tmem_alloc(&bars.tmem_base, 2 * kGAccCols);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.acc_full[b], 1);
      mbar_init(&bars.acc_empty[b], kGEpi);
    }
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;
  const uint32_t nmine = ntiles > (int64_t)blockIdx.x ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
  const uint32_t ngroups = (nmine + kGGroup - 1) / kGGroup;

  if (warp == kGWarpLD) {
    // =========================== TMA loader ===========================
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&p.tm[0]) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&p.tm[1]) : "memory");
    }
    __syncwarp();
    uint32_t s = 0, round = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      if (round > 0) mbar_wait_warp(&bars.empty[s], (round - 1) & 1);
      if (elect_one()) {
        uint8_t* st = smem + p.sm_ring + s * p.stage_bytes;
        mbar_arrive_tx(&bars.full[s], 2 * (uint32_t)(p.GC + p.GR) * 128u);
        tma_load_4d(st, &p.tm[1], 0, 0, 0, (int)t, &bars.full[s]);   // t = b * tiles_per_b + tile
        tma_load_4d(st + p.cpart, &p.tm[1], 0, 0, 1, (int)t, &bars.full[s]);
        tma_load_4d(st + 2 * p.cpart, &p.tm[0], 0, 0, 0, (int)t, &bars.full[s]);
        tma_load_4d(st + 2 * p.cpart + p.gpart, &p.tm[0], 0, 0, 1, (int)t, &bars.full[s]);
      }
      __syncwarp();
      if (++s == NS) {
        s = 0;
        ++round;
      }
    }
  } else if (warp == kGWarpMMA) {
    // =========================== MMA: G += g^T c, three split products, three blocks ===========================
    const uint32_t idA = idesc_bf16(128, p.GC, 0, 0), idB = idesc_bf16(128, 16, 0, 0), idC = idesc_bf16(64, 16, 0, 0);
    const uint32_t ring = smem_u32(smem + p.sm_ring);
    uint32_t s = 0, round = 0;
    for (uint32_t it = 0; it < nmine; ++it) {
      const uint32_t gi = it / kGGroup, buf = gi & 1;
      const bool first = it % kGGroup == 0;
      if (first && gi >= 2) {   // the epilogue has drained this accumulator's previous run
        mbar_wait_warp(&bars.acc_empty[buf], ((gi >> 1) - 1) & 1);
        fence_after();
      }
      const uint32_t acc0 = tbase + buf * kGAccCols;
      mbar_wait_warp(&bars.full[s], round & 1);
      fence_after();
      const uint32_t c0 = ring + s * p.stage_bytes, g0 = c0 + 2 * p.cpart;
      for (int kk = 0; kk < kGV / 16; ++kk) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int i = Pairs<2>::i(k), j = Pairs<2>::j(k);
            const uint32_t gI = g0 + (uint32_t)i * p.gpart + kk * 32u, gJ = g0 + (uint32_t)j * p.gpart + kk * 32u;
            const uint32_t cI = c0 + (uint32_t)i * p.cpart + kk * 32u, cJ = c0 + (uint32_t)j * p.cpart + kk * 32u;
            const uint32_t acc = (!first || kk > 0 || k > 0) ? 1u : 0u;
            mma_ss(acc0 + p.colGA, desc_sw128_k(gI, 1024), desc_sw128_k(cJ, 1024), idA, acc);
            if (p.GR > 128) {
              mma_ss(acc0 + p.colGB, desc_sw128_k(cI, 1024), desc_sw128_k(gJ + 16 * 1024, 1024), idB, acc);
              if (p.GC > 128)
                mma_ss(acc0 + p.colGC, desc_sw128_k(cI + 16 * 1024, 1024), desc_sw128_k(gJ + 16 * 1024, 1024), idC,
                       acc);
            }
          }
        }
        __syncwarp();
      }
      if (elect_one()) {
        commit(&bars.empty[s]);
        if (it % kGGroup == kGGroup - 1 || it + 1 == nmine) commit(&bars.acc_full[buf]);
      }
      __syncwarp();
      if (++s == NS) {
        s = 0;
        ++round;
      }
    }
  } else {
    // =========================== epilogue: drain each run into fp32 registers, then the CTA's partial ===========
    const int qd = warp & 3, row = 32 * qd + lane;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int nck = p.GC / 16;
    float ga[9][16], gb[16], gc[16];   // block A row (lane = g row), block B (lane = c row), block C
#pragma unroll
    for (int c = 0; c < 9; ++c)
#pragma unroll
      for (int e = 0; e < 16; ++e) ga[c][e] = 0.f;
#pragma unroll
    for (int e = 0; e < 16; ++e) gb[e] = gc[e] = 0.f;
    for (uint32_t gi = 0; gi < ngroups; ++gi) {
      const uint32_t buf = gi & 1, acc0 = tq + buf * kGAccCols;
      mbar_wait_warp(&bars.acc_full[buf], (gi >> 1) & 1);
      fence_after();
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        if (c < nck) {
          uint32_t r[16];
          tmem_ld<16>(acc0 + p.colGA + (uint32_t)c * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) ga[c][e] += __uint_as_float(r[e]);
        }
      }
      if (p.GR > 128) {
        uint32_t r[16];
        tmem_ld<16>(acc0 + p.colGB, r);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) gb[e] += __uint_as_float(r[e]);
        if (p.GC > 128) {   // block C (M = 64) lives in lanes 0..15 of quadrant 0; every warp loads (aligned)
          tmem_ld<16>(acc0 + p.colGC, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) gc[e] += __uint_as_float(r[e]);
        }
      }
      fence_before();
      warp_arrive(&bars.acc_empty[buf]);
    }
    float* part = p.partials + (int64_t)blockIdx.x * p.GR * p.GC;
    if (row < p.GR)   // block A: lane = g row, column = c row
#pragma unroll
      for (int c = 0; c < 9; ++c)
        if (c < nck)
#pragma unroll
          for (int e = 0; e < 16; ++e) part[(int64_t)row * p.GC + c * 16 + e] = ga[c][e];
    if (p.GR > 128) {
      if (row < p.GC)   // block B: lane = c row i (< 128), column = g row 128 + e
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (128 + e < p.GR) part[(int64_t)(128 + e) * p.GC + row] = gb[e];
      if (p.GC > 128 && qd == 0 && lane < 16 && 128 + lane < p.GC)   // block C: lanes 0..15 = c rows 128..143
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (128 + e < p.GR) part[(int64_t)(128 + e) * p.GC + 128 + lane] = gc[e];
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kGWarpMMA) tmem_dealloc(tbase, 2 * kGAccCols);
  ktrace_end(p.kt, 2);
}

// ---------------------------------------------------------------------------- operand packing
// `ng` row-major fp32 matrices of (nrb*rb) x (ncb*cb) -> PARTS bf16 images each of (nrb*rbp) x (ncb*cbp)
// in the core-matrix blocked layout, image (q, g) at (q * ng + g) * img_elems.  Padding is zero.
// out_h (optional): the same images as two fp16 terms (the fp16 chain pass).
struct PackJob {
  const float* W;
  uint16_t* out;
  uint16_t* out_h;
  int ng, nrb, rb, rbp, ncb, cb, cbp, parts;
};
struct PackJobs {
  PackJob j[3];
};

__device__ __forceinline__ void pack_job(const PackJob& jb) {
  const float* __restrict__ W = jb.W;
  uint16_t* __restrict__ out = jb.out;
  uint16_t* __restrict__ out_h = jb.out_h;
  const int ng = jb.ng, nrb = jb.nrb, rb = jb.rb, rbp = jb.rbp, ncb = jb.ncb, cb = jb.cb, cbp = jb.cbp;
  const int parts = jb.parts;
  const int R = nrb * rbp, C = ncb * cbp;
  const int64_t img = (int64_t)R * C;
  const int64_t n = img * ng;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(e / img);
    const int rc = (int)(e - (int64_t)g * img);
    const int r = rc / C, c = rc - r * C;
    const int bi = r / rbp, rr = r - bi * rbp, bj = c / cbp, cc = c - bj * cbp;
    float v = 0.f;
    if (rr < rb && cc < cb)
      v = __ldg(W + (int64_t)g * (nrb * rb) * (ncb * cb) + (int64_t)(bi * rb + rr) * (ncb * cb) + bj * cb + cc);
    const int64_t off = ((int64_t)(r >> 3) * (C >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7);
    if (out_h) {
      float u = v;
      for (int q = 0; q < 2; ++q) {
        const uint32_t pk = pack_f16x2(u, 0.f);
        out_h[((int64_t)q * ng + g) * img + off] = (uint16_t)(pk & 0xFFFFu);
        u -= f16lo_to_f32(pk);
      }
    }
    for (int q = 0; q < parts; ++q) {
      const uint32_t pk = pack_bf16x2(v, 0.f);
      out[((int64_t)q * ng + g) * img + off] = (uint16_t)(pk & 0xFFFFu);
      v -= bf16lo_to_f32(pk);
    }
  }
}

// one launch packs up to three operator images (blockIdx.y = job)
__global__ void pack_k(PackJobs jobs) { pack_job(jobs.j[blockIdx.y]); }

// Folded stage-2 operator of chain2h (float64 accumulation, fp32 result):
//   forward  T[(o, n), (s, r)] = sum_q B'[n, q] L[(o, q), (s, r)],   bias3[(o, n)] = sum_q B'[n, q] bvec[(o, q)]
//   adjoint  T[(s, i), (o, q)] = sum_r M_s[r, i] L[(o, q), (s, r)]
// L is (s_out r_out) x (s_in r_in), B' n_out x r_out, M (mg, r_in, n).
__global__ void fold_t_k(const float* __restrict__ L, const float* __restrict__ Bt, const float* __restrict__ M,
                         const float* __restrict__ bvec, float* __restrict__ T, float* __restrict__ bias3, int adjoint,
                         int s_in, int s_out, int r_in, int r_out, int n, int n_out, int mg) {
  const int rows = adjoint ? s_in * n : s_out * n_out, cols = adjoint ? s_out * r_out : s_in * r_in;
  const int LC = s_in * r_in;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols + (adjoint ? 0 : rows);
       e += gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (e >= rows * cols) {   // folded bias (forward)
      const int rr = e - rows * cols, o = rr / n_out, nn = rr - o * n_out;
      if (bvec)
        for (int q = 0; q < r_out; ++q) acc += (double)Bt[nn * r_out + q] * (double)bvec[o * r_out + q];
      bias3[rr] = (float)acc;
      continue;
    }
    const int row = e / cols, col = e - row * cols;
    if (!adjoint) {
      const int o = row / n_out, nn = row - o * n_out;
      for (int q = 0; q < r_out; ++q) acc += (double)Bt[nn * r_out + q] * (double)L[(int64_t)(o * r_out + q) * LC + col];
    } else {
      const int sh = row / n, i = row - sh * n, o = col / r_out, q = col - o * r_out;
      const float* Ms = M + (int64_t)(mg > 1 ? sh : 0) * r_in * n;
      for (int r = 0; r < r_in; ++r) acc += (double)Ms[r * n + i] * (double)L[(int64_t)(o * r_out + q) * LC + sh * r_in + r];
    }
    T[e] = (float)acc;
  }
}

// G[e] = sum over the gram_tc parts of partials[q][e], in float64.  Block (32, 8): lane x takes one e, row y a
// contiguous chunk of parts (eight loads in flight); the eight chunk sums are added in chunk order, so the
// result is fixed for a given part count (deterministic run to run).
__global__ void __launch_bounds__(256) gram_reduce_k(const float* __restrict__ partials, double* __restrict__ G,
                                                     int nparts, int n) {
  __shared__ double red[8][33];
  const int e = blockIdx.x * 32 + threadIdx.x;
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

// dW[o,s,k] = <P_k, G_{o,s}> and db[o] = beta . G[o-block rows][ones column] (= beta . sum_v g_v), in float64
__global__ void gram_finalize_k(const double* __restrict__ G, const float* __restrict__ beta, int ones,
                                const float* __restrict__ P, float* __restrict__ dW, float* __restrict__ db, int s_out,
                                int s_in, int K, int r_out, int r_in, int RPo, int RPi) {
  __shared__ double red[32];
  const int GC = s_in * RPi;
  const int nw = s_out * s_in * K;
  const int id = blockIdx.x;
  double acc = 0.0;
  if (id < nw) {
    const int o = id / (s_in * K), s = (id / K) % s_in, k = id % K;
    for (int e = threadIdx.x; e < r_out * r_in; e += blockDim.x) {
      const int r = e / r_in, t = e - r * r_in;
      acc += (double)__ldg(P + ((int64_t)k * r_out + r) * r_in + t) * G[(int64_t)(o * RPo + r) * GC + s * RPi + t];
    }
  } else {
    const int o = id - nw;
    for (int r = threadIdx.x; r < r_out; r += blockDim.x)
      acc += (double)__ldg(beta + r) * G[(int64_t)(o * RPo + r) * GC + ones];
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) {
      if (id < nw) {
        if (dW) dW[id] = (float)v;
      } else if (db) {
        db[id - nw] = (float)v;
      }
    }
  }
}

}  // namespace tc
}  // namespace dl

// ============================================================================ host side
namespace dl {
namespace tc {
namespace {

inline int r16(int64_t x) { return (int)((x + 15) / 16 * 16); }
inline size_t al(size_t x, size_t a) { return (x + a - 1) / a * a; }
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kMaxParts = 592;    // Gram partials: up to 4 waves of 148 CTAs (gram_waves)

// CTAs per SM-slot of the Gram (DELIMIT_GRAM_WAVES, read per call): each CTA accumulates its share of the voxel
// tiles in fp32 TMEM and writes one partial, so more waves mean shorter fp32 accumulation runs (the partials
// are summed in float64 by gram_reduce_k).
int gram_waves() {
  const char* e = getenv("DELIMIT_GRAM_WAVES");
  const int v = e ? atoi(e) : 1;
  return v < 1 ? 1 : v > 4 ? 4 : v;
}

long long* g_prof = nullptr;   // debug: phase timestamps of the next chain3 forward launch

// Operand precision of the chain kernels (DELIMIT_SPLIT_TERMS): unset (default) = fp16 two-term pass under
// delayed scaling, checked and if needed redone by a 3-term bf16 pass; "3" = 3-term bf16 only; "2" = 2-term
// bf16 only (~3e-5 relative error, below the fp32-class bar; a measurement mode).
int split_terms() {
  static int v = [] {
    const char* e = getenv("DELIMIT_SPLIT_TERMS");
    const int t = e ? atoi(e) : 3;
    return (t == 2 || t == 3) ? t : 3;
  }();
  return v;
}
bool fp16_pass() {
  static const bool v = getenv("DELIMIT_SPLIT_TERMS") == nullptr;
  return v;
}

struct Dims {
  int64_t nbatch, nvox;
  int s_in, s_out, n, r_in, r_out, n_out, mg;
  int NPi, RPi, RPo, NPo, parts;
};

Dims make_dims(int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
               int64_t nvox, int m_per_shell) {
  Dims d;
  d.nbatch = nbatch;
  d.nvox = nvox;
  d.s_in = (int)s_in;
  d.s_out = (int)s_out;
  d.n = (int)n;
  d.r_in = (int)r_in;
  d.r_out = (int)r_out;
  d.n_out = (int)n_out;
  d.mg = m_per_shell ? (int)s_in : 1;
  d.NPi = r16(n);
  d.RPi = r16(r_in);
  d.RPo = r16(r_out);
  d.NPo = r16(n_out);
  d.parts = split_terms();
  return d;
}

struct WsLayout {
  size_t imgM, imgL, imgB, imgMh, imgLh, imgBh, Tf, b3, imgTh, parts, G, total;
};

WsLayout ws_layout(const Dims& d, int nparts) {
  WsLayout w;
  const size_t bM = (size_t)d.RPi * d.NPi * 2, bL = (size_t)(d.s_out * d.RPo) * (d.s_in * d.RPi) * 2,
               bB = (size_t)d.NPo * d.RPo * 2;
  const size_t GR = (size_t)d.s_out * d.RPo, GC = (size_t)d.s_in * d.RPi;
  size_t o = 0;
  w.imgM = o; o = al(o + 3 * d.mg * bM, 256);
  w.imgL = o; o = al(o + 3 * bL, 256);
  w.imgB = o; o = al(o + 3 * bB, 256);
  w.imgMh = o; o = al(o + 2 * d.mg * bM, 256);   // fp16 two-term images
  w.imgLh = o; o = al(o + 2 * bL, 256);
  w.imgBh = o; o = al(o + 2 * bB, 256);
  // chain2h: folded operator (fp32, larger of the two directions), its bias, and its fp16 image
  const size_t tf = std::max((size_t)d.s_out * d.n_out * d.s_in * d.r_in, (size_t)d.s_in * d.n * d.s_out * d.r_out);
  const size_t ti = std::max((size_t)d.s_out * d.NPo * d.s_in * d.RPi, (size_t)d.s_in * d.NPi * d.s_out * d.RPo) * 2;
  w.Tf = o; o = al(o + tf * 4, 256);
  w.b3 = o; o = al(o + (size_t)d.s_out * d.n_out * 4, 256);
  w.imgTh = o; o = al(o + 2 * ti, 256);
  w.parts = o; o = al(o + (size_t)nparts * (GR * GC + d.s_out) * 4, 256);
  w.G = o; o = al(o + GR * GC * 8, 256);
  w.total = o;
  return w;
}

// TMEM / shared-memory plan for one chain3 direction; false if it does not fit.
// Regions: A slots | D1 | A2 | D2 (+ A3, D3).  Lifetimes inside a tile: D1 until A2 is built, A2 until
// the stage-2 MMAs finish, D2 through the last stage-3 read, A3/D3 during stage 3.  A3/D3 may reuse
// a dead region (A2 or D1) but never D2 or the A slots.  "overlap": D1/slots are free as soon as A2 is
// built, so the next tile's stage 1 runs during this tile's stage 3.  free_at tells MID when to
// release D1 (0: after A2 is built, 1: after the last D2 read, 2: after the last D3 read).
bool plan_tmem(Chain3& p, int parts) {
  const int slotw = parts * 8, D1w = p.G1 * p.N1, A2w = parts * D1w / 2, D2w = p.G2 * p.N2, A3w = parts * p.N2 / 2,
            D3w = p.N3, S3 = A3w + D3w;
  for (int na = 4; na >= 2; --na) {
    p.NA = na;
    p.colA = 0;
    p.colD1 = na * slotw;
    p.colA2 = p.colD1 + D1w;
    if ((int)p.colA2 + A2w > 512) continue;
    // overlap layouts: D2 after A2; stage 3 inside A2 or after D2
    const int d2 = p.colA2 + A2w;
    if (d2 + D2w <= 512) {
      p.colD2 = d2;
      p.overlap = 1;
      p.free_at = 0;
      if (S3 <= A2w) { p.colA3 = p.colA2; p.colD3 = p.colA2 + A3w; return true; }
      if (d2 + D2w + S3 <= 512) { p.colA3 = d2 + D2w; p.colD3 = p.colA3 + A3w; return true; }
      // compact variant of the same D2 placement: stage 3 in the (dead, contiguous) D1 + A2 regions
      if (S3 <= D1w + A2w) { p.overlap = 0; p.free_at = 2; p.colA3 = p.colD1; p.colD3 = p.colD1 + A3w; return true; }
    }
    // compact: D2 aliases D1, stage 3 inside A2
    if (D2w <= D1w && S3 <= A2w) {
      p.colD2 = p.colD1;
      p.overlap = 0;
      p.free_at = 1;
      p.colA3 = p.colA2;
      p.colD3 = p.colA2 + A3w;
      return true;
    }
  }
  return false;
}

bool plan_chain3(Chain3& p, int parts) {
  if (p.N1 > 256 || p.N2 > 256 || p.N3 > 256 || p.G1 * p.N1 > 512) return false;
  if (!plan_tmem(p, parts)) return false;
  p.w1_img = (uint32_t)(p.N1 * p.K1 * 2);
  p.w2_img = (uint32_t)((p.G2 * p.N2) * (p.G1 * p.N1) * 2);
  p.w3_img = (uint32_t)(p.N3 * p.N2 * 2);
  size_t o = 0;
  p.sm_w1 = (uint32_t)o; o = al(o + (size_t)parts * p.w1_groups * p.w1_img, 1024);
  p.sm_w2 = (uint32_t)o; o = al(o + (size_t)parts * p.w2_img, 1024);
  p.sm_w3 = (uint32_t)o; o = al(o + (size_t)parts * p.w3_groups * p.w3_img, 1024);
  p.sm_bias = (uint32_t)o; o = al(o + (size_t)p.G2 * p.N2 * 4, 128);
  p.sm_ring = (uint32_t)o;   // TMA destinations: 128-byte aligned
  for (p.ns = 8; p.ns >= 2; p.ns /= 2) {   // cp.async ring depth per IN warp
    size_t q = al(p.sm_ring + (size_t)p.ns * kStageBytes, 16);
    p.sm_bar = (uint32_t)q;
    q = al(q + sizeof(Bars3), 16);
    p.smem_bytes = (uint32_t)q;
    if (q <= kSmemMax) return true;
  }
  return false;
}

// chain3v: D1 | D2 | D3 resident, IN ring (NA) + conversion ring (NAc) in the remaining columns.
bool plan_chain3v(Chain3& p, int parts) {
  if (p.N1 > 256 || p.N2 > 256 || p.N3 > 256 || p.G1 * p.N1 > 512) return false;
  // stage 1 accumulates one input group at a time into two alternating N1-column buffers
  const int slotw = parts * 8, D1w = (p.G1 >= 2 ? 2 : 1) * p.N1, D2w = p.G2 * p.N2, D3w = p.N3;
  const int nslots = (512 - D1w - D2w - D3w) / slotw;
  if (512 - D1w - D2w - D3w < 0 || nslots < 4) return false;
  // stage-1 input chunks are the most frequent handoff (18 per tile vs 9 + 9 conversions): IN gets the
  // larger half of the slot budget
  p.NA = (nslots + 1) / 2 < kMaxSlots ? (nslots + 1) / 2 : kMaxSlots;
  if (const char* e = getenv("DELIMIT_IN_SLOTS")) {   // tuning knob: IN-ring share of the slot budget
    const int v = atoi(e);
    if (v >= 2 && v <= nslots - 2) p.NA = v;
  }
  p.NAc = nslots - p.NA < kMaxSlots ? nslots - p.NA : kMaxSlots;
  if (p.NAc < kCVQ) {   // kCVQ CONV warps alternate items: the ring needs >= kCVQ slots (parity safety)
    p.NAc = kCVQ;
    p.NA = nslots - kCVQ;
  }
  if (p.NA < 2) return false;
  // two input chunks per IN item halve the stage-1 handoffs: needs an even chunk count per group, the
  // TMA path, and >= 2 double items (4 single slots)
  p.cpi = (p.tma && (p.K1 / 16) % 2 == 0 && p.NA >= 4 && !getenv("DELIMIT_IN_SINGLE")) ? 2 : 1;
  if (p.cpi == 2) p.NA /= 2;   // NA counts IN items from here on
  p.colA = 0;
  p.colC = (uint32_t)(p.NA * p.cpi * slotw);
  p.colD1 = p.colC + (uint32_t)(p.NAc * slotw);
  p.colD2 = p.colD1 + (uint32_t)D1w;
  p.colD3 = p.colD2 + (uint32_t)D2w;
  p.w1_img = (uint32_t)(p.N1 * p.K1 * 2);
  p.w2_img = (uint32_t)((p.G2 * p.N2) * (p.G1 * p.N1) * 2);
  p.w3_img = (uint32_t)(p.N3 * p.N2 * 2);
  size_t o = 0;
  p.sm_w1 = (uint32_t)o; o = al(o + (size_t)parts * p.w1_groups * p.w1_img, 1024);
  p.sm_w2 = (uint32_t)o; o = al(o + (size_t)parts * p.w2_img, 1024);
  p.sm_w3 = (uint32_t)o; o = al(o + (size_t)parts * p.w3_groups * p.w3_img, 1024);
  p.sm_bias = (uint32_t)o; o = al(o + (size_t)p.G2 * p.N2 * 4, 128);
  p.sm_ring = (uint32_t)o;
  // even depths: two IN warps take alternate chunks, so each stage keeps one fixed consumer pair
  // (two-chunk items: multiples of 4)
  static const int max_ns = getenv("DELIMIT_MAX_NS") ? atoi(getenv("DELIMIT_MAX_NS")) : 12;   // tuning knob
  for (int ns : {12, 10, 8, 6, 4, 2}) {
    if ((p.cpi == 2 && ns % 4) || (ns > max_ns && ns > 2)) continue;
    p.ns = ns;
    size_t q = al(p.sm_ring + (size_t)p.ns * kStageBytes, 16);
    p.sm_bar = (uint32_t)q;
    q = al(q + sizeof(Bars3v), 16);
    p.smem_bytes = (uint32_t)q;
    if (q <= kSmemMax) return true;
  }
  return false;
}

bool use_2h() {
  static const bool v = getenv("DELIMIT_NO_CHAIN2H") == nullptr;
  return v;
}

// chain2h plan (fp16 pass, TMA input): TMEM = IN items | D1 x 2 | A2 (G1 N1) | D3 x 2; shared memory =
// stage-1 image | folded T images | folded bias | TMA ring (a multiple of 4 deep) | barriers.
bool plan_chain2h(Chain3& p, bool kout) {
  constexpr int parts = 2;
  // (nvox < 2^30: the OUT role steps between output rows by a 32-bit byte stride)
  if ((!p.tma && !p.raw) || p.N1 > 256 || p.N3 > 256 || (p.G1 * p.N1) / 16 > 16 || (p.K1 / 16) % 2 ||
      p.nvox >= (1LL << 30) ||
      (kout && (p.G2 > 4 || p.raw)))
    return false;
  const int D1w = (p.G1 >= 2 ? 2 : 1) * p.N1;
  const int D3w = kout ? p.G2 * p.N3 : 2 * p.N3;
  int A2w = p.G1 * p.N1;
  p.cpi = (getenv("DELIMIT_IN_SINGLE") || p.raw) ? 1 : 2;   // raw input: one chunk per item; else a measurement knob
  if (kout) {   // two IN items, the rest A2 ring slots (>= 2)
    p.NA = 2;
    p.NAc = (512 - D1w - D3w - 2 * 2 * parts * 8) / (parts * 8);
    if (p.NAc > kMaxSlots) p.NAc = kMaxSlots;
    if (p.NAc < 2) return false;
    A2w = p.NAc * parts * 8;
  } else {
    const int spare = 512 - D1w - A2w - D3w;
    p.NA = spare / (p.cpi * parts * 8);
    if (p.NA < 2) return false;
    if (p.NA > kMaxSlots) p.NA = kMaxSlots;
    p.NAc = 0;
  }
  if (D1w + A2w + D3w + p.NA * p.cpi * parts * 8 > 512) return false;
  p.colA = 0;
  p.colD1 = (uint32_t)(p.NA * p.cpi * parts * 8);
  p.colA2 = p.colD1 + (uint32_t)D1w;
  p.colD3 = p.colA2 + (uint32_t)A2w;
  p.w1_img = (uint32_t)(p.N1 * p.K1 * 2);
  p.w2_img = (uint32_t)((p.G2 * p.N3) * (p.G1 * p.N1) * 2);
  size_t o = 0;
  p.sm_w1 = (uint32_t)o; o = al(o + (size_t)parts * p.w1_groups * p.w1_img, 1024);
  static const bool resident = getenv("DELIMIT_T_RESIDENT") != nullptr;   // measurement knob
  const size_t tbufs = 2 * (size_t)parts * p.N3 * (p.G1 * p.N1) * 2;      // two shells' images
  p.tstream = (!kout && !resident && tbufs < (size_t)parts * p.w2_img) ? 1 : 0;
  p.sm_w2 = (uint32_t)o; o = al(o + (p.tstream ? tbufs : (size_t)parts * p.w2_img), 1024);
  p.sm_bias = (uint32_t)o; o = al(o + (size_t)p.G2 * p.N3 * 4, 128);
  p.sm_tring = 0;
  if (p.target && !kout && kOB2h == 1 && !getenv("DELIMIT_NO_TRING")) {   // fused MSE target rings
    p.sm_tring = (uint32_t)o;
    o = al(o + (size_t)kOUT3 * 2 * 16 * 32 * 4, 128);
  }
  p.sm_ring = (uint32_t)o;
  for (int ns : {12, 8, 4}) {
    p.ns = ns;
    size_t q = al(p.sm_ring + (size_t)ns * kStageBytes, 16);
    p.sm_bar = (uint32_t)q;
    q = al(q + sizeof(Bars2h), 16);
    p.smem_bytes = (uint32_t)q;
    if (q <= kSmemMax) return true;
  }
  return false;
}

template <int NS, bool KOUT, bool DIAG = false, bool GONLY = false>
int launch_chain2h(const Chain3& p, int grid, cudaStream_t st) {
  DL_CUDA(cudaFuncSetAttribute(chain2h_tc<NS, KOUT, DIAG, GONLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)p.smem_bytes));
  chain2h_tc<NS, KOUT, DIAG, GONLY><<<grid, kThreads2h, p.smem_bytes, st>>>(p);
  return after_launch(KOUT ? "chain2h_tc(k-outer)" : "chain2h_tc");
}

bool use_kout() {   // DELIMIT_CHAIN2H_KOUT=1 selects the K-outer variant (measurement knob)
  static const bool v = getenv("DELIMIT_CHAIN2H_KOUT") != nullptr;
  return v;
}

bool use_v3() {
  static const bool v = getenv("DELIMIT_CHAIN_V2") == nullptr;
  return v;
}

bool plan_gram(GramP& p) {
  if (p.GR > 144 || p.GC > 144 || p.GR % 16 || p.GC % 16) return false;
  const int grow = p.GR < 128 ? 128 : p.GR;
  p.colGA = 0;
  p.colGB = (uint32_t)p.GC;
  p.colGC = (uint32_t)p.GC + 16;
  p.cpart = (uint32_t)p.GC * 128u;   // rows x one 128-byte K atom (64 bf16 voxels)
  p.gpart = (uint32_t)grow * 128u;
  // block C reads c rows up to 191 of a term plane: they land in the next plane of the same stage
  p.stage_bytes = (uint32_t)al(2 * (size_t)p.cpart + 2 * (size_t)p.gpart, 1024);
  p.sm_ring = 0;
  for (int ns : {4, 3, 2}) {
    p.ns = ns;
    size_t q = al((size_t)ns * p.stage_bytes, 16);
    p.sm_bar = (uint32_t)q;
    q = al(q + sizeof(BarsG), 16);
    p.smem_bytes = (uint32_t)q;
    if (q <= kSmemMax) return true;
  }
  return false;
}

template <int PARTS>
int run_chain3(const Chain3& p, int grid, cudaStream_t st) {
  auto k = p.ns == 8 ? chain3_tc<PARTS, 8> : p.ns == 4 ? chain3_tc<PARTS, 4> : chain3_tc<PARTS, 2>;
  DL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes));
  k<<<grid, kThreads, p.smem_bytes, st>>>(p);
  return after_launch("chain3_tc");
}

template <int PARTS, int NS, bool H>
int launch_chain3v(const Chain3& p, int grid, cudaStream_t st) {
  DL_CUDA(cudaFuncSetAttribute(chain3v_tc<PARTS, NS, H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)p.smem_bytes));
  chain3v_tc<PARTS, NS, H><<<grid, kThreads3, p.smem_bytes, st>>>(p);
  return after_launch(H ? "chain3v_tc(fp16)" : "chain3v_tc");
}

template <int PARTS, bool H = false>
int run_chain3v(const Chain3& p, int grid, cudaStream_t st) {
  switch (p.ns) {
    case 2: return launch_chain3v<PARTS, 2, H>(p, grid, st);
    case 4: return launch_chain3v<PARTS, 4, H>(p, grid, st);
    case 6: return launch_chain3v<PARTS, 6, H>(p, grid, st);
    case 8: return launch_chain3v<PARTS, 8, H>(p, grid, st);
    case 10: return launch_chain3v<PARTS, 10, H>(p, grid, st);
    default: return launch_chain3v<PARTS, 12, H>(p, grid, st);
  }
}

// plan + launch one chain3 direction on the best kernel that fits.  With a delayed-scaling state (and the
// default precision mode): the fp16 pass, then the bf16 pass that checks it and recomputes only if needed.
// p's images are the bf16 ones; hw1/hw2/hw3 the fp16 images.
int run_chain(Chain3 p, const Dims& d, int grid, cudaStream_t st, const char* what, uint32_t* rstate = nullptr,
              const uint16_t* hw1 = nullptr, const uint16_t* hw2 = nullptr, const uint16_t* hw3 = nullptr,
              const uint16_t* hT = nullptr, const float* bias3 = nullptr) {
  Chain3 v = p;
  if (use_v3() && plan_chain3v(v, d.parts)) {
    Chain3 h = p, h2 = p;
    const bool kout = use_kout();
    if (rstate && d.parts == 3 && hw1 && hT && use_2h() && plan_chain2h(h2, kout)) {
      h2.w1 = hw1;
      h2.w2 = hT;
      h2.bias2 = bias3;
      h2.rstate = rstate;
      h2.redo = 0;
      h2.kt = ktrace();
      h2.kt_slot = what[6] == 'f' ? 0 : 1;   // "chain_fwd" / "chain_bwd"
      if (kout) DL_TRY((h2.ns == 8 ? launch_chain2h<8, true>(h2, grid, st) : launch_chain2h<4, true>(h2, grid, st)));
      else if (h2.ns == 12 && h2.t_diag) DL_TRY((launch_chain2h<12, false, true>(h2, grid, st)));
      else if (h2.ns == 12 && !h2.out && h2.mid && !h2.target)   // g-only adjoint
        DL_TRY((launch_chain2h<12, false, false, true>(h2, grid, st)));
      else if (h2.ns == 12) DL_TRY((launch_chain2h<12, false>(h2, grid, st)));   // (a dense T is exact for t_diag too)
      else DL_TRY((h2.ns == 8 ? launch_chain2h<8, false>(h2, grid, st) : launch_chain2h<4, false>(h2, grid, st)));
      v.rstate = rstate;
      v.redo = 1;
      v.prof = nullptr;
      return d.parts == 3 ? run_chain3v<3>(v, grid, st) : run_chain3v<2>(v, grid, st);
    }
    if (rstate && d.parts == 3 && hw1 && plan_chain3v(h, 2)) {
      h.w1 = hw1;
      h.w2 = hw2;
      h.w3 = hw3;
      h.rstate = rstate;
      h.redo = 0;
      DL_TRY((run_chain3v<2, true>(h, grid, st)));
      v.rstate = rstate;
      v.redo = 1;
      v.prof = nullptr;
    }
    return d.parts == 3 ? run_chain3v<3>(v, grid, st) : run_chain3v<2>(v, grid, st);
  }
  if (!plan_chain3(p, d.parts)) return dl::fail(DL_EINVAL, "%s: channel counts exceed the fused kernel's plan", what);
  return d.parts == 3 ? run_chain3<3>(p, grid, st) : run_chain3<2>(p, grid, st);
}

template <int NS>
int launch_gram(const GramP& p, int grid, cudaStream_t st) {
  DL_CUDA(cudaFuncSetAttribute(gram_tc<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes));
  gram_tc<NS><<<grid, kGThreads, p.smem_bytes, st>>>(p);
  return after_launch("gram_tc");
}

int run_gram(const GramP& p, int grid, cudaStream_t st) {
  switch (p.ns) {
    case 2: return launch_gram<2>(p, grid, st);
    case 3: return launch_gram<3>(p, grid, st);
    default: return launch_gram<4>(p, grid, st);
  }
}

PackJob pack_job_of(const float* W, uint16_t* out, uint16_t* out_h, int ng, int nrb, int rb, int rbp, int ncb, int cb,
                    int cbp, int parts) {
  return PackJob{W, out, out_h, ng, nrb, rb, rbp, ncb, cb, cbp, parts};
}

int pack_jobs(const PackJobs& jobs, int njobs, cudaStream_t st) {
  if (njobs == 0) return DL_OK;
  int64_t n = 0;
  for (int i = 0; i < njobs; ++i) {
    const PackJob& j = jobs.j[i];
    const int64_t ni = (int64_t)j.ng * j.nrb * j.rbp * j.ncb * j.cbp;
    n = ni > n ? ni : n;
  }
  const int blocks = (int)((n + 255) / 256 < 2048 ? (n + 255) / 256 : 2048);
  pack_k<<<dim3(blocks, njobs), 256, 0, st>>>(jobs);
  return after_launch("pack_operand");
}

int pack(const float* W, uint16_t* out, uint16_t* out_h, int ng, int nrb, int rb, int rbp, int ncb, int cb, int cbp,
         int parts, cudaStream_t st) {
  PackJobs jobs{};
  jobs.j[0] = pack_job_of(W, out, out_h, ng, nrb, rb, rbp, ncb, cb, cbp, parts);
  return pack_jobs(jobs, 1, st);
}

// bf16 images (d.parts terms) and, for the fp16 pass, the fp16 two-term images, in one launch
int pack_all(const Dims& d, const WsLayout& w, uint8_t* ws, const float* M, const float* L, const float* Bt, bool h,
             cudaStream_t st) {
  auto img = [&](size_t off, size_t off_h) {
    return std::make_pair(reinterpret_cast<uint16_t*>(ws + off), h ? reinterpret_cast<uint16_t*>(ws + off_h) : nullptr);
  };
  PackJobs jobs{};
  int nj = 0;
  if (M) {
    auto [o, oh] = img(w.imgM, w.imgMh);
    jobs.j[nj++] = pack_job_of(M, o, oh, d.mg, 1, d.r_in, d.RPi, 1, d.n, d.NPi, d.parts);
  }
  if (L) {
    auto [o, oh] = img(w.imgL, w.imgLh);
    jobs.j[nj++] = pack_job_of(L, o, oh, 1, d.s_out, d.r_out, d.RPo, d.s_in, d.r_in, d.RPi, d.parts);
  }
  if (Bt) {
    auto [o, oh] = img(w.imgB, w.imgBh);
    jobs.j[nj++] = pack_job_of(Bt, o, oh, 1, 1, d.n_out, d.NPo, 1, d.r_out, d.RPo, d.parts);
  }
  return pack_jobs(jobs, nj, st);
}

// chain2h operands: the folded operator T (and, forward, its bias) in fp32, then its fp16 two-term image
int fold_t(const Dims& d, const WsLayout& w, uint8_t* ws, const float* M, const float* L, const float* Bt,
           const float* bvec, bool adjoint, cudaStream_t st) {
  float* T = reinterpret_cast<float*>(ws + w.Tf);
  float* b3 = reinterpret_cast<float*>(ws + w.b3);
  const int64_t n = adjoint ? (int64_t)d.s_in * d.n * d.s_out * d.r_out : (int64_t)d.s_out * d.n_out * d.s_in * d.r_in;
  const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  fold_t_k<<<blocks, 256, 0, st>>>(L, Bt, M, bvec, T, b3, adjoint ? 1 : 0, d.s_in, d.s_out, d.r_in, d.r_out, d.n,
                                   d.n_out, d.mg);
  DL_TRY(after_launch("fold_t_k"));
  uint16_t* img = reinterpret_cast<uint16_t*>(ws + w.imgTh);
  if (!adjoint) return pack(T, nullptr, img, 1, d.s_out, d.n_out, d.NPo, d.s_in, d.r_in, d.RPi, 0, st);
  return pack(T, nullptr, img, 1, d.s_in, d.n, d.NPi, d.s_out, d.r_out, d.RPo, 0, st);
}

Chain3 chain3_params(const Dims& d, const WsLayout& w, const uint8_t* ws, bool adjoint) {
  Chain3 p{};
  p.redo = 0;
  p.rstate = nullptr;
  p.nbatch = d.nbatch;
  p.nvox = d.nvox;
  p.tiles_per_b = (d.nvox + kTileV - 1) / kTileV;
  p.adjoint = adjoint ? 1 : 0;
  p.w2 = reinterpret_cast<const uint16_t*>(ws + w.imgL);
  if (!adjoint) {
    p.G1 = d.s_in; p.C1 = d.n; p.K1 = d.NPi; p.N1 = d.RPi;
    p.G2 = d.s_out; p.C2 = d.r_out; p.N2 = d.RPo;
    p.C3 = d.n_out; p.N3 = d.NPo;
    p.w1 = reinterpret_cast<const uint16_t*>(ws + w.imgM); p.w1_groups = d.mg;
    p.w3 = reinterpret_cast<const uint16_t*>(ws + w.imgB); p.w3_groups = 1;
    p.in_bs = (int64_t)d.s_in * d.n * d.nvox;
    p.out_bs = (int64_t)d.s_out * d.n_out * d.nvox;
  } else {
    p.G1 = d.s_out; p.C1 = d.n_out; p.K1 = d.NPo; p.N1 = d.RPo;
    p.G2 = d.s_in; p.C2 = d.r_in; p.N2 = d.RPi;
    p.C3 = d.n; p.N3 = d.NPi;
    p.w1 = reinterpret_cast<const uint16_t*>(ws + w.imgB); p.w1_groups = 1;
    p.w3 = reinterpret_cast<const uint16_t*>(ws + w.imgM); p.w3_groups = d.mg;
    p.in_bs = (int64_t)d.s_out * d.n_out * d.nvox;
    p.out_bs = (int64_t)d.s_in * d.n * d.nvox;
  }
  return p;
}

int64_t mid_pitch(int64_t nvox) { return (nvox + kGV - 1) / kGV * kGV; }

GramP gram_params(const Dims& d, const WsLayout& w, uint8_t* ws) {
  GramP p{};
  p.nbatch = d.nbatch;
  p.tiles_per_b = mid_pitch(d.nvox) / kGV;
  p.GR = d.s_out * d.RPo;
  p.GC = d.s_in * d.RPi;
  p.partials = reinterpret_cast<float*>(ws + w.parts);
  return p;
}

bool chain_fits(const Dims& d) {
  if (d.RPi == d.r_in) return false;   // the Gram's bias column needs a zero-weight padding row in c
  Chain3 f = chain3_params(d, ws_layout(d, 1), nullptr, false);
  Chain3 a = chain3_params(d, ws_layout(d, 1), nullptr, true);
  GramP g = gram_params(d, ws_layout(d, 1), nullptr);
  auto fits = [&](Chain3 c) {
    Chain3 v = c;
    return (use_v3() && plan_chain3v(v, d.parts)) || plan_chain3(c, d.parts);
  };
  return fits(f) && fits(a) && plan_gram(g);
}

// Channel-pair view of a (nbatch, rows, nvox) fp32 tensor for TMA: element (u, j, b) is channel 2j + u / nvox,
// voxel u % nvox -- rows 2j and 2j+1 are contiguous, so the row stride 8*nvox bytes is 16-byte aligned for
// any even nvox.  Box = 132 voxels x 8 channel pairs.  False (use the cp.async path) if not expressible.
CUtensorMapL2promotion l2_promotion() {   // tuning knob DELIMIT_L2_PROMO = 0 / 64 / 128 / 256 (default)
  static const CUtensorMapL2promotion v = [] {
    const char* e = getenv("DELIMIT_L2_PROMO");
    const int b = e ? atoi(e) : 256;
    return b == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : b == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : b == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return v;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      fn = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return encode;
}

bool pair_map(CUtensorMap* m, const float* base, int64_t nbatch, int64_t rows, int64_t group_rows, int64_t nvox,
              int boxv = kBoxV) {
  auto encode = tensor_map_encoder();
  if (!encode || !base || nvox % 2 || rows % 2 || group_rows % 2 || ((uintptr_t)base & 15) ||
      2 * nvox + kTileV >= ((int64_t)1 << 31) || nbatch >= ((int64_t)1 << 31) || rows / 2 > ((int64_t)1 << 31))
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * nvox), (cuuint64_t)(rows / 2), (cuuint64_t)nbatch};
  const cuuint64_t strides[2] = {(cuuint64_t)(8 * nvox), (cuuint64_t)(4 * rows * nvox)};
  const cuuint32_t box[3] = {(cuuint32_t)boxv, 8u, 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tiled mid buffer [b][64-voxel tile][term][row][64 voxels] bf16 as a 4-D map (64, rows, 2, nbatch * tiles):
// one box = one term plane of one tile, a contiguous rows x 128-byte block; SWIZZLE_128B makes TMA write
// exactly the K-major operand layout desc_sw128_k reads.
bool mid_map(CUtensorMap* m, const void* base, int64_t nbatch, int rows, int64_t pitch) {
  auto encode = tensor_map_encoder();
  const int64_t nt = nbatch * (pitch / kGV);
  if (!encode || !base || ((uintptr_t)base & 15) || rows > 256 || nt >= ((int64_t)1 << 31)) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)kGV, (cuuint64_t)rows, 2, (cuuint64_t)nt};
  const cuuint64_t strides[3] = {(cuuint64_t)(2 * kGV), (cuuint64_t)(2 * kGV * rows), (cuuint64_t)(4 * kGV * rows)};
  const cuuint32_t box[4] = {(cuuint32_t)kGV, (cuuint32_t)rows, 1u, 1u};
  const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_disabled() {
  static const bool v = getenv("DELIMIT_NO_TMA") != nullptr;
  return v;
}

int grid_for(int64_t ntiles, int sm) { return (int)(ntiles < sm ? (ntiles > 0 ? ntiles : 1) : sm); }


}  // namespace
}  // namespace tc
}  // namespace dl

extern "C" {

// Debug hook (not part of the documented ABI): record chain3 phase timestamps of CTA 0 into
// `buf` (device, >= 8*4*32 int64) on subsequent forward launches; NULL disables.
void dl_debug_chain_prof(void* buf) { dl::tc::g_prof = reinterpret_cast<long long*>(buf); }

int dl_chain_supported(int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                       int m_per_shell) {
  using namespace dl::tc;
  return chain_fits(make_dims(1, s_in, s_out, n, r_in, r_out, n_out, 1, m_per_shell)) ? 1 : 0;
}

int dl_chain_split_terms(void) { return dl::tc::split_terms(); }

size_t dl_chain_state_bytes(void) { return dl::tc::kStateWords * sizeof(uint32_t); }

size_t dl_chain_workspace_bytes(int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out,
                                int64_t n_out, int64_t nvox) {
  using namespace dl::tc;
  return ws_layout(make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, 1), kMaxParts).total;
}

size_t dl_chain_mid_bytes(int64_t nbatch, int64_t shells, int64_t r, int64_t nvox) {
  using namespace dl::tc;
  return (size_t)nbatch * 2 * (size_t)(shells * r16(r)) * (size_t)mid_pitch(nvox) * 2;
}

}  // extern "C"

namespace dl {
namespace tc {
namespace {
// forward of dl_chain_fwd_f32 / dl_chain_fwd_mse_f32 (target != null: out = out_scale (y - target), squared
// residuals summed into loss[0] by the fp16 / plain pass and into loss[1] by a redo pass)
int chain_fwd(const float* x, float* y, void* c_mid, const float* M, int m_per_shell, const float* L,
              const float* bvec, const float* Bt, void* workspace, void* state, int64_t nbatch, int64_t s_in,
              int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream,
              const float* target, float out_scale, double* loss, int diag = 0) {
  int sm = 0;
  DL_TRY(dl::device_check(&sm));
  DL_REQUIRE(x && y && M && L && Bt && workspace, "chain_fwd: null pointer");
  DL_REQUIRE(nbatch >= 0 && nvox >= 0 && s_in >= 1 && s_out >= 1 && n >= 1 && r_in >= 1 && r_out >= 1 && n_out >= 1,
             "chain_fwd: bad sizes");
  Dims d = make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, m_per_shell);
  WsLayout w = ws_layout(d, kMaxParts);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  Chain3 p = chain3_params(d, w, ws, false);
  DL_REQUIRE(chain_fits(d), "chain_fwd: channel counts exceed the fused kernel's TMEM/smem plan");
  if (target) {
    Chain3 v = p;
    DL_REQUIRE(use_v3() && plan_chain3v(v, d.parts), "chain_fwd_mse: these channel counts need the fallback kernel, "
               "which has no fused loss (dl_chain_mse_supported)");
  }
  if (nbatch == 0 || nvox == 0) return DL_OK;
  cudaStream_t st = dl::as_stream(stream);
  const bool h = state && fp16_pass();
  DL_TRY(pack_all(d, w, ws, M, L, Bt, h, st));
  p.in = x;
  p.out = y;
  p.mid = reinterpret_cast<uint16_t*>(c_mid);
  p.mid_pitch = mid_pitch(nvox);
  p.mid_bs = 2 * (int64_t)d.s_in * d.RPi * p.mid_pitch;
  p.mid_ones = d.r_in;   // shell 0's first padding row
  p.bias2 = bvec;
  p.prof = g_prof;
  p.target = target;
  p.out_scale = out_scale;
  p.loss = loss;
  p.tma = !tma_disabled() && pair_map(&p.tm[0], x, nbatch, s_in * n, n, nvox);
  p.t_diag = diag;
  const int grid = grid_for(nbatch * p.tiles_per_b, sm);
  const bool fold = h && use_2h();
  if (fold) DL_TRY(fold_t(d, w, ws, M, L, Bt, bvec, false, st));
  return run_chain(p, d, grid, st, "chain_fwd", h ? reinterpret_cast<uint32_t*>(state) : nullptr,
                   reinterpret_cast<const uint16_t*>(ws + w.imgMh), reinterpret_cast<const uint16_t*>(ws + w.imgLh),
                   reinterpret_cast<const uint16_t*>(ws + w.imgBh),
                   fold ? reinterpret_cast<const uint16_t*>(ws + w.imgTh) : nullptr,
                   reinterpret_cast<const float*>(ws + w.b3));
}

// the pass whose results stand decides which accumulator holds the loss
__global__ void mse_finalize_k(const uint32_t* __restrict__ state, double* __restrict__ loss, double inv_n) {
  const int redo = state ? (int)((volatile const uint32_t*)state)[kStLastRedo] : 0;
  loss[2] = loss[redo ? 1 : 0] * inv_n;
}
}  // namespace
}  // namespace tc
}  // namespace dl

extern "C" {

int dl_chain_fwd_f32(const float* x, float* y, void* c_mid, const float* M, int m_per_shell, const float* L,
                     const float* bvec, const float* Bt, void* workspace, void* state, int64_t nbatch, int64_t s_in,
                     int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream) {
  dl::begin_call();
  return dl::tc::chain_fwd(x, y, c_mid, M, m_per_shell, L, bvec, Bt, workspace, state, nbatch, s_in, s_out, n, r_in,
                           r_out, n_out, nvox, stream, nullptr, 0.f, nullptr);
}

// The fused chain read straight from a raw acquisition (b0 normalisation in the IN role, in_role_raw): the
// 3-term bf16 pass, forward only; y is (s_out * n_out, nvox) in the acquisition's stored voxel order.
int dl_chain_fwd_raw_f32(const void* raw, int raw_dtype, int64_t vstride, const int* sel, const float* vox_a,
                         const float* vox_b, float* y, const float* M, int m_per_shell, const float* L,
                         const float* bvec, const float* Bt, void* workspace, void* state, int64_t s_in,
                         int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox,
                         void* stream) {
  using namespace dl::tc;
  dl::begin_call();
  int sm = 0;
  DL_TRY(dl::device_check(&sm));
  DL_REQUIRE(raw && sel && vox_a && vox_b && y && M && L && Bt && workspace, "chain_fwd_raw: null pointer");
  DL_REQUIRE(raw_dtype == 4 || raw_dtype == 16, "chain_fwd_raw: raw datatype %d (int16 = 4, float32 = 16 only)",
             raw_dtype);
  const int esz = raw_dtype == 4 ? 2 : 4;
  DL_REQUIRE(vstride % 2 == 0 && vstride >= nvox && (uintptr_t)raw % (2 * esz) == 0,
             "chain_fwd_raw: volumes must start on %d-byte boundaries (even stride, aligned base)", 2 * esz);
  DL_REQUIRE(nvox >= 0 && s_in >= 1 && s_out >= 1 && n >= 1 && r_in >= 1 && r_out >= 1 && n_out >= 1,
             "chain_fwd_raw: bad sizes");
  Dims d = make_dims(1, s_in, s_out, n, r_in, r_out, n_out, nvox, m_per_shell);
  DL_REQUIRE(chain_fits(d), "chain_fwd_raw: channel counts exceed the fused kernel's TMEM/smem plan");
  if (nvox == 0) return DL_OK;
  WsLayout w = ws_layout(d, kMaxParts);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  cudaStream_t st = dl::as_stream(stream);
  const bool h = state && fp16_pass();
  DL_TRY(pack_all(d, w, ws, M, L, Bt, h, st));
  Chain3 p = chain3_params(d, w, ws, false);
  p.in = nullptr;
  p.out = y;
  p.mid = nullptr;
  p.mid_pitch = mid_pitch(nvox);
  p.mid_ones = -1;
  p.bias2 = bvec;
  p.tma = 0;
  p.raw = raw;
  p.raw_type = raw_dtype;
  p.raw_vstride = vstride;
  p.raw_sel = sel;
  p.vox_a = vox_a;
  p.vox_b = vox_b;
  Chain3 v = p;
  DL_REQUIRE(use_v3() && plan_chain3v(v, d.parts), "chain_fwd_raw: needs the chain3v plan");
  // with a state: the fp16 pass (chain2h with SH2Signal folded into T, else chain3v; delayed scaling) and the bf16
  // check pass, all reading the raw volumes
  const bool fold = h && use_2h();
  if (fold) DL_TRY(fold_t(d, w, ws, M, L, Bt, bvec, false, st));
  return run_chain(p, d, grid_for(p.tiles_per_b, sm), st, "chain_fwd", h ? reinterpret_cast<uint32_t*>(state) : nullptr,
                   reinterpret_cast<const uint16_t*>(ws + w.imgMh), reinterpret_cast<const uint16_t*>(ws + w.imgLh),
                   reinterpret_cast<const uint16_t*>(ws + w.imgBh),
                   fold ? reinterpret_cast<const uint16_t*>(ws + w.imgTh) : nullptr,
                   reinterpret_cast<const float*>(ws + w.b3));
}

int dl_chain_fwd_mse_f32(const float* x, const float* target, float* dy, void* c_mid, const float* M, int m_per_shell,
                         const float* L, const float* bvec, const float* Bt, void* workspace, void* state,
                         double* loss, int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in,
                         int64_t r_out, int64_t n_out, int64_t nvox, void* stream) {
  dl::begin_call();
  DL_REQUIRE(target && dy && loss, "chain_fwd_mse: null pointer");
  const double count = (double)nbatch * (double)s_out * (double)n_out * (double)nvox;
  cudaStream_t st = dl::as_stream(stream);
  DL_CUDA(cudaMemsetAsync(loss, 0, 2 * sizeof(double), st));
  DL_TRY(dl::tc::chain_fwd(x, dy, c_mid, M, m_per_shell, L, bvec, Bt, workspace, state, nbatch, s_in, s_out, n, r_in,
                           r_out, n_out, nvox, stream, target, count > 0 ? (float)(2.0 / count) : 0.f, loss));
  dl::tc::mse_finalize_k<<<1, 1, 0, st>>>(reinterpret_cast<const uint32_t*>(state && dl::tc::fp16_pass() ? state : nullptr),
                                         loss, count > 0 ? 1.0 / count : 0.0);
  return dl::after_launch("mse_finalize_k");
}

int dl_chain_mse_supported(int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                           int m_per_shell) {
  using namespace dl::tc;
  const Dims d = make_dims(1, s_in, s_out, n, r_in, r_out, n_out, 1, m_per_shell);
  if (!chain_fits(d) || !use_v3()) return 0;
  Chain3 v = chain3_params(d, ws_layout(d, 1), nullptr, false);
  return plan_chain3v(v, d.parts) ? 1 : 0;
}

}  // extern "C"

namespace dl {
namespace tc {
namespace {
// The backward of dl_chain_bwd_f32 / dl_chain_bwd_gram_f64: gram_out (optional) receives the float64 Gram
// instead of the finalized dW / db.
int chain_bwd(const void* c_mid, const float* dy, float* dx, float* dW, float* db, double* gram_out, void* g_mid,
              const float* M, int m_per_shell, const float* L, const float* Bt, const float* P, const float* beta,
              void* workspace, void* state, int64_t nbatch, int64_t s_in, int64_t s_out, int64_t K, int64_t n,
              int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream, int diag = 0) {
  int sm = 0;
  DL_TRY(dl::device_check(&sm));
  DL_REQUIRE(dy && M && L && Bt && workspace, "chain_bwd: null pointer");
  DL_REQUIRE(dx || dW || db || gram_out, "chain_bwd: nothing requested (dx, dW, db and the Gram are all null)");
  DL_REQUIRE(!(dW || db) || (c_mid && g_mid && P && beta), "chain_bwd: the weight gradient needs c_mid, g_mid, P, beta");
  DL_REQUIRE(!gram_out || (c_mid && g_mid), "chain_bwd: the Gram needs c_mid and g_mid");
  Dims d = make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, m_per_shell);
  DL_REQUIRE(chain_fits(d), "chain_bwd: channel counts exceed the fused kernel's TMEM/smem plan");
  WsLayout w = ws_layout(d, kMaxParts);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  cudaStream_t st = dl::as_stream(stream);
  const int64_t ntiles = nbatch * ((nvox + kTileV - 1) / kTileV);
  const bool wgrad = dW || db || gram_out;
  const bool h = state && fp16_pass();
  DL_TRY(pack_all(d, w, ws, M, L, Bt, h, st));
  if (ntiles > 0) {
    // adjoint chain dy -> dx; its stage-1 accumulator g = B'^T dy goes to g_mid for the Gram
    Chain3 p = chain3_params(d, w, ws, true);
    p.in = dy;
    p.out = dx;
    p.mid = wgrad ? reinterpret_cast<uint16_t*>(g_mid) : nullptr;
    p.mid_pitch = mid_pitch(nvox);
    p.mid_bs = 2 * (int64_t)d.s_out * d.RPo * p.mid_pitch;
    p.mid_ones = -1;
    p.bias2 = nullptr;
    p.tma = !tma_disabled() && pair_map(&p.tm[0], dy, nbatch, s_out * n_out, n_out, nvox);
    p.t_diag = diag;
    // adjoint: stage 1 uses B' (w1 = imgB), stage 3 uses M (w3 = imgM)
    const bool fold = h && use_2h();
    if (fold) DL_TRY(fold_t(d, w, ws, M, L, Bt, nullptr, true, st));
    DL_TRY(run_chain(p, d, grid_for(ntiles, sm), st, "chain_bwd", h ? reinterpret_cast<uint32_t*>(state) : nullptr,
                     reinterpret_cast<const uint16_t*>(ws + w.imgBh), reinterpret_cast<const uint16_t*>(ws + w.imgLh),
                     reinterpret_cast<const uint16_t*>(ws + w.imgMh),
                     fold ? reinterpret_cast<const uint16_t*>(ws + w.imgTh) : nullptr, nullptr));
  }
  if (wgrad) {
    GramP g = gram_params(d, w, ws);
    DL_REQUIRE(plan_gram(g), "chain_bwd: channel counts exceed the fused Gram plan");
    const int GR = g.GR, GC = g.GC;
    const int64_t gtiles = nbatch * g.tiles_per_b;
    int nparts = 0;
    if (gtiles > 0) {
      DL_REQUIRE(mid_map(&g.tm[0], g_mid, nbatch, GR, mid_pitch(nvox)) &&
                     mid_map(&g.tm[1], c_mid, nbatch, GC, mid_pitch(nvox)),
                 "chain_bwd: c_mid / g_mid must be 16-byte aligned buffers of dl_chain_mid_bytes()");
      const int cap = sm * gram_waves();
      nparts = grid_for(gtiles, cap < kMaxParts ? cap : kMaxParts);
      g.kt = ktrace();
      DL_TRY(run_gram(g, nparts, st));
    }
    double* G = gram_out ? gram_out : reinterpret_cast<double*>(ws + w.G);
    if (nparts == 0) {
      DL_CUDA(cudaMemsetAsync(G, 0, (size_t)GR * GC * 8, st));
    } else {
      gram_reduce_k<<<(GR * GC + 31) / 32, dim3(32, 8), 0, st>>>(reinterpret_cast<float*>(ws + w.parts), G, nparts, GR * GC);
      DL_TRY(dl::after_launch("gram_reduce"));
    }
    if (!gram_out) {
    gram_finalize_k<<<(unsigned)(s_out * s_in * K + s_out), 256, 0, st>>>(G, beta, (int)r_in, P, dW, db, (int)s_out,
                                                                            (int)s_in, (int)K, (int)r_out, (int)r_in,
                                                                            d.RPo, d.RPi);
      DL_TRY(dl::after_launch("gram_finalize"));
    }
  }
  return DL_OK;
}
}  // namespace
}  // namespace tc
}  // namespace dl

extern "C" {

int dl_chain_bwd_f32(const void* c_mid, const float* dy, float* dx, float* dW, float* db, void* g_mid,
                     const float* M, int m_per_shell, const float* L, const float* Bt, const float* P,
                     const float* beta, void* workspace, void* state, int64_t nbatch, int64_t s_in, int64_t s_out,
                     int64_t K, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream) {
  dl::begin_call();
  return dl::tc::chain_bwd(c_mid, dy, dx, dW, db, nullptr, g_mid, M, m_per_shell, L, Bt, P, beta, workspace, state,
                           nbatch, s_in, s_out, K, n, r_in, r_out, n_out, nvox, stream);
}

int dl_chain_bwd_gram_f64(const void* c_mid, const float* dy, float* dx, double* gram, void* g_mid, const float* M,
                          int m_per_shell, const float* L, const float* Bt, void* workspace, void* state,
                          int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out,
                          int64_t n_out, int64_t nvox, void* stream) {
  dl::begin_call();
  if (!gram) return dl::fail(DL_EINVAL, "chain_bwd_gram: null Gram output");
  return dl::tc::chain_bwd(c_mid, dy, dx, nullptr, nullptr, gram, g_mid, M, m_per_shell, L, Bt, nullptr, nullptr,
                           workspace, state, nbatch, s_in, s_out, 1, n, r_in, r_out, n_out, nvox, stream);
}

int dl_chain_gram_dims(int64_t s_in, int64_t s_out, int64_t r_in, int64_t r_out, int64_t* rows, int64_t* cols) {
  if (!rows || !cols) return dl::fail(DL_EINVAL, "chain_gram_dims: null output");
  *rows = s_out * ((r_out + 15) / 16 * 16);
  *cols = s_in * ((r_in + 15) / 16 * 16);
  return DL_OK;
}

}  // extern "C"

namespace dl {
namespace tc {
namespace {
__global__ void eye_k(float* L, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
    L[e] = (e / n == e % n) ? 1.f : 0.f;
}
// the identity standing in for the LSC operator of the round trip, at the end of the caller's workspace
float* round_trip_eye(void* workspace, int64_t s, int64_t r, int64_t n, int64_t n_out, int64_t nvox, cudaStream_t st,
                      int* status) {
  const size_t off = al(ws_layout(make_dims(1, s, s, n, r, r, n_out, nvox, 1), kMaxParts).total, 256);
  float* eye = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + off);
  const int m = (int)(s * r);
  eye_k<<<(m * m + 255) / 256 < 256 ? (m * m + 255) / 256 : 256, 256, 0, st>>>(eye, m);
  *status = dl::after_launch("round_trip_eye");
  return eye;
}
}  // namespace
}  // namespace tc
}  // namespace dl

extern "C" {

size_t dl_round_trip_workspace_bytes(int64_t nbatch, int64_t shells, int64_t n, int64_t r, int64_t n_out,
                                     int64_t nvox) {
  using namespace dl::tc;
  return al(ws_layout(make_dims(nbatch, shells, shells, n, r, r, n_out, nvox, 1), kMaxParts).total, 256) +
         (size_t)(shells * r) * (size_t)(shells * r) * 4;
}

int dl_round_trip_fwd_f32(const float* x, float* y, const float* M, int m_per_shell, const float* Bt, void* workspace,
                          void* state, int64_t nbatch, int64_t shells, int64_t n, int64_t r, int64_t n_out,
                          int64_t nvox, void* stream) {
  dl::begin_call();
  DL_REQUIRE(workspace, "round_trip_fwd: null workspace");
  int st = DL_OK;
  const float* eye = dl::tc::round_trip_eye(workspace, shells, r, n, n_out, nvox, dl::as_stream(stream), &st);
  DL_TRY(st);
  return dl::tc::chain_fwd(x, y, nullptr, M, m_per_shell, eye, nullptr, Bt, workspace, state, nbatch, shells, shells,
                           n, r, r, n_out, nvox, stream, nullptr, 0.f, nullptr, 1);
}

int dl_round_trip_bwd_f32(const float* dy, float* dx, const float* M, int m_per_shell, const float* Bt,
                          void* workspace, void* state, int64_t nbatch, int64_t shells, int64_t n, int64_t r,
                          int64_t n_out, int64_t nvox, void* stream) {
  dl::begin_call();
  DL_REQUIRE(workspace, "round_trip_bwd: null workspace");
  int st = DL_OK;
  const float* eye = dl::tc::round_trip_eye(workspace, shells, r, n, n_out, nvox, dl::as_stream(stream), &st);
  DL_TRY(st);
  return dl::tc::chain_bwd(nullptr, dy, dx, nullptr, nullptr, nullptr, nullptr, M, m_per_shell, eye, Bt, nullptr,
                           nullptr, workspace, state, nbatch, shells, shells, 1, n, r, r, n_out, nvox, stream, 1);
}

}  // extern "C"
