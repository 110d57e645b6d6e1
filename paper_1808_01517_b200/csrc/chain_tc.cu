// Fused tensor-core (tcgen05) kernels for the Signal2SH -> LSC -> SH2Signal chain.
//
// Reference path (/root/reference/pkg/src/sphdwi/): fitting.signal_to_sh (fitting.py:206-236) ->
// lsc.lsc_forward (lsc.py:158-199, folded as c_out = L c + bias*beta) ->
// fitting.sh_to_signal (fitting.py:239-250); the backward is the adjoint (SPEC.md:12 leaves it out).
//
// Design (one persistent CTA per SM, voxel tiles of 128 = the MMA M dimension):
//  * thread t of a TMEM lane quadrant owns voxel t of the tile: it loads its voxel's channels
//    with coalesced 4-byte loads (a warp covers 32 consecutive voxels of one channel row),
//    splits every fp32 value into PARTS bf16 terms and writes them into TMEM as the A operand;
//  * all weights (M, folded LSC operator L, B') are staged ONCE per CTA in shared memory as
//    PARTS bf16 terms (core-matrix blocked images; the same image serves the forward (K-major)
//    and the adjoint (MN-major) product);
//  * one elected thread issues tcgen05.mma kind::f16 (A from TMEM, B from smem, fp32 accumulate in
//    TMEM) for every product pair (a_i, w_j) with i + j < PARTS, i.e. an fp32-accurate split product;
//  * the accumulators of a stage are read back (tcgen05.ld), split again and written as the next
//    stage's A operand -- the intermediates c and u never touch HBM.
// chain3_tc runs stage1 (per input group) -> stage2 (dense across groups) -> stage3 (per output
// group): forward x -> y (W1 = M, W2 = L, W3 = B', + bias) and adjoint dy -> dx (W1 = B', W2 = L,
// W3 = M; transposed descriptors).  gram_tc computes the LSC weight Gram G = sum_v g c^T with
// g = B'^T dy and c = M x produced on the tensor cores and staged in SWIZZLE_128B smem tiles.
#include "common.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace dl {
namespace tc {

using namespace dl::umma;

constexpr int kTileV = 128;          // voxels per tile (MMA M)
constexpr int kEW = 2;               // epilogue warps per TMEM lane quadrant
constexpr int kEWarps = 4 * kEW;     // 8 epilogue warps
constexpr int kThreads = (kEWarps + 1) * 32;

__host__ __device__ constexpr int npairs(int parts) { return parts * (parts + 1) / 2; }

// (i, j) product pairs of a `parts`-term split with i + j < parts, small terms first.
__device__ __forceinline__ void pair_of(int parts, int idx, int& i, int& j) {
  if (parts == 3) {
    const int pi[6] = {2, 1, 0, 1, 0, 0}, pj[6] = {0, 1, 2, 0, 1, 0};
    i = pi[idx];
    j = pj[idx];
  } else if (parts == 2) {
    const int pi[3] = {1, 0, 0}, pj[3] = {0, 1, 0};
    i = pi[idx];
    j = pj[idx];
  } else {
    i = j = 0;
  }
}

// Compile-time (i, j) pair lists (activation term i, weight term j).
template <int P> struct Pairs;
template <> struct Pairs<3> {
  static constexpr int n = 6;
  __device__ static constexpr int i(int k) { return k == 0 ? 2 : k == 1 ? 1 : k == 2 ? 0 : k == 3 ? 1 : 0; }
  __device__ static constexpr int j(int k) { return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 0 : k == 4 ? 1 : 0; }
};
template <> struct Pairs<2> {
  static constexpr int n = 3;
  __device__ static constexpr int i(int k) { return k == 0 ? 1 : 0; }
  __device__ static constexpr int j(int k) { return k == 1 ? 1 : 0; }
};

// Byte advance of a weight descriptor per K-step (added to the start-address field, >> 4).
__device__ __forceinline__ uint64_t wkstep(int cols, int kmajor) {
  return kmajor ? (uint64_t)(256 >> 4) : (uint64_t)((2u * (uint32_t)(cols / 8) * 128u) >> 4);
}

// Issue all product pairs of one K-step: D (+)= A_i(TMEM) . B_j for i + j < P.
template <int P>
__device__ __forceinline__ void kstep_ts(uint32_t d, uint32_t a0, uint32_t a_part_cols, const uint64_t (&b)[P],
                                         uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < Pairs<P>::n; ++k)
    mma_ts(d, a0 + (uint32_t)Pairs<P>::i(k) * a_part_cols, b[Pairs<P>::j(k)], idesc, (first && k == 0) ? 0u : 1u);
}

// Descriptor of a weight image (rows x cols bf16, core-matrix blocked) for K-step kk.
//  kmajor: MN = rows, K = cols;  else: K = rows, MN = cols.  mn0 = first MN index (multiple of 8).
__device__ __forceinline__ uint64_t wdesc(uint32_t img, int rows, int cols, int kmajor, int mn0, int kk) {
  if (kmajor) {
    const uint32_t sbo = (uint32_t)(cols / 8) * 128u;
    return desc_noswz(img + (uint32_t)(mn0 / 8) * sbo + (uint32_t)kk * 256u, 128u, sbo);
  }
  const uint32_t lbo = (uint32_t)(cols / 8) * 128u;
  return desc_noswz(img + (uint32_t)(mn0 / 8) * 128u + (uint32_t)kk * 2u * lbo, lbo, 128u);
  (void)rows;
}

struct Chain3 {
  const float* in;
  float* out;
  const float* bias2;                 // real stage-2 bias per (group, channel < C2) or null
  const uint16_t* w1;                 // images, part-major: (q * groups + g) * img_bytes
  const uint16_t* w2;
  const uint16_t* w3;
  int64_t nbatch, nvox, in_bs, out_bs, tiles_per_b;
  int G1, C1, K1, N1;                 // stage 1: groups, real in-ch/group, padded K, padded N
  int G2, C2, N2;                     // stage 2: groups, real out-ch/group, padded N
  int C3, N3;                         // stage 3: real / padded out-ch per group
  int w1_groups, w3_groups;
  int adjoint;
  uint32_t w1_img, w2_img, w3_img;    // bytes per image
  uint32_t sm_w1, sm_w2, sm_w3, sm_tab, sm_bar, smem_bytes;
  uint32_t colA1, colD1, colA2, colD2, colA3, colD3;
  int d3_sync;
  long long* prof;                    // optional phase timestamps (CTA 0, first 8 tiles), debug only
};

struct Bars {
  uint64_t ax_full, ax_empty, c_full, ac_full, au_full, y_full;
  uint64_t u_full[4];
  uint32_t tmem_base;
};

// ---------------------------------------------------------------------------- epilogue helpers
template <int PARTS>
__device__ __forceinline__ void split_store16(uint32_t taddr_part0, uint32_t part_stride_cols, const float (&v)[16]) {
  uint32_t w[PARTS][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t p[PARTS];
    split_pair<PARTS>(v[2 * i], v[2 * i + 1], p);
#pragma unroll
    for (int q = 0; q < PARTS; ++q) w[q][i] = p[q];
  }
#pragma unroll
  for (int q = 0; q < PARTS; ++q) tmem_st<8>(taddr_part0 + (uint32_t)q * part_stride_cols, w[q]);
}

__device__ __forceinline__ void ld16f(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tmem_ld<16>(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

#define DL_PROF(ev)                                                                    \
  do {                                                                                 \
    if (p.prof && blockIdx.x == 0 && it < 8 && (threadIdx.x & 31) == 0)                \
      p.prof[(it * 2 + (warp == kEWarps)) * 32 + (ev)] = clock64();                    \
  } while (0)

__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// One MMA of an issue table: B descriptor, A TMEM column, D TMEM column | accumulate << 31.
struct MmaEnt {
  uint64_t b;
  uint32_t a;
  uint32_t d;
};

// One SS MMA (both operands from shared memory) with its own instruction descriptor.
struct SsEnt {
  uint64_t a;
  uint64_t b;
  uint32_t d;
  uint32_t idesc;
};

__device__ __forceinline__ void issue_ts(const MmaEnt* e, int n, uint32_t tbase, uint32_t idesc) {
#pragma unroll 4
  for (int k = 0; k < n; ++k) {
    const MmaEnt m = e[k];
    mma_ts(tbase + (m.d & 0x7FFFFFFFu), tbase + m.a, m.b, idesc, m.d >> 31);
  }
}

// ---------------------------------------------------------------------------- chain3 kernel
template <int PARTS, int MAXC>
__global__ void __launch_bounds__(kThreads, 1) chain3_tc(const Chain3 p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- stage all weight images once per CTA ----
  {
    const uint32_t b1 = (uint32_t)PARTS * p.w1_groups * p.w1_img;
    const uint32_t b2 = (uint32_t)PARTS * p.w2_img;
    const uint32_t b3 = (uint32_t)PARTS * p.w3_groups * p.w3_img;
    const uint4* s1 = reinterpret_cast<const uint4*>(p.w1);
    const uint4* s2 = reinterpret_cast<const uint4*>(p.w2);
    const uint4* s3 = reinterpret_cast<const uint4*>(p.w3);
    uint4* d1 = reinterpret_cast<uint4*>(smem + p.sm_w1);
    uint4* d2 = reinterpret_cast<uint4*>(smem + p.sm_w2);
    uint4* d3 = reinterpret_cast<uint4*>(smem + p.sm_w3);
    for (uint32_t i = threadIdx.x; i < b1 / 16; i += blockDim.x) d1[i] = __ldg(s1 + i);
    for (uint32_t i = threadIdx.x; i < b2 / 16; i += blockDim.x) d2[i] = __ldg(s2 + i);
    for (uint32_t i = threadIdx.x; i < b3 / 16; i += blockDim.x) d3[i] = __ldg(s3 + i);
  }
  if (warp == kEWarps) tmem_alloc(&bars.tmem_base, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bars.ax_full, kEWarps);
    mbar_init(&bars.ax_empty, 1);
    mbar_init(&bars.c_full, 1);
    mbar_init(&bars.ac_full, kEWarps);
    mbar_init(&bars.au_full, kEWarps);
    mbar_init(&bars.y_full, 1);
    for (int o = 0; o < 4; ++o) mbar_init(&bars.u_full[o], 1);
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;

  if (warp < kEWarps) {
    // =========================== epilogue / loader warps ===========================
    const int qd = warp & 3, cg = warp >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int row = 32 * qd + lane;
    const int nck1 = p.K1 / 16;
    float pf[MAXC][16];
    auto load_item = [&](int64_t t, int g) {
      const int64_t b = t / p.tiles_per_b;
      const int64_t v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool ok = v < p.nvox;
      const float* src = p.in + b * p.in_bs + (int64_t)g * p.C1 * p.nvox + v;
#pragma unroll
      for (int ci = 0; ci < MAXC; ++ci) {
        const int ck = cg + ci * kEW;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = ck * 16 + i;
          pf[ci][i] = (ck < nck1 && n < p.C1 && ok) ? __ldg(src + (int64_t)n * p.nvox) : 0.f;
        }
      }
    };
    uint32_t n_ax = 0, n_y = 0, it = 0;
    int64_t t = blockIdx.x;
    if (t < ntiles) load_item(t, 0);
    for (; t < ntiles; t += gridDim.x, ++it) {
      const int64_t b = t / p.tiles_per_b;
      const int64_t v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool vok = v < p.nvox;
      if (warp == 0) DL_PROF(0);
      // ---- stage-1 inputs, one group at a time (register prefetch of the next group) ----
      for (int g = 0; g < p.G1; ++g) {
        float cur[MAXC][16];
#pragma unroll
        for (int ci = 0; ci < MAXC; ++ci)
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[ci][i] = pf[ci][i];
        if (g + 1 < p.G1) load_item(t, g + 1);
        else if (t + gridDim.x < ntiles) load_item(t + gridDim.x, 0);
        if (warp == 0) DL_PROF(1 + 2 * g);
        if (n_ax > 0) mbar_wait(&bars.ax_empty, (n_ax - 1) & 1);
        fence_after();
#pragma unroll
        for (int ci = 0; ci < MAXC; ++ci) {
          const int ck = cg + ci * kEW;
          if (ck < nck1) split_store16<PARTS>(tq + p.colA1 + (uint32_t)ck * 8, p.K1 / 2, cur[ci]);
        }
        tmem_wait_st();
        fence_before();
        warp_arrive(&bars.ax_full);
        if (warp == 0) DL_PROF(2 + 2 * g);
        ++n_ax;
      }
      // ---- stage-1 accumulators -> stage-2 A operand ----
      mbar_wait(&bars.c_full, it & 1);
      if (warp == 0) DL_PROF(8);
      fence_after();
      {
        const int D1 = p.G1 * p.N1, nck = D1 / 16;
        for (int ck = cg; ck < nck; ck += kEW) {
          float vv[16];
          ld16f(tq + p.colD1 + (uint32_t)ck * 16, vv);
          split_store16<PARTS>(tq + p.colA2 + (uint32_t)ck * 8, D1 / 2, vv);
        }
      }
      tmem_wait_st();
      fence_before();
      warp_arrive(&bars.ac_full);
      // ---- per output group: stage-2 accumulators (+bias) -> stage-3 A; stage-3 -> HBM ----
      mbar_wait(&bars.u_full[0], it & 1);
      fence_after();
      for (int o = 0; o < p.G2; ++o) {
        const int nck2 = p.N2 / 16;
        for (int ck = cg; ck < nck2; ck += kEW) {
          float vv[16];
          ld16f(tq + p.colD2 + (uint32_t)(o * p.N2 + ck * 16), vv);
          if (p.bias2) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int r = ck * 16 + i;
              if (r < p.C2) vv[i] += __ldg(p.bias2 + o * p.C2 + r);
            }
          }
          split_store16<PARTS>(tq + p.colA3 + (uint32_t)ck * 8, p.N2 / 2, vv);
        }
        tmem_wait_st();
        fence_before();
        warp_arrive(&bars.au_full);
        if (warp == 0) DL_PROF(11 + 3 * o);
        mbar_wait(&bars.y_full, n_y & 1);
        if (warp == 0) DL_PROF(12 + 3 * o);
        ++n_y;
        fence_after();
        float* dst = p.out + b * p.out_bs + (int64_t)o * p.C3 * p.nvox + v;
        const int nck3 = p.N3 / 16;
        for (int ck = cg; ck < nck3; ck += kEW) {
          float vv[16];
          ld16f(tq + p.colD3 + (uint32_t)ck * 16, vv);
          if (vok) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int n = ck * 16 + i;
              if (n < p.C3) __stcs(dst + (int64_t)n * p.nvox, vv[i]);
            }
          }
        }
        if (warp == 0) DL_PROF(13 + 3 * o);
        fence_before();
      }
    }
  } else {
    // =========================== MMA issuer (converged warp, one elected lane issues) ===========
    const uint32_t sw1 = smem_u32(smem + p.sm_w1), sw2 = smem_u32(smem + p.sm_w2), sw3 = smem_u32(smem + p.sm_w3);
    const int km = p.adjoint ? 0 : 1;   // forward: K-major weights; adjoint: MN-major
    const int K2 = p.G1 * p.N1, NT2 = p.G2 * p.N2;
    const bool merge2 = NT2 <= 256;     // one MMA spans every stage-2 output group
    const uint32_t id1 = idesc_bf16(128, p.N1, 0, 1 - km);
    const uint32_t id2 = idesc_bf16(128, merge2 ? NT2 : p.N2, 0, 1 - km);
    const uint32_t id3 = idesc_bf16(128, p.N3, 0, 1 - km);
    const int r1 = km ? p.N1 : p.K1, c1 = km ? p.K1 : p.N1;
    const int r2 = km ? NT2 : K2, c2 = km ? K2 : NT2;
    const int r3 = km ? p.N3 : p.N2, c3 = km ? p.N2 : p.N3;
    const uint64_t ks1 = wkstep(c1, km), ks2 = wkstep(c2, km), ks3 = wkstep(c3, km);
    const int nk1 = p.K1 / 16, nk2 = K2 / 16, nk3 = p.N2 / 16;
    uint32_t n_ax = 0, n_au = 0, it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      for (int g = 0; g < p.G1; ++g) {
        const int wg = p.w1_groups > 1 ? g : 0;
        uint64_t b[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) b[j] = wdesc(sw1 + (uint32_t)(j * p.w1_groups + wg) * p.w1_img, r1, c1, km, 0, 0);
        DL_PROF(1 + 2 * g);
        mbar_wait(&bars.ax_full, n_ax & 1);
        DL_PROF(2 + 2 * g);
        ++n_ax;
        fence_after();
        const uint32_t d = tbase + p.colD1 + (uint32_t)(g * p.N1);
        for (int kk = 0; kk < nk1; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(d, tbase + p.colA1 + 8u * kk, p.K1 / 2, b, id1, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) b[j] += ks1;
        }
        if (elect_one()) commit(&bars.ax_empty);
        __syncwarp();
      }
      if (elect_one()) commit(&bars.c_full);
      __syncwarp();
      DL_PROF(8);
      mbar_wait(&bars.ac_full, it & 1);
      DL_PROF(9);
      fence_after();
      for (int o = 0; o < (merge2 ? 1 : p.G2); ++o) {
        uint64_t b[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) b[j] = wdesc(sw2 + (uint32_t)j * p.w2_img, r2, c2, km, o * p.N2, 0);
        const uint32_t d = tbase + p.colD2 + (uint32_t)(o * p.N2);
        for (int kk = 0; kk < nk2; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(d, tbase + p.colA2 + 8u * kk, K2 / 2, b, id2, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) b[j] += ks2;
        }
      }
      if (elect_one()) commit(&bars.u_full[0]);
      __syncwarp();
      DL_PROF(10);
      if (p.d3_sync) {
        mbar_wait(&bars.u_full[0], it & 1);
        fence_after();
      }
      for (int o = 0; o < p.G2; ++o) {
        const int wg = p.w3_groups > 1 ? o : 0;
        uint64_t b[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) b[j] = wdesc(sw3 + (uint32_t)(j * p.w3_groups + wg) * p.w3_img, r3, c3, km, 0, 0);
        mbar_wait(&bars.au_full, n_au & 1);
        DL_PROF(11 + 3 * o);
        ++n_au;
        fence_after();
        for (int kk = 0; kk < nk3; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(tbase + p.colD3, tbase + p.colA3 + 8u * kk, p.N2 / 2, b, id3, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) b[j] += ks3;
        }
        if (elect_one()) commit(&bars.y_full);
        __syncwarp();
        DL_PROF(12 + 3 * o);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kEWarps) tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------- operand packing
// `ng` row-major fp32 matrices of (nrb*rb) x (ncb*cb) -> PARTS bf16 images each of (nrb*rbp) x (ncb*cbp)
// in the core-matrix blocked layout, image (q, g) at (q * ng + g) * img_elems.  Padding is zero.
__global__ void pack_k(const float* __restrict__ W, uint16_t* __restrict__ out, int ng, int nrb, int rb, int rbp,
                       int ncb, int cb, int cbp, int parts) {
  const int R = nrb * rbp, C = ncb * cbp;
  const int64_t img = (int64_t)R * C;
  const int64_t n = img * ng;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(e / img);
    const int rc = (int)(e - (int64_t)g * img);
    const int r = rc / C, c = rc - r * C;
    const int bi = r / rbp, rr = r - bi * rbp, bj = c / cbp, cc = c - bj * cbp;
    float v = 0.f;
    if (rr < rb && cc < cb) v = __ldg(W + (int64_t)g * (nrb * rb) * (ncb * cb) + (int64_t)(bi * rb + rr) * (ncb * cb) + bj * cb + cc);
    const int64_t off = ((int64_t)(r >> 3) * (C >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7);
    for (int q = 0; q < parts; ++q) {
      const uint32_t pk = pack_bf16x2(v, 0.f);
      out[((int64_t)q * ng + g) * img + off] = (uint16_t)(pk & 0xFFFFu);
      v -= bf16lo_to_f32(pk);
    }
  }
}

// ---------------------------------------------------------------------------- LSC weight Gram
struct GramP {
  const float* x;
  const float* dy;
  const uint16_t* wM;        // M images (rows RPi, cols NPi), PARTS x groups
  const uint16_t* wB;        // B' images (rows NPo, cols RPo), PARTS
  const float* beta;         // R_out
  float* partials;           // [grid][GR*GC] then db [grid][S_out]
  int64_t nbatch, nvox, x_bs, dy_bs, tiles_per_b;
  int S_in, N, NPi, RPi, S_out, N_out, NPo, RPo, R_out;
  int wM_groups;
  uint32_t wM_img, wB_img;
  uint32_t sm_wM, sm_wB, sm_c, sm_g, sm_tab, sm_bar, smem_bytes, ctile, gtile;   // per-part tile bytes
  uint32_t colGA, colGB, colGC, colA, colD;
  int GR, GC;                // g rows (S_out*RPo), c rows (S_in*RPi)
};

struct GBars {
  uint64_t a_full, a_empty, d_full, tiles_full, gram_done;
  float db[4];
  uint32_t tmem_base;
};

// byte offset of (row j, voxel k) in a SWIZZLE_128B K-major tile with `rows` rows (K = 128 voxels)
__device__ __forceinline__ uint32_t sw128_off(int j, int k, int rows) {
  return (uint32_t)(k >> 6) * (uint32_t)(rows >> 3) * 1024u + (uint32_t)(j >> 3) * 1024u + (uint32_t)(j & 7) * 128u +
         (uint32_t)((((k & 63) >> 3) ^ (j & 7)) << 4) + (uint32_t)(k & 7) * 2u;
}

template <int PARTS, int MAXC>
__global__ void __launch_bounds__(kThreads, 1) gram_tc(const GramP p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  GBars& bars = *reinterpret_cast<GBars*>(smem + p.sm_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const uint32_t bM = (uint32_t)PARTS * p.wM_groups * p.wM_img, bB = (uint32_t)PARTS * p.wB_img;
    const uint4* sM = reinterpret_cast<const uint4*>(p.wM);
    const uint4* sB = reinterpret_cast<const uint4*>(p.wB);
    uint4* dM = reinterpret_cast<uint4*>(smem + p.sm_wM);
    uint4* dB = reinterpret_cast<uint4*>(smem + p.sm_wB);
    for (uint32_t i = threadIdx.x; i < bM / 16; i += blockDim.x) dM[i] = __ldg(sM + i);
    for (uint32_t i = threadIdx.x; i < bB / 16; i += blockDim.x) dB[i] = __ldg(sB + i);
    // zero both operand tiles once: padding rows/garbage rows must stay finite
    uint4* z = reinterpret_cast<uint4*>(smem + p.sm_c);
    const uint32_t zb = p.sm_bar - p.sm_c;
    for (uint32_t i = threadIdx.x; i < zb / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (warp == kEWarps) tmem_alloc(&bars.tmem_base, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bars.a_full, kEWarps);
    mbar_init(&bars.a_empty, 1);
    mbar_init(&bars.d_full, 1);
    mbar_init(&bars.tiles_full, kEWarps);
    mbar_init(&bars.gram_done, 1);
    for (int o = 0; o < 4; ++o) bars.db[o] = 0.f;
    mbar_fence_init();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = bars.tmem_base;
  const int64_t ntiles = p.nbatch * p.tiles_per_b;

  if (warp < kEWarps) {
    const int qd = warp & 3, cg = warp >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16);
    const int row = 32 * qd + lane;
    float dbacc[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t n_a = 0, n_d = 0, it = 0;
    // one "item" = one group of one operand: items 0..S_out-1 are dy groups, S_out.. are x groups
    auto load_group = [&](const float* base, int64_t bs, int C, int K, int64_t t, int g, float (&buf)[MAXC][16]) {
      const int64_t b = t / p.tiles_per_b;
      const int64_t v = (t - b * p.tiles_per_b) * kTileV + row;
      const bool ok = v < p.nvox;
      const float* src = base + b * bs + (int64_t)g * C * p.nvox + v;
      const int nck = K / 16;
#pragma unroll
      for (int ci = 0; ci < MAXC; ++ci) {
        const int ck = cg + ci * kEW;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = ck * 16 + i;
          buf[ci][i] = (ck < nck && n < C && ok) ? __ldg(src + (int64_t)n * p.nvox) : 0.f;
        }
      }
    };
    auto put_a = [&](const float (&cur)[MAXC][16], int K) {
      if (n_a > 0) mbar_wait(&bars.a_empty, (n_a - 1) & 1);
      fence_after();
      const int nck = K / 16;
#pragma unroll
      for (int ci = 0; ci < MAXC; ++ci) {
        const int ck = cg + ci * kEW;
        if (ck < nck) split_store16<PARTS>(tq + p.colA + (uint32_t)ck * 8, K / 2, cur[ci]);
      }
      tmem_wait_st();
      fence_before();
      warp_arrive(&bars.a_full);
      ++n_a;
    };
    // D (fp32) -> two bf16 terms in the SW128 tile; for g also accumulate beta . g per output shell
    auto drain = [&](uint32_t tile, int rows, int nch, bool is_g) {
      mbar_wait(&bars.d_full, n_d & 1);
      ++n_d;
      fence_after();
      for (int ck = cg; ck < nch / 16; ck += kEW) {
        float vv[16];
        ld16f(tq + p.colD + (uint32_t)ck * 16, vv);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = ck * 16 + i;
          if (is_g) {
            const int o = j / p.RPo, r = j - o * p.RPo;
            if (r < p.R_out && o < 4) dbacc[o] += __ldg(p.beta + r) * vv[i];
          }
          const uint32_t pk0 = pack_bf16x2(vv[i], 0.f);
          const float rem = vv[i] - bf16lo_to_f32(pk0);
          const uint32_t pk1 = pack_bf16x2(rem, 0.f);
          const uint32_t off = sw128_off(j, row, rows);
          *reinterpret_cast<uint16_t*>(smem + tile + off) = (uint16_t)pk0;
          *reinterpret_cast<uint16_t*>(smem + tile + p.gtile * 0 + (is_g ? p.gtile : p.ctile) + off) = (uint16_t)pk1;
        }
      }
    };
    float pf[MAXC][16];
    int64_t t = blockIdx.x;
    if (t < ntiles) load_group(p.dy, p.dy_bs, p.N_out, p.NPo, t, 0, pf);
    for (; t < ntiles; t += gridDim.x, ++it) {
      // ---- g = B'^T dy, one output shell at a time ----
      for (int o = 0; o < p.S_out; ++o) {
        float cur[MAXC][16];
#pragma unroll
        for (int ci = 0; ci < MAXC; ++ci)
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[ci][i] = pf[ci][i];
        if (o + 1 < p.S_out) load_group(p.dy, p.dy_bs, p.N_out, p.NPo, t, o + 1, pf);
        else load_group(p.x, p.x_bs, p.N, p.NPi, t, 0, pf);
        put_a(cur, p.NPo);
      }
      if (it > 0) mbar_wait(&bars.gram_done, (it - 1) & 1);   // operand tiles free again
      drain(p.sm_g, p.GR < 128 ? 128 : p.GR, p.GR, true);
      // ---- c = M x, one input shell at a time ----
      for (int s = 0; s < p.S_in; ++s) {
        float cur[MAXC][16];
#pragma unroll
        for (int ci = 0; ci < MAXC; ++ci)
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[ci][i] = pf[ci][i];
        if (s + 1 < p.S_in) load_group(p.x, p.x_bs, p.N, p.NPi, t, s + 1, pf);
        else if (t + gridDim.x < ntiles) load_group(p.dy, p.dy_bs, p.N_out, p.NPo, t + gridDim.x, 0, pf);
        put_a(cur, p.NPi);
      }
      drain(p.sm_c, p.GC, p.GC, false);
      fence_proxy_async();
      fence_before();
      warp_arrive(&bars.tiles_full);
    }
    if (it > 0) mbar_wait(&bars.gram_done, (it - 1) & 1);
    fence_after();
    // ---- write this CTA's Gram partial: G[j (g row)][i (c row)] ----
    float* part = p.partials + (int64_t)blockIdx.x * p.GR * p.GC;
    const int rA = row;  // block A: lane = g row
    for (int ck = cg; ck < p.GC / 16; ck += kEW) {
      float vv[16];
      ld16f(tq + p.colGA + (uint32_t)ck * 16, vv);
      if (rA < p.GR)
#pragma unroll
        for (int i = 0; i < 16; ++i) part[(int64_t)rA * p.GC + ck * 16 + i] = vv[i];
    }
    if (p.GR > 128 && cg == 0) {
      float vv[16];
      ld16f(tq + p.colGB, vv);   // block B: lane = c row i (< 128), col = g row 128 + c
      if (row < p.GC)
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (128 + c < p.GR) part[(int64_t)(128 + c) * p.GC + row] = vv[c];
      if (p.GC > 128 && qd == 0) {
        ld16f(tq + p.colGC, vv);   // block C (M=64): lanes 0..15 = c rows 128..143
        if (lane < 16 && 128 + lane < p.GC)
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (128 + c < p.GR) part[(int64_t)(128 + c) * p.GC + 128 + lane] = vv[c];
      }
    }
    // ---- db partial: sum over this CTA's voxels of beta . g[o] ----
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      float s = dbacc[o];
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0 && o < p.S_out) atomicAdd(&bars.db[o], s);
    }
    named_sync(1, kEWarps * 32);
    if (threadIdx.x == 0) {
      float* dbp = p.partials + (int64_t)gridDim.x * p.GR * p.GC + (int64_t)blockIdx.x * p.S_out;
      for (int o = 0; o < p.S_out; ++o) dbp[o] = bars.db[o];
    }
  } else {
    // =========================== MMA issuer (converged warp, one elected lane issues) ===========
    const uint32_t sM = smem_u32(smem + p.sm_wM), sB = smem_u32(smem + p.sm_wB);
    const uint32_t sc = smem_u32(smem + p.sm_c), sg = smem_u32(smem + p.sm_g);
    const uint32_t idg = idesc_bf16(128, p.RPo, 0, 1);   // g: A = dy (TMEM), B = B' image MN-major
    const uint32_t idc = idesc_bf16(128, p.RPi, 0, 0);   // c: B = M image K-major
    const uint32_t idA = idesc_bf16(128, p.GC, 0, 0), idB = idesc_bf16(128, 16, 0, 0), idC = idesc_bf16(64, 16, 0, 0);
    const int grow = p.GR < 128 ? 128 : p.GR;
    const uint32_t ASg = (uint32_t)(grow / 8) * 1024u, ASc = (uint32_t)(p.GC / 8) * 1024u;
    const uint64_t ksg = wkstep(p.RPo, 0), ksc = wkstep(p.NPi, 1);
    const int nkg = p.NPo / 16, nkc = p.NPi / 16;
    uint32_t n_a = 0, it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      for (int o = 0; o < p.S_out; ++o) {
        uint64_t b[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) b[j] = wdesc(sB + (uint32_t)j * p.wB_img, p.NPo, p.RPo, 0, 0, 0);
        mbar_wait(&bars.a_full, n_a & 1);
        ++n_a;
        fence_after();
        const uint32_t d = tbase + p.colD + (uint32_t)(o * p.RPo);
        for (int kk = 0; kk < nkg; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(d, tbase + p.colA + 8u * kk, p.NPo / 2, b, idg, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) b[j] += ksg;
        }
        if (elect_one()) commit(&bars.a_empty);
        __syncwarp();
      }
      if (elect_one()) commit(&bars.d_full);
      __syncwarp();
      for (int s = 0; s < p.S_in; ++s) {
        const int wg = p.wM_groups > 1 ? s : 0;
        uint64_t b[PARTS];
#pragma unroll
        for (int j = 0; j < PARTS; ++j) b[j] = wdesc(sM + (uint32_t)(j * p.wM_groups + wg) * p.wM_img, p.RPi, p.NPi, 1, 0, 0);
        mbar_wait(&bars.a_full, n_a & 1);
        ++n_a;
        fence_after();
        const uint32_t d = tbase + p.colD + (uint32_t)(s * p.RPi);
        for (int kk = 0; kk < nkc; ++kk) {
          if (elect_one()) kstep_ts<PARTS>(d, tbase + p.colA + 8u * kk, p.NPi / 2, b, idc, kk == 0);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < PARTS; ++j) b[j] += ksc;
        }
        if (elect_one()) commit(&bars.a_empty);
        __syncwarp();
      }
      if (elect_one()) commit(&bars.d_full);
      __syncwarp();
      // ---- Gram over this tile's 128 voxels (two-term split operands, three blocks) ----
      mbar_wait(&bars.tiles_full, it & 1);
      fence_after();
      for (int kk = 0; kk < kTileV / 16; ++kk) {
        const uint32_t ko = (uint32_t)(kk >> 2), kb = (uint32_t)(kk & 3) * 32u;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int i = Pairs<2>::i(k), j = Pairs<2>::j(k);
            const uint32_t gI = sg + (uint32_t)i * p.gtile + ko * ASg + kb, gJ = sg + (uint32_t)j * p.gtile + ko * ASg + kb;
            const uint32_t cI = sc + (uint32_t)i * p.ctile + ko * ASc + kb, cJ = sc + (uint32_t)j * p.ctile + ko * ASc + kb;
            const uint32_t acc = (it > 0 || kk > 0 || k > 0) ? 1u : 0u;
            mma_ss(tbase + p.colGA, desc_sw128_k(gI, 1024), desc_sw128_k(cJ, 1024), idA, acc);
            if (p.GR > 128) {
              mma_ss(tbase + p.colGB, desc_sw128_k(cI, 1024), desc_sw128_k(gJ + 16 * 1024, 1024), idB, acc);
              if (p.GC > 128)
                mma_ss(tbase + p.colGC, desc_sw128_k(cI + 16 * 1024, 1024), desc_sw128_k(gJ + 16 * 1024, 1024), idC, acc);
            }
          }
        }
        __syncwarp();
      }
      if (elect_one()) commit(&bars.gram_done);
      __syncwarp();
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kEWarps) tmem_dealloc(tbase, 512);
}

// fixed-order float64 reduction of the per-CTA Gram partials, then dW = <P_k, G_{o,s}>, db = sum of partials
__global__ void gram_reduce_k(const float* __restrict__ partials, double* __restrict__ G, int nparts, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nparts; ++q) s += (double)__ldg(partials + (int64_t)q * n + e);
    G[e] = s;
  }
}

__global__ void gram_finalize_k(const double* __restrict__ G, const float* __restrict__ dbparts, int nparts,
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
    for (int q = threadIdx.x; q < nparts; q += blockDim.x) acc += (double)__ldg(dbparts + (int64_t)q * s_out + o);
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

}  // namespace tc
}  // namespace dl

// ============================================================================ host side
namespace dl {
namespace tc {
namespace {

inline int r16(int64_t x) { return (int)((x + 15) / 16 * 16); }
inline size_t al(size_t x, size_t a) { return (x + a - 1) / a * a; }

long long* g_prof = nullptr;   // debug: phase timestamps of the next chain3 launch

int split_terms() {
  static int v = [] {
    const char* e = getenv("DELIMIT_SPLIT_TERMS");
    const int t = e ? atoi(e) : 3;
    return (t == 2 || t == 3) ? t : 3;
  }();
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
  size_t imgM, imgL, imgB, parts, G, total;
  uint32_t bM, bL, bB;   // bytes per image
  int nparts;
};

WsLayout ws_layout(const Dims& d, int nparts) {
  WsLayout w;
  w.bM = (uint32_t)(d.RPi * d.NPi * 2);
  w.bL = (uint32_t)((d.s_out * d.RPo) * (d.s_in * d.RPi) * 2);
  w.bB = (uint32_t)(d.NPo * d.RPo * 2);
  const int GR = d.s_out * d.RPo, GC = d.s_in * d.RPi;
  size_t o = 0;
  w.imgM = o; o = al(o + (size_t)3 * d.mg * w.bM, 256);
  w.imgL = o; o = al(o + (size_t)3 * w.bL, 256);
  w.imgB = o; o = al(o + (size_t)3 * w.bB, 256);
  w.parts = o; o = al(o + (size_t)nparts * ((size_t)GR * GC + d.s_out) * 4, 256);
  w.G = o; o = al(o + (size_t)GR * GC * 8, 256);
  w.total = o;
  w.nparts = nparts;
  return w;
}

constexpr int kMaxParts = 256;

// TMEM / smem plan for one chain3 direction; returns false if it does not fit.
bool plan_chain3(Chain3& p, int parts) {
  const int A1 = parts * p.K1 / 2, D1 = p.G1 * p.N1, A2 = parts * D1 / 2, D2 = p.G2 * p.N2, A3 = parts * p.N2 / 2;
  if (p.N1 > 256 || p.N2 > 256 || p.N3 > 256 || p.G2 > 4 || (p.K1 / 16 + kEW - 1) / kEW > 8) return false;
  p.colA1 = 0;
  p.colD1 = A1;
  p.colA2 = A1 + D1;
  p.colD2 = 0;
  // D2 reuses [0, ...) once stage 1 is drained; it must not overlap A2 (read by stage-2 MMAs).
  if ((int)p.colA2 + A2 > 512 || D2 > (int)p.colA2 || D1 > 512) return false;
  p.d3_sync = 0;
  if (D2 + A3 <= (int)p.colA2) {
    // A3 right after D2 (below A2); D3 after A2, or over A2 once all stage-2 MMAs completed
    p.colA3 = D2;
    if ((int)p.colA2 + A2 + p.N3 <= 512) {
      p.colD3 = p.colA2 + A2;
    } else if (D2 + A3 + p.N3 <= 512) {
      p.colD3 = D2 + A3;
      p.d3_sync = 1;
    } else {
      return false;
    }
  } else if ((int)p.colA2 + A2 + A3 + p.N3 <= 512) {
    p.colA3 = p.colA2 + A2;  // both stage-3 buffers above A2
    p.colD3 = p.colA3 + A3;
  } else {
    return false;
  }
  p.w1_img = (uint32_t)(p.N1 * p.K1 * 2);
  p.w2_img = (uint32_t)((p.G2 * p.N2) * (p.G1 * p.N1) * 2);
  p.w3_img = (uint32_t)(p.N3 * p.N2 * 2);
  size_t o = 0;
  p.sm_w1 = (uint32_t)o; o = al(o + (size_t)parts * p.w1_groups * p.w1_img, 1024);
  p.sm_w2 = (uint32_t)o; o = al(o + (size_t)parts * p.w2_img, 1024);
  p.sm_w3 = (uint32_t)o; o = al(o + (size_t)parts * p.w3_groups * p.w3_img, 1024);
  {
    const int np = parts * (parts + 1) / 2, NT2 = p.G2 * p.N2;
    const int n2g = NT2 <= 256 ? 1 : p.G2;
    const size_t ents = (size_t)np * (p.G1 * (p.K1 / 16) + n2g * (p.G1 * p.N1 / 16) + p.G2 * (p.N2 / 16));
    p.sm_tab = (uint32_t)o; o = al(o + ents * 16, 16);
  }
  p.sm_bar = (uint32_t)o; o = al(o + sizeof(Bars), 16);
  p.smem_bytes = (uint32_t)o;
  return o <= 227 * 1024;
}

bool plan_gram(GramP& p, int parts) {
  p.GR = p.S_out * p.RPo;
  p.GC = p.S_in * p.RPi;
  if (p.GR > 144 || p.GC > 144 || p.S_out > 4) return false;
  const int grow = p.GR < 128 ? 128 : p.GR;
  p.colGA = 0;
  p.colGB = p.GC;
  p.colGC = p.GC + 16;
  p.colA = p.GC + 32;
  const int amax = parts * (p.NPo > p.NPi ? p.NPo : p.NPi) / 2;
  p.colD = p.colA + amax;
  const int dmax = p.GR > p.GC ? p.GR : p.GC;
  if ((int)p.colD + dmax > 512) return false;
  if ((p.NPo / 16 + kEW - 1) / kEW > 8 || (p.NPi / 16 + kEW - 1) / kEW > 8) return false;
  p.wM_img = (uint32_t)(p.RPi * p.NPi * 2);
  p.wB_img = (uint32_t)(p.NPo * p.RPo * 2);
  p.ctile = (uint32_t)(p.GC / 8) * 1024u * 2u;
  p.gtile = (uint32_t)(grow / 8) * 1024u * 2u;
  size_t o = 0;
  p.sm_wM = (uint32_t)o; o = al(o + (size_t)parts * p.wM_groups * p.wM_img, 1024);
  p.sm_wB = (uint32_t)o; o = al(o + (size_t)parts * p.wB_img, 1024);
  p.sm_c = (uint32_t)o; o = al(o + (size_t)2 * p.ctile, 1024);
  p.sm_g = (uint32_t)o; o = al(o + (size_t)2 * p.gtile, 1024);
  // block C reads c rows up to 191 of every K-atom: keep >= 8 KB of mapped smem after the g tile
  o = al(o + 8192, 1024);
  {
    const int np = parts * (parts + 1) / 2;
    const size_t ts = (size_t)np * (p.S_out * (p.NPo / 16) + p.S_in * (p.NPi / 16)) * 16;
    p.sm_tab = (uint32_t)o; o = al(o + ts + (size_t)(kTileV / 16) * 3 * 3 * sizeof(SsEnt), 16);
  }
  p.sm_bar = (uint32_t)o; o = al(o + sizeof(GBars), 16);
  p.smem_bytes = (uint32_t)o;
  return o <= 227 * 1024;
}

template <int PARTS, int MAXC>
int run_chain3_t(const Chain3& p, int grid, cudaStream_t st) {
  auto k = chain3_tc<PARTS, MAXC>;
  DL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes));
  k<<<grid, kThreads, p.smem_bytes, st>>>(p);
  return after_launch("chain3_tc");
}

template <int PARTS>
int run_chain3_p(const Chain3& p, int grid, cudaStream_t st) {
  const int mc = (p.K1 / 16 + kEW - 1) / kEW;
  if (mc <= 1) return run_chain3_t<PARTS, 1>(p, grid, st);
  if (mc <= 2) return run_chain3_t<PARTS, 2>(p, grid, st);
  if (mc <= 3) return run_chain3_t<PARTS, 3>(p, grid, st);
  if (mc <= 4) return run_chain3_t<PARTS, 4>(p, grid, st);
  return run_chain3_t<PARTS, 8>(p, grid, st);
}

template <int PARTS, int MAXC>
int run_gram_t(const GramP& p, int grid, cudaStream_t st) {
  auto k = gram_tc<PARTS, MAXC>;
  DL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes));
  k<<<grid, kThreads, p.smem_bytes, st>>>(p);
  return after_launch("gram_tc");
}

template <int PARTS>
int run_gram_p(const GramP& p, int grid, cudaStream_t st) {
  const int kmax = p.NPo > p.NPi ? p.NPo : p.NPi;
  const int mc = (kmax / 16 + kEW - 1) / kEW;
  if (mc <= 1) return run_gram_t<PARTS, 1>(p, grid, st);
  if (mc <= 2) return run_gram_t<PARTS, 2>(p, grid, st);
  if (mc <= 3) return run_gram_t<PARTS, 3>(p, grid, st);
  if (mc <= 4) return run_gram_t<PARTS, 4>(p, grid, st);
  return run_gram_t<PARTS, 8>(p, grid, st);
}

int pack(const float* W, uint16_t* out, int ng, int nrb, int rb, int rbp, int ncb, int cb, int cbp, int parts,
         cudaStream_t st) {
  const int64_t n = (int64_t)ng * nrb * rbp * ncb * cbp;
  const int blocks = (int)((n + 255) / 256 < 2048 ? (n + 255) / 256 : 2048);
  pack_k<<<blocks, 256, 0, st>>>(W, out, ng, nrb, rb, rbp, ncb, cb, cbp, parts);
  return after_launch("pack_operand");
}

int pack_all(const Dims& d, const WsLayout& w, uint8_t* ws, const float* M, const float* L, const float* Bt,
             cudaStream_t st) {
  if (M) DL_TRY(pack(M, reinterpret_cast<uint16_t*>(ws + w.imgM), d.mg, 1, d.r_in, d.RPi, 1, d.n, d.NPi, d.parts, st));
  if (L)
    DL_TRY(pack(L, reinterpret_cast<uint16_t*>(ws + w.imgL), 1, d.s_out, d.r_out, d.RPo, d.s_in, d.r_in, d.RPi,
                d.parts, st));
  if (Bt)
    DL_TRY(pack(Bt, reinterpret_cast<uint16_t*>(ws + w.imgB), 1, 1, d.n_out, d.NPo, 1, d.r_out, d.RPo, d.parts, st));
  return DL_OK;
}

Chain3 chain3_params(const Dims& d, const WsLayout& w, const uint8_t* ws, bool adjoint) {
  Chain3 p{};
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

GramP gram_params(const Dims& d, const WsLayout& w, uint8_t* ws) {
  GramP p{};
  p.nbatch = d.nbatch;
  p.nvox = d.nvox;
  p.tiles_per_b = (d.nvox + kTileV - 1) / kTileV;
  p.S_in = d.s_in; p.N = d.n; p.NPi = d.NPi; p.RPi = d.RPi;
  p.S_out = d.s_out; p.N_out = d.n_out; p.NPo = d.NPo; p.RPo = d.RPo; p.R_out = d.r_out;
  p.wM_groups = d.mg;
  p.wM = reinterpret_cast<const uint16_t*>(ws + w.imgM);
  p.wB = reinterpret_cast<const uint16_t*>(ws + w.imgB);
  p.partials = reinterpret_cast<float*>(ws + w.parts);
  p.x_bs = (int64_t)d.s_in * d.n * d.nvox;
  p.dy_bs = (int64_t)d.s_out * d.n_out * d.nvox;
  return p;
}

bool chain_fits(const Dims& d) {
  Chain3 f = chain3_params(d, ws_layout(d, 1), nullptr, false);
  Chain3 a = chain3_params(d, ws_layout(d, 1), nullptr, true);
  GramP g = gram_params(d, ws_layout(d, 1), nullptr);
  return plan_chain3(f, d.parts) && plan_chain3(a, d.parts) && plan_gram(g, d.parts);
}

int grid_for(int64_t ntiles, int sm) { return (int)(ntiles < sm ? (ntiles > 0 ? ntiles : 1) : sm); }

}  // namespace
}  // namespace tc
}  // namespace dl

extern "C" {

// Debug hook (not part of the documented ABI): record chain3 phase timestamps into `buf`
// (device, >= 8*2*32 int64) on subsequent forward launches; NULL disables.
void dl_debug_chain_prof(void* buf) { dl::tc::g_prof = reinterpret_cast<long long*>(buf); }

int dl_chain_supported(int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                       int m_per_shell) {
  using namespace dl::tc;
  return chain_fits(make_dims(1, s_in, s_out, n, r_in, r_out, n_out, 1, m_per_shell)) ? 1 : 0;
}

int dl_chain_split_terms(void) { return dl::tc::split_terms(); }

size_t dl_chain_workspace_bytes(int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out,
                                int64_t n_out, int64_t nvox) {
  using namespace dl::tc;
  return ws_layout(make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, 1), kMaxParts).total;
}

int dl_chain_fwd_f32(const float* x, float* y, const float* M, int m_per_shell, const float* L, const float* bvec,
                     const float* Bt, void* workspace, int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n,
                     int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream) {
  using namespace dl::tc;
  dl::begin_call();
  int sm = 0;
  DL_TRY(dl::device_check(&sm));
  DL_REQUIRE(x && y && M && L && Bt && workspace, "chain_fwd: null pointer");
  DL_REQUIRE(nbatch >= 0 && nvox >= 0 && s_in >= 1 && s_out >= 1 && n >= 1 && r_in >= 1 && r_out >= 1 && n_out >= 1,
             "chain_fwd: bad sizes");
  Dims d = make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, m_per_shell);
  WsLayout w = ws_layout(d, kMaxParts);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  Chain3 p = chain3_params(d, w, ws, false);
  DL_REQUIRE(plan_chain3(p, d.parts), "chain_fwd: channel counts exceed the fused kernel's TMEM/smem plan");
  if (nbatch == 0 || nvox == 0) return DL_OK;
  cudaStream_t st = dl::as_stream(stream);
  DL_TRY(pack_all(d, w, ws, M, L, Bt, st));
  p.in = x;
  p.out = y;
  p.bias2 = bvec;
  p.prof = g_prof;
  const int grid = grid_for(nbatch * p.tiles_per_b, sm);
  return d.parts == 3 ? run_chain3_p<3>(p, grid, st) : run_chain3_p<2>(p, grid, st);
}

int dl_chain_bwd_f32(const float* x, const float* dy, float* dx, float* dW, float* db, const float* M, int m_per_shell,
                     const float* L, const float* Bt, const float* P, const float* beta, void* workspace,
                     int64_t nbatch, int64_t s_in, int64_t s_out, int64_t K, int64_t n, int64_t r_in, int64_t r_out,
                     int64_t n_out, int64_t nvox, void* stream) {
  using namespace dl::tc;
  dl::begin_call();
  int sm = 0;
  DL_TRY(dl::device_check(&sm));
  DL_REQUIRE(dy && M && Bt && workspace, "chain_bwd: null pointer");
  DL_REQUIRE(!dx || L, "chain_bwd: dx needs L");
  DL_REQUIRE(!(dW || db) || (x && P && beta), "chain_bwd: weight grad needs x, P, beta");
  Dims d = make_dims(nbatch, s_in, s_out, n, r_in, r_out, n_out, nvox, m_per_shell);
  WsLayout w = ws_layout(d, kMaxParts);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  cudaStream_t st = dl::as_stream(stream);
  const int64_t ntiles = nbatch * ((nvox + kTileV - 1) / kTileV);
  DL_TRY(pack_all(d, w, ws, M, dx ? L : nullptr, Bt, st));
  if (dx && ntiles > 0) {
    Chain3 p = chain3_params(d, w, ws, true);
    DL_REQUIRE(plan_chain3(p, d.parts), "chain_bwd: channel counts exceed the fused kernel's plan");
    p.in = dy;
    p.out = dx;
    p.bias2 = nullptr;
    const int grid = grid_for(ntiles, sm);
    DL_TRY(d.parts == 3 ? run_chain3_p<3>(p, grid, st) : run_chain3_p<2>(p, grid, st));
  }
  if (dW || db) {
    GramP g = gram_params(d, w, ws);
    DL_REQUIRE(plan_gram(g, d.parts), "chain_bwd: channel counts exceed the fused Gram plan");
    const int GR = g.GR, GC = g.GC;
    int nparts = 0;
    if (ntiles > 0) {
      g.x = x;
      g.dy = dy;
      g.beta = beta;
      nparts = grid_for(ntiles, sm < kMaxParts ? sm : kMaxParts);
      DL_TRY(d.parts == 3 ? run_gram_p<3>(g, nparts, st) : run_gram_p<2>(g, nparts, st));
    }
    float* partials = reinterpret_cast<float*>(ws + w.parts);
    double* G = reinterpret_cast<double*>(ws + w.G);
    if (nparts == 0) {
      DL_CUDA(cudaMemsetAsync(G, 0, (size_t)GR * GC * 8, st));
    } else {
      gram_reduce_k<<<(GR * GC + 255) / 256, 256, 0, st>>>(partials, G, nparts, GR * GC);
      DL_TRY(dl::after_launch("gram_reduce"));
    }
    const float* dbparts = partials + (size_t)nparts * GR * GC;
    gram_finalize_k<<<(unsigned)(s_out * s_in * K + s_out), 256, 0, st>>>(G, dbparts, nparts, P, dW, db, (int)s_out,
                                                                          (int)s_in, (int)K, (int)r_out, (int)r_in,
                                                                          d.RPo, d.RPi);
    DL_TRY(dl::after_launch("gram_finalize"));
  }
  return DL_OK;
}

}  // extern "C"
