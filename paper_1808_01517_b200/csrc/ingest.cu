// Raw-acquisition ingest: b0 normalisation fused with the layout change to the 5-D channel-major contract.
//
// Reference (/root/reference/pkg/src/sphdwi/): fitting.normalize_b0 (fitting.py:253-342) over the 4-D
// acquisition dwio.read_nifti returns (dwio.py:312-391: X, Y, Z, volume, scl_slope / scl_inter applied).
//   mean_b0 = mean of the b0 volumes per voxel (float64), eps = 1e-6 * max(mean_b0),
//   excluded = mean_b0 <= eps (-> 0), out[k] = raw[..., sel[k]] / mean_b0 (sel = the shell volumes, shell-blocked)
// The raw volume is read in its stored layout (NIfTI keeps x fastest, volumes slowest; an in-memory
// (X, Y, Z, V) array keeps the volume fastest) and in its stored integer / float type: the copy to the device
// is the file's own bytes, and one pass writes the normalised fp32 (channels, X, Y, Z) volume.
// All arithmetic is float64 and rounds once to fp32, so results equal the reference's rounded to fp32.
//
// Kernels (HBM-bound streams):
//   b0_mean_k   per-voxel b0 mean in float64, per-block maxima            reads n_b0 volumes
//   b0_eps_k    fixed-order max of the block maxima -> eps                  (one block)
//   ingest_x_k  32 x 32 shared-memory tile transpose for x-fastest storage (NIfTI): read along x, write along z
//               of (channel, X, Y, Z), 48 channels per block sharing the b0 means held in registers; ingest_k: the same
//               over (channel, z) tiles for other layouts.  Divide / zero excluded voxels.  reads n_sel volumes
//   mask_k      excluded mask (X, Y, Z) bytes
#include <float.h>

#include "common.cuh"

namespace dl {
namespace {

constexpr int kMeanBlocks = 1024;
constexpr int kT = 32;   // transpose tile

template <typename T>
__device__ __forceinline__ double load_val(const void* raw, int64_t off, double slope, double inter) {
  const double v = (double)reinterpret_cast<const T*>(raw)[off];
  return slope != 0.0 ? v * slope + inter : v;
}

struct Geo {
  int64_t X, Y, Z;          // spatial extents
  int64_t sx, sy, sz, sv;   // element strides of the stored layout
  int64_t e0, e1;           // spatial extents in increasing-stride order (fast, middle); the slow one is implied
  int d0, d1, d2;           // which spatial axis (0 x, 1 y, 2 z) is fast / middle / slow in the stored layout
};

__device__ __forceinline__ void axes_of(const Geo& g, int64_t t, int64_t (&c)[3]) {
  const int64_t a = t % g.e0, r = t / g.e0;
  c[g.d0] = a;
  c[g.d1] = r % g.e1;
  c[g.d2] = r / g.e1;
}
// inverse of axes_of: the stored-order walk index of voxel (x, y, z); the b0 means are kept in this order
__device__ __forceinline__ int64_t walk_of(const Geo& g, int64_t x, int64_t y, int64_t z) {
  const int64_t c[3] = {x, y, z};
  return c[g.d0] + g.e0 * (c[g.d1] + g.e1 * c[g.d2]);
}

// per-voxel mean of the b0 volumes (threads walk voxels in stored order, so b0 reads coalesce when a spatial
// axis is the fastest); writes mean[(x * Y + y) * Z + z] and per-block maxima
template <typename T>
__global__ void b0_mean_k(const void* __restrict__ raw, Geo g, double slope, double inter,
                          const int64_t* __restrict__ b0, int n_b0, double* __restrict__ mean,
                          double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t nvox = g.X * g.Y * g.Z;
  double m = -DBL_MAX;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nvox; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    axes_of(g, t, c);
    const int64_t off = c[0] * g.sx + c[1] * g.sy + c[2] * g.sz;
    double s = 0.0;
    int i = 0;
    for (; i + 8 <= n_b0; i += 8) {   // eight loads in flight, summed in index order
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = load_val<T>(raw, off + __ldg(b0 + i + j) * g.sv, slope, inter);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; i < n_b0; ++i) s += load_val<T>(raw, off + __ldg(b0 + i) * g.sv, slope, inter);
    const double mu = s / (double)n_b0;
    mean[t] = mu;              // stored (walk) order: coalesced
    mean[nvox + t] = 1.0 / mu; // reciprocal for the corrected-product quotient
    m = fmax(m, mu);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -DBL_MAX;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) part[blockIdx.x] = m;
  }
}

__global__ void b0_eps_k(const double* __restrict__ part, int nparts, int64_t nvox, double* __restrict__ eps) {
  double m = -DBL_MAX;   // max is order-independent: any reduction order gives the same eps
  for (int i = threadIdx.x; i < nparts; i += 32) m = fmax(m, part[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) *eps = nvox > 0 ? 1e-6 * m : 0.0;
}

// exclusion mask in (X, Y, Z) order (the x-fastest path writes it from ingest_x_k instead)
__global__ void mask_k(Geo g, const double* __restrict__ mean, const double* __restrict__ eps,
                       uint8_t* __restrict__ excluded) {
  const double e = *eps;
  const int64_t nvox = g.X * g.Y * g.Z;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvox; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % g.Z, r = i / g.Z;
    excluded[i] = mean[walk_of(g, r / g.Y, r % g.Y, z)] <= e ? 1 : 0;
  }
}

// Per-voxel normalisation factors for the chain's raw-input path (in_role_raw), in stored (walk) order:
// x = raw * a + b with a = slope / mean_b0, b = inter / mean_b0 (slope 0: no scaling, a = 1 / mean_b0, b = 0),
// both 0 for excluded voxels (mean_b0 <= eps); excluded (optional) in walk order.
__global__ void voxel_scale_k(int64_t nvox, const double* __restrict__ mean, const double* __restrict__ eps,
                              double slope, double inter, float* __restrict__ a, float* __restrict__ b,
                              uint8_t* __restrict__ excluded) {
  const double e = *eps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvox; i += (int64_t)gridDim.x * blockDim.x) {
    const double mu = mean[i];
    const bool ex = mu <= e;
    a[i] = ex ? 0.f : (float)((slope != 0.0 ? slope : 1.0) / mu);
    b[i] = ex ? 0.f : (float)((slope != 0.0 ? inter : 0.0) / mu);
    if (excluded) excluded[i] = ex ? 1 : 0;
  }
}

// x-fastest stored layout (a NIfTI file's bytes): tile over (x, z) for one y and kKB consecutive output
// channels; the tile's float64 b0 means are staged in shared memory once and reused for every channel.
// Grid: (ceil(X / 32), ceil(Z / 32), Y * ceil(n_sel / kKB)); block 32 x 8.
constexpr int kKB = 48;
#ifndef DL_INGEST_PRE
#define DL_INGEST_PRE 2
#endif
constexpr int kPre = DL_INGEST_PRE;   // channels of raw values a thread keeps in flight
template <typename T>
__global__ void __launch_bounds__(256) ingest_x_k(const void* __restrict__ raw, Geo g, double slope, double inter,
                                                  const int64_t* __restrict__ sel, int n_sel,
                                                  const double* __restrict__ mean, const double* __restrict__ eps,
                                                  float* __restrict__ out, uint8_t* __restrict__ excluded, int64_t zoff) {
  __shared__ T tile[2][kT][kT + 1];      // raw values in their stored type, double-buffered
  __shared__ double mt[2][kT][kT + 1];   // b0 means / reciprocals of the tile, [z][x] as read
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x0 = blockIdx.x * kT, z0 = blockIdx.y * kT;
  const int64_t bz = (int64_t)blockIdx.z + zoff;   // launched in grid.z chunks of <= 65535
  const int64_t y = bz % g.Y, k0 = (bz / g.Y) * kKB;
  const int64_t nvox = g.X * g.Y * g.Z;
  const double e = *eps;
  const int X = (int)g.X, Z = (int)g.Z, sz = (int)g.sz;   // the host checks X*Y*Z < 2^31
  // means are stored x-fastest like the input: read them along x, transpose through shared memory
#pragma unroll
  for (int q = 0; q < kT / 8; ++q) {
    const int x = x0 + tx, z = z0 + ty + 8 * q;
    const bool in = x < X && z < Z;
    const int64_t w = walk_of(g, x, y, z);
    mt[0][ty + 8 * q][tx] = in ? mean[w] : 1.0;
    mt[1][ty + 8 * q][tx] = in ? mean[nvox + w] : 1.0;
  }
  __syncthreads();
  // this thread's output voxels (x = x0 + j, z = z0 + tx): b0 mean and reciprocal held in registers
  double mu[kT / 8], rc[kT / 8];
  int vo[kT / 8];
#pragma unroll
  for (int q = 0; q < kT / 8; ++q) {
    const int x = x0 + ty + 8 * q, z = z0 + tx;
    const bool in = x < X && z < Z;
    vo[q] = in ? (int)(((int64_t)x * g.Y + y) * Z + z) : -1;
    mu[q] = mt[0][tx][ty + 8 * q];
    rc[q] = mt[1][tx][ty + 8 * q];
    if (in && excluded && k0 == 0) excluded[vo[q]] = mu[q] <= e ? 1 : 0;
  }
  const T* base = reinterpret_cast<const T*>(raw) + y * g.sy;
  const int64_t k1 = k0 + kKB < n_sel ? k0 + kKB : n_sel;
  // Raw values are loaded kPre channels ahead (registers) and transposed through a double-buffered
  // shared-memory tile in their stored type, so a block keeps kPre + 1 channels' reads in flight and meets
  // one barrier per channel.
  T pf[kPre][kT / 8];   // channels k + 1 ... k + kPre, oldest first
  auto load = [&](int64_t k, T (&dst)[kT / 8]) {
    const T* src = base + __ldg(sel + k) * g.sv;
#pragma unroll
    for (int q = 0; q < kT / 8; ++q) {   // read along x
      const int x = x0 + tx, z = z0 + ty + 8 * q;
      dst[q] = (x < X && z < Z) ? src[x + z * sz] : (T)0;
    }
  };
#pragma unroll
  for (int i = 0; i < kPre; ++i)
    if (k0 + i < k1) load(k0 + i, pf[i]);
  for (int64_t k = k0; k < k1; ++k) {
    const int buf = (int)((k - k0) & 1);
#pragma unroll
    for (int q = 0; q < kT / 8; ++q) {
      tile[buf][ty + 8 * q][tx] = pf[0][q];
#pragma unroll
      for (int i = 0; i + 1 < kPre; ++i) pf[i][q] = pf[i + 1][q];
    }
    if (k + kPre < k1) load(k + kPre, pf[kPre - 1]);
    __syncthreads();
    float* ok = out + k * nvox;
#pragma unroll
    for (int q = 0; q < kT / 8; ++q) {   // out, written along z: v / mu as a corrected product
      if (vo[q] < 0) continue;
      double v = (double)tile[buf][tx][ty + 8 * q];
      if (slope != 0.0) v = fma(v, slope, inter);
      double r = v * rc[q];
      r = fma(fma(-r, mu[q], v), rc[q], r);
      ok[vo[q]] = mu[q] <= e ? 0.f : (float)r;
    }
  }
}

// Other stored layouts (e.g. an in-memory (X, Y, Z, V) array, volume fastest): tile over (k, z) for one (x, y).
// Grid: (ceil(n_sel / 32), ceil(Z / 32), Y * X); block 32 x 8.
template <typename T>
__global__ void __launch_bounds__(256) ingest_k(const void* __restrict__ raw, Geo g, double slope, double inter,
                                                const int64_t* __restrict__ sel, int n_sel,
                                                const double* __restrict__ mean, const double* __restrict__ eps,
                                                float* __restrict__ out, int xfast, int64_t zoff) {
  __shared__ double tile[kT][kT + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t a0 = (int64_t)blockIdx.x * kT, z0 = (int64_t)blockIdx.y * kT;
  const int64_t bz = (int64_t)blockIdx.z + zoff;   // launched in grid.z chunks of <= 65535
  const int64_t y = bz % g.Y, w = bz / g.Y;   // w = k (xfast) or x (otherwise)
  const int64_t A = xfast ? g.X : n_sel;
  const int64_t nvox = g.X * g.Y * g.Z;
  // load: thread tx walks a (the stored-fast axis), rows j = z
  for (int j = ty; j < kT; j += blockDim.y) {
    const int64_t a = a0 + tx, z = z0 + j;
    double v = 0.0;
    if (a < A && z < g.Z) {
      const int64_t x = xfast ? a : w, k = xfast ? w : a;
      v = load_val<T>(raw, x * g.sx + y * g.sy + z * g.sz + __ldg(sel + k) * g.sv, slope, inter);
    }
    tile[j][tx] = v;
  }
  __syncthreads();
  const double e = *eps;
  // store: thread tx walks z, rows j = a
  for (int j = ty; j < kT; j += blockDim.y) {
    const int64_t a = a0 + j, z = z0 + tx;
    if (a < A && z < g.Z) {
      const int64_t x = xfast ? a : w, k = xfast ? w : a;
      const int64_t vox = (x * g.Y + y) * g.Z + z;
      const double mu = mean[walk_of(g, x, y, z)];
      out[k * nvox + vox] = mu <= e ? 0.f : (float)(tile[tx][j] / mu);
    }
  }
}

constexpr int64_t kMaxGridZ = 65535;

template <typename T>
int launch_all(const void* raw, const Geo& g, double slope, double inter, const int64_t* b0, int n_b0,
               const int64_t* sel, int n_sel, float* out, uint8_t* excluded, double* mean, double* part,
               double* eps, cudaStream_t st) {
  const int64_t nvox = g.X * g.Y * g.Z;
  const int nb = (int)(ceil_div<int64_t>(nvox, 256) < kMeanBlocks ? ceil_div<int64_t>(nvox, 256) : kMeanBlocks);
  b0_mean_k<T><<<nb, 256, 0, st>>>(raw, g, slope, inter, b0, n_b0, mean, part);
  DL_TRY(after_launch("b0_mean_k"));
  b0_eps_k<<<1, 32, 0, st>>>(part, nb, nvox, eps);
  DL_TRY(after_launch("b0_eps_k"));
  if (n_sel > 0 && g.sx == 1) {
    const int64_t nz = g.Y * ceil_div<int64_t>(n_sel, kKB);
    for (int64_t z0 = 0; z0 < nz; z0 += kMaxGridZ) {   // grid.z is capped at 65535
      const dim3 grid((unsigned)ceil_div<int64_t>(g.X, kT), (unsigned)ceil_div<int64_t>(g.Z, kT),
                      (unsigned)(nz - z0 < kMaxGridZ ? nz - z0 : kMaxGridZ));
      ingest_x_k<T><<<grid, dim3(kT, 8), 0, st>>>(raw, g, slope, inter, sel, n_sel, mean, eps, out, excluded, z0);
      DL_TRY(after_launch("ingest_x_k"));
    }
    if (excluded) return DL_OK;   // written by ingest_x_k
  } else if (n_sel > 0) {
    const int64_t nz = g.Y * g.X;
    for (int64_t z0 = 0; z0 < nz; z0 += kMaxGridZ) {   // grid.z is capped at 65535 (e.g. 256 x 256 in-memory volumes)
      const dim3 grid((unsigned)ceil_div<int64_t>(n_sel, kT), (unsigned)ceil_div<int64_t>(g.Z, kT),
                      (unsigned)(nz - z0 < kMaxGridZ ? nz - z0 : kMaxGridZ));
      ingest_k<T><<<grid, dim3(kT, 8), 0, st>>>(raw, g, slope, inter, sel, n_sel, mean, eps, out, 0, z0);
      DL_TRY(after_launch("ingest_k"));
    }
  }
  if (excluded) {
    const int mb = (int)(ceil_div<int64_t>(nvox, 256) < 4096 ? ceil_div<int64_t>(nvox, 256) : 4096);
    mask_k<<<mb, 256, 0, st>>>(g, mean, eps, excluded);
    DL_TRY(after_launch("mask_k"));
  }
  return DL_OK;
}

template <typename T>
int launch_scale(const void* raw, const Geo& g, double slope, double inter, const int64_t* b0, int n_b0, float* va,
                 float* vb, uint8_t* excluded, double* mean, double* part, double* eps, cudaStream_t st) {
  const int64_t nvox = g.X * g.Y * g.Z;
  const int nb = (int)(ceil_div<int64_t>(nvox, 256) < kMeanBlocks ? ceil_div<int64_t>(nvox, 256) : kMeanBlocks);
  b0_mean_k<T><<<nb, 256, 0, st>>>(raw, g, slope, inter, b0, n_b0, mean, part);
  DL_TRY(after_launch("b0_mean_k"));
  b0_eps_k<<<1, 32, 0, st>>>(part, nb, nvox, eps);
  DL_TRY(after_launch("b0_eps_k"));
  const int mb = (int)(ceil_div<int64_t>(nvox, 256) < 4096 ? ceil_div<int64_t>(nvox, 256) : 4096);
  voxel_scale_k<<<mb, 256, 0, st>>>(nvox, mean, eps, slope, inter, va, vb, excluded);
  return after_launch("voxel_scale_k");
}

}  // namespace
}  // namespace dl

extern "C" {

int dl_b0_voxel_scale_f32(const void* raw, int nifti_dtype, int64_t X, int64_t Y, int64_t Z, int64_t sx, int64_t sy,
                          int64_t sz, int64_t sv, double slope, double inter, const int64_t* b0_idx, int64_t n_b0,
                          float* vox_a, float* vox_b, uint8_t* excluded, void* workspace, void* stream) {
  using namespace dl;
  begin_call();
  DL_TRY(device_check(nullptr));
  DL_REQUIRE(X >= 1 && Y >= 1 && Z >= 1 && n_b0 >= 1 && n_b0 < (1 << 30) && X * Y * Z < 2147483647LL,
             "b0_voxel_scale: bad sizes (X %lld, Y %lld, Z %lld, b0 %lld)", (long long)X, (long long)Y, (long long)Z,
             (long long)n_b0);
  DL_REQUIRE(raw && b0_idx && vox_a && vox_b && workspace, "b0_voxel_scale: null pointer");
  DL_REQUIRE(sx == 1 && sy == X && sz == X * Y, "b0_voxel_scale: needs the x-fastest dense volume layout (NIfTI)");
  Geo g;
  g.X = X; g.Y = Y; g.Z = Z; g.sx = sx; g.sy = sy; g.sz = sz; g.sv = sv;
  g.d0 = 0; g.d1 = 1; g.d2 = 2; g.e0 = X; g.e1 = Y;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  double* mean = reinterpret_cast<double*>(ws);
  double* part = mean + 2 * X * Y * Z;
  double* eps = part + kMeanBlocks;
  cudaStream_t st = as_stream(stream);
  switch (nifti_dtype) {
    case 2: return launch_scale<uint8_t>(raw, g, slope, inter, b0_idx, (int)n_b0, vox_a, vox_b, excluded, mean, part, eps, st);
    case 4: return launch_scale<int16_t>(raw, g, slope, inter, b0_idx, (int)n_b0, vox_a, vox_b, excluded, mean, part, eps, st);
    case 8: return launch_scale<int32_t>(raw, g, slope, inter, b0_idx, (int)n_b0, vox_a, vox_b, excluded, mean, part, eps, st);
    case 16: return launch_scale<float>(raw, g, slope, inter, b0_idx, (int)n_b0, vox_a, vox_b, excluded, mean, part, eps, st);
    case 64: return launch_scale<double>(raw, g, slope, inter, b0_idx, (int)n_b0, vox_a, vox_b, excluded, mean, part, eps, st);
    default: return fail(DL_EINVAL, "b0_voxel_scale: unsupported NIfTI datatype code %d", nifti_dtype);
  }
}

size_t dl_normalize_b0_workspace_bytes(int64_t X, int64_t Y, int64_t Z) {
  const int64_t nvox = X * Y * Z;
  return (size_t)(nvox > 0 ? nvox : 0) * 16 + (size_t)(dl::kMeanBlocks + 2) * 8 + 256;
}

int dl_normalize_b0_f32(const void* raw, int nifti_dtype, int64_t X, int64_t Y, int64_t Z, int64_t sx, int64_t sy,
                        int64_t sz, int64_t sv, double slope, double inter, const int64_t* b0_idx, int64_t n_b0,
                        const int64_t* sel, int64_t n_sel, float* out, uint8_t* excluded, void* workspace,
                        void* stream) {
  using namespace dl;
  begin_call();
  DL_TRY(device_check(nullptr));
  DL_REQUIRE(X >= 1 && Y >= 1 && Z >= 1 && n_b0 >= 1 && n_sel >= 0 && n_b0 < (1 << 30) && n_sel < (1 << 30),
             "normalize_b0: bad sizes (X %lld, Y %lld, Z %lld, b0 %lld, selected %lld)", (long long)X, (long long)Y,
             (long long)Z, (long long)n_b0, (long long)n_sel);
  DL_REQUIRE(raw && b0_idx && workspace && (n_sel == 0 || (sel && out)), "normalize_b0: null pointer");
  DL_REQUIRE(Y * (sx == 1 ? (n_sel + 47) / 48 : X) < 2147483647LL && X * Y * Z < 2147483647LL &&
                 (sx != 1 || (sz < 2147483647LL && sz * Z < 2147483647LL)),
             "normalize_b0: volume too large for 32-bit voxel indexing");
  Geo g;
  g.X = X; g.Y = Y; g.Z = Z; g.sx = sx; g.sy = sy; g.sz = sz; g.sv = sv;
  // spatial axes in increasing-stride order (stable: x, y, z on ties)
  int ord[3] = {0, 1, 2};
  const int64_t s[3] = {sx < 0 ? -sx : sx, sy < 0 ? -sy : sy, sz < 0 ? -sz : sz};
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && s[ord[j]] < s[ord[j - 1]]; --j) {
      const int t = ord[j]; ord[j] = ord[j - 1]; ord[j - 1] = t;
    }
  const int64_t ext[3] = {X, Y, Z};
  g.d0 = ord[0]; g.d1 = ord[1]; g.d2 = ord[2];
  g.e0 = ext[ord[0]]; g.e1 = ext[ord[1]];
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  double* mean = reinterpret_cast<double*>(ws);
  double* part = mean + 2 * X * Y * Z;   // mean | reciprocal | block maxima | eps
  double* eps = part + kMeanBlocks;
  cudaStream_t st = as_stream(stream);
  switch (nifti_dtype) {
    case 2: return launch_all<uint8_t>(raw, g, slope, inter, b0_idx, (int)n_b0, sel, (int)n_sel, out, excluded, mean, part, eps, st);
    case 4: return launch_all<int16_t>(raw, g, slope, inter, b0_idx, (int)n_b0, sel, (int)n_sel, out, excluded, mean, part, eps, st);
    case 8: return launch_all<int32_t>(raw, g, slope, inter, b0_idx, (int)n_b0, sel, (int)n_sel, out, excluded, mean, part, eps, st);
    case 16: return launch_all<float>(raw, g, slope, inter, b0_idx, (int)n_b0, sel, (int)n_sel, out, excluded, mean, part, eps, st);
    case 64: return launch_all<double>(raw, g, slope, inter, b0_idx, (int)n_b0, sel, (int)n_sel, out, excluded, mean, part, eps, st);
    default: return fail(DL_EINVAL, "normalize_b0: unsupported NIfTI datatype code %d", nifti_dtype);
  }
}

}  // extern "C"
