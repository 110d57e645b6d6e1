/*
 * delimit.h -- C ABI of libdelimit_sm100a.so, the B200 (sm_100a) kernels behind
 * the Signal2SH -> LocalSphericalConvolution -> SH2Signal path.
 *
 * Every entry point takes raw DEVICE pointers to float32 buffers, int64 sizes
 * and a cudaStream_t (passed as void*), enqueues work on that stream only and
 * returns 0 on success or a DL_E* code; dl_last_error() then holds a message.
 * The library never allocates device memory: callers own outputs and
 * workspaces (sizes from the *_workspace_bytes queries).  There is no CPU
 * fallback: with no usable sm_100a device every compute entry returns
 * DL_ENODEVICE.
 *
 * Volume layout (the reference's 5-D contract, fitting.py:33-89):
 *   (subjects, shells * C, X, Y, Z) C-contiguous; shell s owns channels
 *   [s*C, (s+1)*C); nvox = X*Y*Z voxels are contiguous per channel.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/sphdwi/):
 *   dl_chan_contract_f32    <- fitting._apply_channel_matrix  fitting.py:155-188
 *                              (and thus signal_to_sh fitting.py:206-236,
 *                               sh_to_signal fitting.py:239-250, the LSC refit lsc.py:197)
 *   dl_lsc_build_operator_f32, dl_lsc_forward via dl_chan_contract_f32
 *                           <- _kernels.lsc_combine _kernels.py:187-206 + refit lsc.py:194-198
 *   dl_lsc_wgrad_f32        <- (no reference counterpart: backward is out of the
 *                               reference's scope)
 *   dl_chain_fwd_f32 / dl_chain_bwd_f32
 *                           <- signal_to_sh -> lsc_forward -> sh_to_signal as the
 *                              CLI chains them (cli.py:159-245), fused.
 */
#ifndef DELIMIT_H_
#define DELIMIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DL_OK = 0,
  DL_EINVAL = 1,       /* bad argument (shape, null pointer, alignment) */
  DL_ECUDA = 2,        /* CUDA runtime / launch error */
  DL_ENODEVICE = 3,    /* no sm_100a device available */
};

/* ABI version (major*100 + minor). */
int dl_abi_version(void);
/* Message for the last non-zero status returned on this host thread. */
const char* dl_last_error(void);
/* 1 if the current CUDA device is sm_100 (B200), else 0 (sets dl_last_error). */
int dl_device_supported(void);

/*
 * Per-voxel channel contraction with optional bias:
 *   out[b, g*c_out + i, v] = bias_g[i] + sum_j W_g[i, j] * in[b, g*c_in + j, v]
 * W is row-major (c_out, c_in); with w_per_group != 0 W holds `groups`
 * consecutive matrices (and bias `groups` consecutive vectors), else one
 * matrix is shared by every group.  bias may be NULL.  in_bs / out_bs are the
 * subject strides in elements.  in and out must not alias.
 * Replaces fitting._apply_channel_matrix (fitting.py:155-188); groups = shells.
 */
int dl_chan_contract_f32(const float* in, float* out, const float* W, const float* bias,
                         int64_t nbatch, int64_t groups, int64_t c_in, int64_t c_out,
                         int64_t nvox, int64_t in_bs, int64_t out_bs, int w_per_group,
                         void* stream);

/*
 * Folded LSC operator from the kernel parameters:
 *   L[o*r_out + r, s*r_in + t]  = sum_k w[o, s, k] * P[k, r, t]
 *   Lt = L^T,  bvec[o*r_out + r] = bias[o] * beta[r]
 * P_k = refit . resample[k::K] (K, r_out, r_in), beta = refit . 1 (r_out).
 * w is (s_out, s_in, K) (the .sconv.weight (s_out, s_in, 1, K) memory).
 * L, Lt: (s_out*r_out) x (s_in*r_in) resp. transposed; bvec: s_out*r_out.
 * Equivalent to lsc_combine + refit (_kernels.py:91-104, lsc.py:197) in exact arithmetic.
 */
int dl_lsc_build_operator_f32(const float* P, const float* beta, const float* w, const float* bias,
                              float* L, float* Lt, float* bvec, int64_t s_out, int64_t s_in,
                              int64_t K, int64_t r_out, int64_t r_in, void* stream);

/*
 * LSC weight/bias gradient.  With g = dL/dc_out (nbatch, s_out*r_out, nvox)
 * and c = c_in (nbatch, s_in*r_in, nvox):
 *   G      = sum_{b,v} g[b,:,v] c[b,:,v]^T          ((s_out r_out) x (s_in r_in))
 *   dW[o,s,k] = <P_k, G_{o,s}>_F,   db[o] = beta . sum_{b,v} g[b, o*r_out:(o+1)*r_out, v]
 * Deterministic (fixed partition + fixed-order float64 reduction).
 * workspace: dl_lsc_wgrad_workspace_bytes() bytes of device memory.
 */
size_t dl_lsc_wgrad_workspace_bytes(int64_t s_out, int64_t s_in, int64_t r_out, int64_t r_in);
int dl_lsc_wgrad_f32(const float* g, const float* c, const float* P, const float* beta,
                     float* dW, float* db, void* workspace, int64_t nbatch, int64_t s_out,
                     int64_t s_in, int64_t K, int64_t r_out, int64_t r_in, int64_t nvox,
                     int64_t g_bs, int64_t c_bs, void* stream);

/*
 * Fused chain Signal2SH -> LSC -> SH2Signal on the 5th-generation tensor cores (tcgen05).
 *   M:  r_in x n fit matrix, one per input shell (m_per_shell) or shared;
 *   L:  (s_out*r_out) x (s_in*r_in) folded LSC operator, bvec its bias response
 *       (dl_lsc_build_operator_f32); Bt: n_out x r_out SH basis at the output directions.
 * Forward: x (nbatch, s_in*n, nvox) -> y (nbatch, s_out*n_out, nvox) in one kernel.  If c_mid
 * is not NULL the Signal2SH coefficients c = M x are also written there, as the backward's Gram
 * operand: an opaque buffer of dl_chain_mid_bytes(nbatch, s_in, r_in, nvox) bytes (16-byte aligned)
 * holding c's first two bf16 split terms per element (rows padded per shell to 16, voxels to 64).
 * Every product is an fp32-accurate split product with fp32 accumulation.  Default: each fp32 operand
 * as two fp16 terms, activations scaled by a power of two (delayed scaling), then a 3-term bf16 pass
 * that checks the recorded ranges and recomputes everything only when they were out of bounds.
 * DELIMIT_SPLIT_TERMS=3 / 2 forces the 3-term / 2-term bf16 kernels alone.
 * state: dl_chain_state_bytes() bytes of zero-initialised device memory the caller keeps between
 * calls, one per direction and stream (the scale history); NULL runs the 3-term bf16 kernel only.
 * Backward: dy -> dx with the adjoint chain kernel, which also writes g = B'^T dy to g_mid
 * (dl_chain_mid_bytes(nbatch, s_out, r_out, nvox) bytes) when dW or db is requested; then the LSC
 * parameter gradient dW (s_out, s_in, K), db (s_out) from a streaming Gram kernel over
 * (g_mid, c_mid) plus a float64 finalize.  dW / db may be NULL (then c_mid, g_mid, P, beta may be
 * NULL).  dx may be NULL when dW / db are requested: the adjoint kernel then skips the dx stores (a g-only
 * pass for training steps whose input needs no gradient).
 * workspace: dl_chain_workspace_bytes() bytes.  dl_chain_supported() says whether the
 * channel counts fit the kernels' TMEM/shared-memory plan (3 shells x order 8 x 90 dirs do).
 */
int dl_chain_supported(int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                       int m_per_shell);
int dl_chain_split_terms(void);
size_t dl_chain_mid_bytes(int64_t nbatch, int64_t shells, int64_t r, int64_t nvox);
size_t dl_chain_workspace_bytes(int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in,
                                int64_t r_out, int64_t n_out, int64_t nvox);
size_t dl_chain_state_bytes(void);
/* The fused Signal2SH -> LSC -> SH2Signal forward read straight from a raw acquisition: the b0 normalisation of
 * fitting.normalize_b0 (fitting.py:253-342) runs in the kernel's input role, x[c][v] = raw[sel[c]][v] * vox_a[v] +
 * vox_b[v], so the normalised volume never exists in memory.  raw: the acquisition's
 * volumes, `vstride` elements apart (even), int16 (raw_dtype 4) or float32 (16), voxels in stored order; sel
 * (device int32, s_in * n): the stored volume of every chain input channel (shell-blocked); vox_a / vox_b from
 * dl_b0_voxel_scale_f32.  y: (s_out * n_out, nvox) fp32 in the same stored voxel order.  state: as for
 * dl_chain_fwd_f32 (fp16 pass + bf16 check; NULL: the 3-term bf16 pass alone). */
int dl_chain_fwd_raw_f32(const void* raw, int raw_dtype, int64_t vstride, const int* sel, const float* vox_a,
                         const float* vox_b, float* y, const float* M, int m_per_shell, const float* L,
                         const float* bvec, const float* Bt, void* workspace, void* state, int64_t s_in,
                         int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox,
                         void* stream);
/* Per-voxel factors of the raw-input chain from the b0 volumes (fitting.py:253-342 in float64, rounded once):
 * vox_a = slope / mean_b0, vox_b = inter / mean_b0 (slope 0: no scaling), 0 where mean_b0 <= 1e-6 max(mean_b0);
 * excluded (optional) the mask; all in stored voxel order.  Needs the x-fastest NIfTI layout (sx = 1, sy = X,
 * sz = X Y); workspace: dl_normalize_b0_workspace_bytes(X, Y, Z). */
int dl_b0_voxel_scale_f32(const void* raw, int nifti_dtype, int64_t X, int64_t Y, int64_t Z, int64_t sx, int64_t sy,
                          int64_t sz, int64_t sv, double slope, double inter, const int64_t* b0_idx, int64_t n_b0,
                          float* vox_a, float* vox_b, uint8_t* excluded, void* workspace, void* stream);
/*
 * Forward fused with a mean-squared-error loss against `target` (same layout as y): writes
 * dy = 2 (y - target) / numel(y) instead of y, and loss[2] = mean((y - target)^2) (loss: 4 doubles of
 * device memory; [0], [1] are per-pass accumulators).  y itself is not stored.  Needs the chain3v/chain2h
 * plan (dl_chain_mse_supported).  dy then feeds dl_chain_bwd_f32 / dl_chain_bwd_gram_f64 directly.
 */
int dl_chain_fwd_mse_f32(const float* x, const float* target, float* dy, void* c_mid, const float* M,
                         int m_per_shell, const float* L, const float* bvec, const float* Bt, void* workspace,
                         void* state, double* loss, int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n,
                         int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox, void* stream);
int dl_chain_mse_supported(int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                           int m_per_shell);
int dl_chain_fwd_f32(const float* x, float* y, void* c_mid, const float* M, int m_per_shell, const float* L,
                     const float* bvec, const float* Bt, void* workspace, void* state, int64_t nbatch,
                     int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                     int64_t nvox, void* stream);
int dl_chain_bwd_f32(const void* c_mid, const float* dy, float* dx, float* dW, float* db, void* g_mid,
                     const float* M, int m_per_shell, const float* L, const float* Bt, const float* P,
                     const float* beta, void* workspace, void* state, int64_t nbatch, int64_t s_in,
                     int64_t s_out, int64_t K, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out,
                     int64_t nvox, void* stream);

/*
 * Raw-acquisition ingest: b0 normalisation fused with the change to the channel-major 5-D layout.
 * Replaces fitting.normalize_b0 (fitting.py:253-342) applied to dwio.read_nifti output (dwio.py:312-391).
 *   raw: device copy of the stored 4-D acquisition, element (x, y, z, v) at raw[x*sx + y*sy + z*sz + v*sv]
 *        (element strides: a NIfTI file's own bytes have sx = 1, sy = X, sz = X*Y, sv = X*Y*Z), of NIfTI
 *        datatype code 2 (u8), 4 (i16), 8 (i32), 16 (f32) or 64 (f64), native byte order;
 *        value = stored * slope + inter when slope != 0 (scl_slope / scl_inter).
 *   b0_idx: n_b0 volume indices; sel: n_sel volume indices in output channel order (shell blocks).
 *   out: (n_sel, X, Y, Z) fp32 = value / mean_b0, or 0 where mean_b0 <= 1e-6 * max(mean_b0);
 *   excluded (optional): (X, Y, Z) bytes, 1 where excluded.  float64 arithmetic, one rounding to fp32.
 *   workspace: dl_normalize_b0_workspace_bytes(X, Y, Z) bytes.  Index ranges are the caller's contract.
 */
size_t dl_normalize_b0_workspace_bytes(int64_t X, int64_t Y, int64_t Z);
int dl_normalize_b0_f32(const void* raw, int nifti_dtype, int64_t X, int64_t Y, int64_t Z, int64_t sx,
                        int64_t sy, int64_t sz, int64_t sv, double slope, double inter, const int64_t* b0_idx,
                        int64_t n_b0, const int64_t* sel, int64_t n_sel, float* out, uint8_t* excluded,
                        void* workspace, void* stream);

/*
 * Backward of a chain whose LSC is a product of several layers (L = L_n ... L_1, folded by the caller):
 * dx as dl_chain_bwd_f32, plus the float64 Gram G = sum_v g c^T of g = B'^T dy and c = M x (from c_mid),
 * rows s_out x 16-padded r_out, columns s_in x 16-padded r_in (dl_chain_gram_dims); column r_in (shell 0's
 * first padding row) holds sum_v g.  Per-layer dW / db follow from G by small products (SphericalChain).
 */
int dl_chain_bwd_gram_f64(const void* c_mid, const float* dy, float* dx, double* gram, void* g_mid, const float* M,
                          int m_per_shell, const float* L, const float* Bt, void* workspace, void* state,
                          int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in, int64_t r_out,
                          int64_t n_out, int64_t nvox, void* stream);
int dl_chain_gram_dims(int64_t s_in, int64_t s_out, int64_t r_in, int64_t r_out, int64_t* rows, int64_t* cols);

/* Number of kernel launches the last call on this host thread enqueued. */
int dl_last_launch_count(void);
/* Kernel launches enqueued by this library since it was loaded (all threads). */
int64_t dl_total_launch_count(void);

/* Fused Signal2SH -> SH2Signal round trip (fitting.py:206-250 composed; acceptance criterion 1): the chain kernels
 * with the identity as the LSC operator (built in the workspace) and a block-diagonal stage 2 (output shell s reads
 * only shell s's coefficients, which never reach memory).  Forward y[s] = B' M_s x[s]; backward dx[s] = M_s^T B'^T dy[s].
 * workspace: dl_round_trip_workspace_bytes; state as for dl_chain_fwd_f32 (one per direction). */
size_t dl_round_trip_workspace_bytes(int64_t nbatch, int64_t shells, int64_t n, int64_t r, int64_t n_out,
                                     int64_t nvox);
int dl_round_trip_fwd_f32(const float* x, float* y, const float* M, int m_per_shell, const float* Bt, void* workspace,
                          void* state, int64_t nbatch, int64_t shells, int64_t n, int64_t r, int64_t n_out,
                          int64_t nvox, void* stream);
int dl_round_trip_bwd_f32(const float* dy, float* dx, const float* M, int m_per_shell, const float* Bt,
                          void* workspace, void* state, int64_t nbatch, int64_t shells, int64_t n, int64_t r,
                          int64_t n_out, int64_t nvox, void* stream);

/* Small dense float64 products of the stacked-LSC path (csrc/dense.cu): C = alpha op(A) op(B) + beta C with
 * row-major A (m x k, or k x m when ta), B (k x n, or n x k when tb), C (m x n); and the LSC weight gradient of one
 * layer from its operator gradient, dW[o,s,k] = sum_{r,t} P[k,r,t] dL[(o,r),(s,t)] -- the folded-layer gradients
 * of ops.ChainStackFunction (SURVEY.md Appendix A applied per layer; the reference has no backward). */
int dl_gemm_f64(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, int ta, const double* B, int64_t ldb,
                int tb, double* C, int64_t ldc, double alpha, double beta, void* stream);
int dl_lsc_dw_from_dl_f64(const double* dL, const float* P, float* dW, int64_t s_out, int64_t s_in, int64_t K,
                          int64_t r_out, int64_t r_in, void* stream);

/* Kernel timer (measurement aid for bench.py; no reference counterpart): while armed, the fused chain kernel's
 * fp16-pass launches (slot 0 forward, 1 adjoint) and the LSC weight-gradient Gram launches (slot 2) stamp the
 * device's %globaltimer when their first CTA starts and when their last CTA ends, into a per-slot device ring
 * of 64 launches.  The stamps are kernel arguments' work, so they record the same way eagerly and inside
 * replayed CUDA graphs, and they time the kernel alone.  dl_ktimer_count: launches recorded so far in a slot.
 * dl_ktimer_read: duration in ms of the launch `back` places before the last one (0 = the last; back < 63).
 * Both synchronize the device. */
int dl_ktimer_arm(int on);
int64_t dl_ktimer_count(int slot);
int dl_ktimer_read(int slot, int back, float* ms);

/* Debug hook (not part of the stable ABI): record chain phase timestamps of CTA 0. */
void dl_debug_chain_prof(void* buf);

#ifdef __cplusplus
}
#endif

#endif /* DELIMIT_H_ */
