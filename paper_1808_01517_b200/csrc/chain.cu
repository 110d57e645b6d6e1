// Chain Signal2SH -> LSC -> SH2Signal, forward and backward.
//
// Reference: the in-memory layers the CLI chains (/root/reference/pkg/src/sphdwi/cli.py:159-245):
// fitting.signal_to_sh (fitting.py:206-236) -> lsc.lsc_forward (lsc.py:158-199) ->
// fitting.sh_to_signal (fitting.py:239-250).  Backward is new (SPEC.md:12 puts it out of
// the reference's scope): dx = M^T L^T B'^T dy, plus the LSC gradient.
//
// This version composes the K1 chan_contract and the LSC gradient kernels through a
// caller-provided workspace (c, u/g, dc intermediates in HBM).
#include "common.cuh"
#include "kernels.cuh"

namespace dl {
namespace {

struct ChainWs {
  float* c;   // nbatch x s_in r_in x nvox
  float* u;   // nbatch x s_out r_out x nvox   (u in forward, g in backward)
  float* dc;  // nbatch x s_in r_in x nvox
  void* wg;   // lsc_wgrad workspace
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

ChainWs carve(void* ws, int64_t nbatch, int64_t s_in, int64_t s_out, int64_t r_in, int64_t r_out,
              int64_t nvox) {
  char* p = reinterpret_cast<char*>(ws);
  ChainWs w;
  w.c = reinterpret_cast<float*>(p);
  p += align256((size_t)nbatch * s_in * r_in * nvox * sizeof(float));
  w.u = reinterpret_cast<float*>(p);
  p += align256((size_t)nbatch * s_out * r_out * nvox * sizeof(float));
  w.dc = reinterpret_cast<float*>(p);
  p += align256((size_t)nbatch * s_in * r_in * nvox * sizeof(float));
  w.wg = p;
  return w;
}

}  // namespace
}  // namespace dl

extern "C" {

size_t dl_chain_workspace_bytes(int64_t nbatch, int64_t s_in, int64_t s_out, int64_t n, int64_t r_in,
                                int64_t r_out, int64_t n_out, int64_t nvox) {
  (void)n;
  (void)n_out;
  return dl::align256((size_t)nbatch * s_in * r_in * nvox * sizeof(float)) * 2 +
         dl::align256((size_t)nbatch * s_out * r_out * nvox * sizeof(float)) +
         dl::lsc_wgrad_workspace_bytes(s_out, s_in, r_out, r_in);
}

int dl_chain_fwd_f32(const float* x, float* y, const float* M, int m_per_shell, const float* L,
                     const float* bvec, const float* Bt, void* workspace, int64_t nbatch, int64_t s_in,
                     int64_t s_out, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox,
                     void* stream) {
  dl::begin_call();
  DL_REQUIRE(x && y && M && L && Bt && workspace, "chain_fwd: null pointer");
  cudaStream_t st = dl::as_stream(stream);
  dl::ChainWs w = dl::carve(workspace, nbatch, s_in, s_out, r_in, r_out, nvox);
  DL_TRY(dl::chan_contract(x, w.c, M, nullptr, nbatch, s_in, n, r_in, nvox, s_in * n * nvox,
                           s_in * r_in * nvox, m_per_shell, st));
  DL_TRY(dl::chan_contract(w.c, w.u, L, bvec, nbatch, 1, s_in * r_in, s_out * r_out, nvox,
                           s_in * r_in * nvox, s_out * r_out * nvox, 0, st));
  return dl::chan_contract(w.u, y, Bt, nullptr, nbatch, s_out, r_out, n_out, nvox, s_out * r_out * nvox,
                           s_out * n_out * nvox, 0, st);
}

int dl_chain_bwd_f32(const float* x, const float* dy, float* dx, float* dW, float* db, const float* M,
                     const float* M_t, int m_per_shell, const float* Lt, const float* Bt_t, const float* P,
                     const float* beta, void* workspace, int64_t nbatch, int64_t s_in, int64_t s_out,
                     int64_t K, int64_t n, int64_t r_in, int64_t r_out, int64_t n_out, int64_t nvox,
                     void* stream) {
  dl::begin_call();
  DL_REQUIRE(dy && Bt_t && workspace, "chain_bwd: null pointer");
  DL_REQUIRE(!dx || (M_t && Lt), "chain_bwd: dx needs M_t and Lt");
  DL_REQUIRE(!(dW || db) || (x && M && P && beta), "chain_bwd: weight grad needs x, M, P, beta");
  cudaStream_t st = dl::as_stream(stream);
  dl::ChainWs w = dl::carve(workspace, nbatch, s_in, s_out, r_in, r_out, nvox);
  const int64_t cbs = s_in * r_in * nvox, gbs = s_out * r_out * nvox;
  // g = B'^T dy per output shell
  DL_TRY(dl::chan_contract(dy, w.u, Bt_t, nullptr, nbatch, s_out, n_out, r_out, nvox, s_out * n_out * nvox,
                           gbs, 0, st));
  if (dW || db) {
    DL_TRY(dl::chan_contract(x, w.c, M, nullptr, nbatch, s_in, n, r_in, nvox, s_in * n * nvox, cbs,
                             m_per_shell, st));
    DL_TRY(dl::lsc_wgrad(w.u, w.c, P, beta, dW, db, w.wg, nbatch, s_out, s_in, K, r_out, r_in, nvox, gbs,
                         cbs, st));
  }
  if (dx) {
    DL_TRY(dl::chan_contract(w.u, w.dc, Lt, nullptr, nbatch, 1, s_out * r_out, s_in * r_in, nvox, gbs, cbs,
                             0, st));
    DL_TRY(dl::chan_contract(w.dc, dx, M_t, nullptr, nbatch, s_in, r_in, n, nvox, cbs, s_in * n * nvox,
                             m_per_shell, st));
  }
  return DL_OK;
}

}  // extern "C"
