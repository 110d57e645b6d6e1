// Internal launchers shared between the C-ABI entry points (no status reset,
// no launch-counter reset: callers own that).
#pragma once

#include "common.cuh"

namespace dl {

int chan_contract(const float* in, float* out, const float* W, const float* bias, int64_t nbatch,
                  int64_t groups, int64_t c_in, int64_t c_out, int64_t nvox, int64_t in_bs,
                  int64_t out_bs, int w_per_group, cudaStream_t st);

int lsc_build_operator(const float* P, const float* beta, const float* w, const float* bias, float* L,
                       float* Lt, float* bvec, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
                       int64_t r_in, cudaStream_t st);

size_t lsc_wgrad_workspace_bytes(int64_t s_out, int64_t s_in, int64_t r_out, int64_t r_in);

int lsc_wgrad(const float* g, const float* c, const float* P, const float* beta, float* dW, float* db,
              void* workspace, int64_t nbatch, int64_t s_out, int64_t s_in, int64_t K, int64_t r_out,
              int64_t r_in, int64_t nvox, int64_t g_bs, int64_t c_bs, cudaStream_t st);

}  // namespace dl
