// Launchers of the adaptive-step kernels (iht_adaptive.cu); internal to libiht.
#pragma once
#include "iht_internal.cuh"

int ad_gather(const float* g, int64_t N, int64_t col_offset, const int32_t* gi, const int32_t* gn, int ldg,
              int32_t* xi, float* xv, int32_t* xn, float* num, int B, cudaStream_t st);
int ad_norm(const float* r, int64_t vlen, float* nrm, int B, cudaStream_t st);
int ad_step(const float* num, const float* den, float fallback, int B, float* mu, int32_t* state, cudaStream_t st);
int ad_delta(const int32_t* pi, const float* pv, const int32_t* pn, const int32_t* gi, const int32_t* gn, int ldg,
             const int32_t* xi, const float* xv, const int32_t* xn, int s, int32_t* state, int32_t* di, float* dv,
             int32_t* dn, float* dnum, int B, cudaStream_t st);
int ad_decide(const float* dnum, const float* dden, float c, float k, int max_shrink, int B, float* mu, int32_t* state,
              float* mu_rec, int32_t* shr_rec, cudaGraphConditionalHandle handle, int use_handle, int32_t* pending,
              cudaStream_t st);
