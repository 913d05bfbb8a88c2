// kernels.h — host-side launch interface of the device kernels (kernels_vm.cu, kernels_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devplan.h"

namespace mbx {

struct VmLaunch {
  const DPlan* plan;           // device copy of the compiled plan
  float* arena;                // arena base (device)
  int b;                       // nodes in the batch
  int tm;                      // nodes per CTA (<= kMaxTM)
  int nsplit;                  // column tiles
  int unit_chunk;              // columns per tile
  int threads;
  int smem_bytes;              // temps (tm * temp_floats) + weight staging
  int temp_floats_total;       // tm * temp_floats
  int wst_floats;              // weight staging floats (0: stream weights from L2)
  const int64_t* shared_off;   // [nshared]
  const int64_t* batched_off;  // [b * nbatched]
  const int64_t* out_base;     // [nout] region base offsets
};

cudaError_t launch_plan_vm(const VmLaunch& L, cudaStream_t stream);
cudaError_t launch_dense_argmax(float* arena, const int64_t* shared_off, const int64_t* batched_off, int b, int nb,
                                int a_batched, int a_idx, int w_idx, int K, int N, const int64_t* out_base, int nout,
                                int out0, int out1, cudaStream_t stream);
cudaError_t launch_gather_rows(float* arena, const int64_t* src_off, int64_t dst_off, int b, int size,
                               cudaStream_t stream);
cudaError_t launch_scatter_ranges(const float* src, const int64_t* ranges, int n, float* arena, cudaStream_t stream);
cudaError_t launch_pack_ranges(const float* arena, const int64_t* ranges, int n, float* dst,
                               cudaStream_t stream);
cudaError_t launch_fill(float* arena, int64_t off, int64_t n, float v, cudaStream_t stream);
cudaError_t launch_primop(float* arena, int op, int64_t a_off, int ar, int ac, int64_t b_off, int br, int bc,
                          int64_t out_off, int orows, int ocols, cudaStream_t stream);

}  // namespace mbx
