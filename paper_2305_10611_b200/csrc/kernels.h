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

// MV-RNN combine cell, optionally fused with the next batch's matrix add (kernels_mv.cu).
struct MvCellLaunch {
  float* arena;
  const int64_t* shared_off;   // the cell plan's shared offsets
  const int64_t* batched_off;  // [b * nb]
  int b, nb;
  int x[2], m[2];              // batched slots of the two GEMVs' rows and matrices
  int first;                   // concat position of x[0] . m[0] (0 or 1)
  int w;                       // shared slot of the 2N x U weight
  int K, N, U;
  int nlinks;
  int link_op[4], link_rhs[4];  // chain on the dense result; rhs: shared slot of a 1 x U row, -1 none
  const int64_t* cell_out;      // [1] output region base
  const int64_t* add_out;       // [1] fused matrix-add output region base, or nullptr
  int cs;                       // column slices per node (set by launch_mv_cell)
  int pdl;                      // programmatic dependent launch: W may be read before the wait
  const float* wt;              // W^T, rows of 2N + 4 floats (launch_mv_transpose)
  int late_wt;                  // W^T's slice loaded once the matrices are consumed (set by launch_mv_cell)
};
size_t mv_wt_floats(int N, int U);
cudaError_t launch_mv_transpose(const float* w, float* wt, int N, int U, cudaStream_t stream);
bool pdl_enabled();
bool mv_cell_supported(int K, int N, int U);
cudaError_t launch_mv_cell(const MvCellLaunch& L, cudaStream_t stream);
cudaError_t launch_dense_argmax(float* arena, const int64_t* shared_off, const int64_t* batched_off, int b, int nb,
                                int a_batched, int a_idx, int w_idx, int K, int N, const int64_t* out_base,
                                const int64_t* out_node, int nout, int out0, int out1, int pdl, cudaStream_t stream);
size_t dense_argmax_smem(int K, int N);
// [concat(rows...)] plans: out row i = the whole rows r_k(i) side by side (kernels_vm.cu).
struct ConcatLaunch {
  const int64_t* shared_off;
  const int64_t* batched_off;
  const int64_t* out_base;  // [1]
  int b, nb, nin, width;
  int kind[8], idx[8], cols[8];  // kind 1 batched, 0 shared
};
cudaError_t launch_concat_rows(float* arena, const ConcatLaunch& L, cudaStream_t stream);
cudaError_t launch_gather_rows(float* arena, const int64_t* src_off, int64_t dst_off, int b, int size,
                               cudaStream_t stream);
cudaError_t launch_scatter_ranges(const float* src, const int64_t* ranges, int n, float* arena, cudaStream_t stream);
cudaError_t launch_pack_ranges(const float* arena, const int64_t* ranges, int n, float* dst,
                               cudaStream_t stream);
cudaError_t launch_fill(float* arena, int64_t off, int64_t n, float v, cudaStream_t stream);
cudaError_t launch_primop(float* arena, int op, int64_t a_off, int ar, int ac, int64_t b_off, int br, int bc,
                          int64_t out_off, int orows, int ocols, cudaStream_t stream);

}  // namespace mbx
