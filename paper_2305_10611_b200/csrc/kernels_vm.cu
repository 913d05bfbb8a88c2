// kernels_vm.cu — the FP32 plan VM: one generic sm_100a kernel that executes ANY
// backend::ExecutablePlan over a batch of DFG nodes, bit-identical to the reference.
//
// Reference semantics being reproduced (proj/src/exec_batched.cpp:80-145, backend.cpp:105-181):
//   for each instance: for each step: kOp -> exec_primop, kFusedDense -> one dense per stacked
//   weight into its column range, kChain -> v = base[k]; v = op(v, rhs[k]) ...; then copy the
//   plan outputs into batch-contiguous output regions.
// Bit-exactness: dense accumulates c = 0; c += a[p] * w[p][j] for p ascending with separately
// rounded fp32 multiply and add (__fmul_rn/__fadd_rn, no FMA contraction), exactly the
// reference's i-k-j loop per output element; activations use the glibc-exact restatements in
// libm_fp32.cuh.
//
// Mapping: grid = (ceil(b / tm) node tiles) x (nsplit column tiles).  A CTA keeps the temps of
// its tm nodes in shared memory, computes "full" steps entirely and "split" steps (column-local
// w.r.t. the plan's output unit, see devplan.h) only over its column tile, so a shared weight
// tile is read once per node tile instead of once per node, and wide layers spread over many
// SMs.  Operands are read straight from the arena through the per-node offset arrays (the
// gather is fused into the operand loads; nothing is materialized).
#include <cuda_runtime.h>
#include <mutex>
#include <stdint.h>

#include "devplan.h"
#include "kernels.h"
#include "libm_fp32.cuh"

namespace mbx {

using namespace mbx_libm;

namespace {

__device__ __forceinline__ float apply_op(int op, float v, float rhs) {
  switch (op) {
    case kAdd: return fadd(v, rhs);
    case kMul: return fmul(v, rhs);
    case kSigmoid: return sigmoidf_exact(v);
    case kTanh: return tanhf_exact(v);
    case kRelu: return reluf_exact(v);
    default: return v;
  }
}

struct Ctx {
  const DPlan* P;
  float* arena;
  const int64_t* shared_off;
  const int64_t* batched_off;
  float* temps;   // smem base
  int node0, nn;  // first node of the tile, nodes in the tile
  float* wst;     // weight staging area (after the temps), wst_floats long
  int wst_floats;
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
__device__ __forceinline__ void group_sync(int gi, int count) {
  if (count == int(blockDim.x)) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(count) : "memory");
}

__device__ __forceinline__ const float* ref_ptr(const Ctx& c, const DRef& r, int t) {
  int64_t slice = r.cols >= 0 ? r.col_off : 0;
  switch (r.kind) {
    case kRefShared: return c.arena + c.shared_off[r.index] + slice;
    case kRefBatched:
      return c.arena + c.batched_off[int64_t(c.node0 + t) * c.P->nbatched + r.index] + slice;
    default: return c.temps + int64_t(t) * c.P->temp_floats + c.P->steps[r.index].temp_off + slice;
  }
}

__device__ __forceinline__ float* temp_ptr(const Ctx& c, int step, int t) {
  return c.temps + int64_t(t) * c.P->temp_floats + c.P->steps[step].temp_off;
}

// out[i, j] for j in [j0, j1) of a (m x n) = A (m x k) . W (k x n), written at column
// out_col0 + j of an out row of width out_ld.  W is shared (same for all tile nodes) or
// batched (per node).
// Threads [tbase, tbase + tcount) of the CTA take part (the weights of a FusedDense run side by
// side on disjoint thread groups).
constexpr int kMaxCPT = 8;  // output elements per thread in the staged shared-weight path

__device__ void dense_range(const Ctx& c, const DRef& a, const DRef& w, int s, int out_ld,
                            int out_col0, int j0, int j1, int tbase = 0, int tcount = -1, int gi = 0, int ngroups = 1) {
  const int m = a.rows_r, k = a.cols_r, n = w.cols_r;
  const int ncr = j1 - j0;
  if (tcount < 0) tcount = blockDim.x;
  const int tid = int(threadIdx.x) - tbase;
  if (ncr <= 0 || tid < 0 || tid >= tcount) return;
  const int per_group = (c.wst_floats / ngroups) & ~3;
  // Output elements (row i, column jj) per thread: up to kMaxCPT, all accumulated side by side.
  const int cpt = (m * ncr + tcount - 1) / tcount;
  if (w.kind == kRefShared && cpt <= kMaxCPT && per_group >= (ncr + m * c.nn) * 16) {
    // Shared weights: stage W[:, j0:j1] through shared memory in passes of KB rows, every row of
    // a pass in flight at once (cp.async), then run each output's strictly sequential
    // accumulation (p ascending, separate multiply and add) from shared memory.  A thread owns
    // up to kMaxCPT output elements (elements e = tid + q * tcount) for every tile node, so the
    // chains of one thread are independent (ILP) and wide FusedDense steps use every thread.
    const float* W = ref_ptr(c, w, 0) + j0;
    float* ws = c.wst + gi * per_group;
    // Pass of KB rows: W rows [KB][ncr] then the A rows of every tile node [nn][m][KB].
    const int arow = m * c.nn;
    const int KB = min(k, (per_group / (ncr + arow)) & ~3);
    float* as = ws + KB * ncr;
    const bool vec = (ncr % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0);
    int ei[kMaxCPT], ej[kMaxCPT];
    bool act[kMaxCPT];
#pragma unroll
    for (int q = 0; q < kMaxCPT; ++q) {
      const int e = tid + q * tcount;
      act[q] = q < cpt && e < m * ncr;
      ei[q] = act[q] ? e / ncr : 0;
      ej[q] = act[q] ? e % ncr : 0;
    }
    float acc[kMaxCPT][kMaxTM];
#pragma unroll
    for (int q = 0; q < kMaxCPT; ++q)
#pragma unroll
      for (int t = 0; t < kMaxTM; ++t) acc[q][t] = 0.0f;
    for (int p0 = 0; p0 < k; p0 += KB) {
      const int kb = min(KB, k - p0);
      if (vec) {
        const int q4 = ncr / 4;
        for (int idx = tid; idx < kb * q4; idx += tcount) {
          const int r = idx / q4, q = idx - r * q4;
          cp_async16(ws + r * ncr + 4 * q, W + int64_t(p0 + r) * n + 4 * q);
        }
      } else {
        for (int idx = tid; idx < kb * ncr; idx += tcount) {
          const int r = idx / ncr, q = idx - r * ncr;
          cp_async4(ws + idx, W + int64_t(p0 + r) * n + q);
        }
      }
      for (int idx = tid; idx < arow * kb; idx += tcount) {
        const int rr = idx / kb, p = idx - rr * kb;  // rr = t * m + row
        const int t = rr / m, row = rr - t * m;
        const float* src = ref_ptr(c, a, t) + row * k + p0 + p;
        if (a.kind == kRefTemp) as[idx] = *src;  // already in shared memory
        else cp_async4(as + idx, src);
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      group_sync(gi, tcount);
#pragma unroll
      for (int q = 0; q < kMaxCPT; ++q) {
        if (!act[q]) continue;
        const float* wc = ws + ej[q];
        if (c.nn == 1) {  // one node (the hoisted shared prefix): a single dependent chain
          const float* a0 = as + ei[q] * kb;
          float acc0 = acc[q][0];
#pragma unroll 8
          for (int p = 0; p < kb; ++p) acc0 = fadd(acc0, fmul(a0[p], wc[p * ncr]));
          acc[q][0] = acc0;
        } else {
#pragma unroll 4
          for (int p = 0; p < kb; ++p) {
            const float wv = wc[p * ncr];
#pragma unroll
            for (int t = 0; t < kMaxTM; ++t)
              if (t < c.nn) acc[q][t] = fadd(acc[q][t], fmul(as[(t * m + ei[q]) * kb + p], wv));
          }
        }
      }
      group_sync(gi, tcount);
    }
#pragma unroll
    for (int q = 0; q < kMaxCPT; ++q) {
      if (!act[q]) continue;
#pragma unroll
      for (int t = 0; t < kMaxTM; ++t)
        if (t < c.nn) temp_ptr(c, s, t)[ei[q] * out_ld + out_col0 + j0 + ej[q]] = acc[q][t];
    }
    return;
  }
  if (w.kind == kRefShared) {
    const float* W = ref_ptr(c, w, 0);
    const float* A[kMaxTM];
#pragma unroll
    for (int t = 0; t < kMaxTM; ++t) A[t] = t < c.nn ? ref_ptr(c, a, t) : nullptr;
    const int total = m * ncr;
    for (int idx = tid; idx < total; idx += tcount) {
      const int i = idx / ncr, j = j0 + idx % ncr;
      float acc[kMaxTM];
#pragma unroll
      for (int t = 0; t < kMaxTM; ++t) acc[t] = 0.0f;
      const float* wc = W + j;
      // Weights for 8 consecutive p are loaded into registers before they are consumed, so the
      // loads overlap; the accumulation itself stays strictly sequential in p (reference order).
      int p = 0;
      for (; p + 8 <= k; p += 8) {
        float w8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w8[q] = __ldg(wc + int64_t(p + q) * n);
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int t = 0; t < kMaxTM; ++t)
            if (t < c.nn) acc[t] = fadd(acc[t], fmul(A[t][i * k + p + q], w8[q]));
      }
      for (; p < k; ++p) {
        const float wv = __ldg(wc + int64_t(p) * n);
#pragma unroll
        for (int t = 0; t < kMaxTM; ++t)
          if (t < c.nn) acc[t] = fadd(acc[t], fmul(A[t][i * k + p], wv));
      }
#pragma unroll
      for (int t = 0; t < kMaxTM; ++t)
        if (t < c.nn) temp_ptr(c, s, t)[i * out_ld + out_col0 + j] = acc[t];
    }
  } else {
    const int total = c.nn * m * ncr;
    for (int idx = tid; idx < total; idx += tcount) {
      const int t = idx / (m * ncr);
      const int r = idx % (m * ncr);
      const int i = r / ncr, j = j0 + r % ncr;
      const float* A = ref_ptr(c, a, t);
      const float* W = ref_ptr(c, w, t);
      float acc = 0.0f;
#pragma unroll 8
      for (int p = 0; p < k; ++p) acc = fadd(acc, fmul(A[i * k + p], W[int64_t(p) * n + j]));
      temp_ptr(c, s, t)[i * out_ld + out_col0 + j] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) plan_vm_kernel(VmLaunch L) {
  extern __shared__ float smem[];
  const DPlan* P = L.plan;
  Ctx c;
  c.P = P;
  c.arena = L.arena;
  c.shared_off = L.shared_off;
  c.batched_off = L.batched_off;
  c.temps = smem;
  c.wst = smem + ((L.temp_floats_total + 3) & ~3);  // 16-byte aligned for cp.async
  c.wst_floats = L.wst_floats;
  c.node0 = blockIdx.x * L.tm;
  c.nn = min(L.tm, L.b - c.node0);
  if (c.nn <= 0) return;
  const int u0 = blockIdx.y * L.unit_chunk;
  const int u1 = min(u0 + L.unit_chunk, P->unit > 0 ? P->unit : 0);
  const bool tiled = L.nsplit > 1;

  for (int s = 0; s < P->nsteps; ++s) {
    const DStep& st = P->steps[s];
    const bool sp = tiled && st.split;
    switch (st.kind) {
      case kStepFused: {
        int col = 0;
        const int nw = st.nin - 1;
        // Disjoint thread groups of whole warps (named barriers need multiples of 32).
        const int group = nw == 1 ? int(blockDim.x) : (int(blockDim.x) / nw) & ~31;
        for (int w = 1; w < st.nin; ++w) {
          const DRef& wr = st.ins[w];
          if (sp) dense_range(c, st.ins[0], wr, s, st.cols, col, u0, u1, (w - 1) * group, group, w - 1, nw);
          else dense_range(c, st.ins[0], wr, s, st.cols, col, 0, wr.cols_r, (w - 1) * group, group, w - 1, nw);
          col += wr.cols_r;
        }
        break;
      }
      case kStepOp: {
        if (st.op == kDense) {
          if (sp) dense_range(c, st.ins[0], st.ins[1], s, st.cols, 0, u0, u1);
          else dense_range(c, st.ins[0], st.ins[1], s, st.cols, 0, 0, st.cols);
        } else if (st.op == kConcat) {
          const int rows = st.rows, ca = st.ins[0].cols_r, cb = st.ins[1].cols_r;
          const int total = c.nn * rows * (ca + cb);
          for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int t = idx / (rows * (ca + cb));
            const int e = idx % (rows * (ca + cb));
            const int r = e / (ca + cb), j = e % (ca + cb);
            float v = j < ca ? ref_ptr(c, st.ins[0], t)[r * ca + j] : ref_ptr(c, st.ins[1], t)[r * cb + j - ca];
            temp_ptr(c, s, t)[e] = v;
          }
        } else if (st.op == kArgmax) {
          // first index of the max (backend.cpp:164-173); one thread per node.
          for (int t = threadIdx.x; t < c.nn; t += blockDim.x) {
            const float* a = ref_ptr(c, st.ins[0], t);
            int best = 0;
            for (int i = 1; i < st.ins[0].cols_r; ++i)
              if (a[i] > a[best]) best = i;
            temp_ptr(c, s, t)[0] = static_cast<float>(best);
          }
        } else {
          // elementwise add / mul / sigmoid / tanh / relu
          const int n = st.rows * st.cols;
          const int e0 = sp ? u0 : 0, e1 = sp ? u1 : n;
          const int ncr = e1 - e0;
          const int total = c.nn * ncr;
          for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int t = idx / ncr, e = e0 + idx % ncr;
            const float a = ref_ptr(c, st.ins[0], t)[e];
            const float b = st.nin > 1 ? ref_ptr(c, st.ins[1], t)[e] : 0.0f;
            temp_ptr(c, s, t)[e] = apply_op(st.op, a, b);
          }
        }
        break;
      }
      case kStepChain: {
        const int n = st.rows * st.cols;
        const int e0 = sp ? u0 : 0, e1 = sp ? u1 : n;
        const int ncr = e1 - e0;
        const int total = c.nn * ncr;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
          const int t = idx / ncr, e = e0 + idx % ncr;
          float v = ref_ptr(c, st.ins[0], t)[e];
          for (int l = 0; l < st.nchain; ++l) {
            const DLink& lk = st.chain[l];
            const float rhs = lk.has_rhs ? ref_ptr(c, lk.rhs, t)[e] : 0.0f;
            v = apply_op(lk.op, v, rhs);
          }
          temp_ptr(c, s, t)[e] = v;
        }
        break;
      }
    }
    __syncthreads();
  }

  // Plan outputs -> batch-contiguous regions (exec_batched.cpp:146-154).
  for (int k = 0; k < P->nout; ++k) {
    const DRef& o = P->outputs[k];
    const int size = o.rows_r * o.cols_r;
    const bool osp = tiled && P->out_split[k];
    if (!osp && blockIdx.y != 0) continue;
    const int e0 = osp ? u0 : 0, e1 = osp ? u1 : size;
    const int ncr = e1 - e0;
    const int total = c.nn * ncr;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int t = idx / ncr, e = e0 + idx % ncr;
      c.arena[L.out_base[k] + int64_t(c.node0 + t) * size + e] = ref_ptr(c, o, t)[e];
    }
  }
}

// EXPLICIT gather (exec_batched.cpp:46-65): copy each instance's batched slot into a
// contiguous scratch region.
// [concat(rows...)] plans (BiRNN's output concat, zoo.cpp:47-76): out[i] = [r_0(i) | r_1(i) | ...]
// for whole 1 x c_k rows (batched: per node; shared: the same row for every node).  A block per
// node row; 16-byte copies when a piece and its destination are both 16-byte aligned.
__global__ void __launch_bounds__(256) concat_rows_kernel(float* arena, ConcatLaunch L) {
  const int64_t i = blockIdx.x;
  float* out = arena + L.out_base[0] + i * L.width;
  int col = 0;
  for (int k = 0; k < L.nin; ++k) {
    const int c = L.cols[k];
    const float* src = arena + (L.kind[k] == 1 ? L.batched_off[i * L.nb + L.idx[k]] : L.shared_off[L.idx[k]]);
    float* dst = out + col;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && (c & 3) == 0) {
      for (int e = threadIdx.x; e < (c >> 2); e += blockDim.x)
        reinterpret_cast<float4*>(dst)[e] = reinterpret_cast<const float4*>(src)[e];
    } else {
      for (int e = threadIdx.x; e < c; e += blockDim.x) dst[e] = src[e];
    }
    col += c;
  }
}

__global__ void gather_rows_kernel(float* arena, const int64_t* src_off, int64_t dst_off, int b,
                                   int size) {
  const int64_t total = int64_t(b) * size;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / size, e = idx % size;
    arena[dst_off + idx] = arena[src_off[i] + e];
  }
}

// Packs n arena ranges (offset, size) into a contiguous staging buffer (one D2H copy for all
// outputs / scalar decisions of a flush).
// One warp per range (a range is typically one node row of H floats): 16-byte copies when the
// range and both ends are 16-byte aligned, else 4-byte ones.  Used for the outputs' D2H pack
// (arena -> contiguous) and, inverted, for the inputs' scatter (contiguous -> arena).
__device__ __forceinline__ void copy_range_warp(const float* __restrict__ s, float* __restrict__ d, int64_t size,
                                                int lane) {
  if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0 && (size & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4* d4 = reinterpret_cast<float4*>(d);
    for (int64_t e = lane; e < size / 4; e += 32) d4[e] = s4[e];
  } else {
    for (int64_t e = lane; e < size; e += 32) d[e] = s[e];
  }
}

__global__ void pack_ranges_kernel(const float* arena, const int64_t* ranges, int n, float* dst) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
    const int64_t off = ranges[3 * r], size = ranges[3 * r + 1], dst_off = ranges[3 * r + 2];
    copy_range_warp(arena + off, dst + dst_off, size, lane);
  }
}

// The inverse of pack_ranges: contiguous src -> arena ranges (mini-batch inputs copied H2D in one
// piece from the caller's pinned buffer, then scattered to their arena offsets on the device).
// ranges: (src offset, size, arena offset) triples.
__global__ void scatter_ranges_kernel(const float* src, const int64_t* ranges, int n, float* arena) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
    const int64_t so = ranges[3 * r], size = ranges[3 * r + 1], dof = ranges[3 * r + 2];
    copy_range_warp(src + so, arena + dof, size, lane);
  }
}

// exec_primop on arena tensors of any size (backend.cpp:105-181), one output element per thread
// (grid-stride), same arithmetic as the plan VM.
__global__ void primop_kernel(float* arena, int op, int64_t a_off, int ar, int ac, int64_t b_off, int br, int bc,
                              int64_t out_off, int orows, int ocols) {
  const float* A = arena + a_off;
  const float* B = arena + b_off;
  float* O = arena + out_off;
  const int64_t n = int64_t(orows) * ocols;
  if (op == kArgmax) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int best = 0;
      for (int i = 1; i < ac; ++i)
        if (A[i] > A[best]) best = i;
      O[0] = static_cast<float>(best);
    }
    return;
  }
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n; idx += int64_t(gridDim.x) * blockDim.x) {
    float v;
    if (op == kDense) {
      const int64_t i = idx / ocols, j = idx % ocols;
      float acc = 0.0f;
      for (int p = 0; p < ac; ++p) acc = fadd(acc, fmul(A[i * ac + p], B[int64_t(p) * bc + j]));
      v = acc;
    } else if (op == kConcat) {
      const int64_t r = idx / ocols, j = idx % ocols;
      v = j < ac ? A[r * ac + j] : B[r * bc + (j - ac)];
    } else {
      v = apply_op(op, A[idx], (op == kAdd || op == kMul) ? B[idx] : 0.0f);
    }
    O[idx] = v;
  }
}

__global__ void fill_kernel(float* arena, int64_t off, int64_t n, float v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    arena[off + i] = v;
}

}  // namespace

// dense + argmax plans (backend.cpp:116-131, :164-173), one CTA per node: the weight (K x N) and
// the node's row go to shared memory, N threads run the exact sequential chains (p ascending,
// separately rounded multiply and add), thread 0 takes the first index of the maximum.
// [dense(a . W), argmax] per node (NestedRNN's decision tail), exact: one CTA per node.  W
// (K x N, N <= 32) and the row stream into shared memory with cp.async (W before the PDL wait: it
// is a session parameter whenever PDL is on); every product a[p] * W[p][j] is formed by all
// threads into a transposed buffer; thread j < N then adds column j's products in p order (the
// reference's chain, backend.cpp:116-131) with 16-byte loads, and warp 0 takes the argmax (first
// maximum, backend.cpp:164-173).
__global__ void __launch_bounds__(256) dense_argmax_kernel(float* arena, const int64_t* shared_off,
                                                           const int64_t* batched_off, int nb, int a_batched, int a_idx,
                                                           int w_idx, int K, int N, const int64_t* out_base,
                                                           const int64_t* out_node, int nout, int out0, int out1,
                                                           int pdl) {
  extern __shared__ __align__(16) float sm[];
  const int KP = (K + 7) & ~3;           // transposed row stride: 16-byte aligned, K + 4 .. K + 7
  float* ws = sm;                         // [K][N]
  float* as = ws + ((K * N + 3) & ~3);    // [K]
  float* pt = as + ((K + 3) & ~3);        // [N][KP]
  float* row = pt + N * KP;               // [N]
  const int tid = threadIdx.x;
  const int64_t node = blockIdx.x;
  {
    const float* w = arena + shared_off[w_idx];
    if ((reinterpret_cast<uintptr_t>(w) & 15) == 0 && (K * N) % 4 == 0) {
      for (int i = tid; i < K * N / 4; i += 256) cp_async16(ws + 4 * i, w + 4 * i);
    } else {
      for (int i = tid; i < K * N; i += 256) cp_async4(ws + i, w + i);
    }
  }
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    const float* a = arena + (a_batched ? batched_off[node * nb + a_idx] : shared_off[a_idx]);
    for (int i = tid; i < K; i += 256) cp_async4(as + i, a + i);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  for (int p = tid; p < K; p += 256) {
    const float av = as[p];
    for (int j = 0; j < N; ++j) pt[j * KP + p] = fmul(av, ws[p * N + j]);
  }
  __syncthreads();
  if (tid < N) {
    const float* q = pt + tid * KP;
    float acc = 0.0f;  // the reference zero-fills the output, then accumulates in p order
    int p = 0;
#pragma unroll 4
    for (; p + 4 <= K; p += 4) {
      const float4 v = *reinterpret_cast<const float4*>(q + p);
      acc = fadd(fadd(fadd(fadd(acc, v.x), v.y), v.z), v.w);
    }
    for (; p < K; ++p) acc = fadd(acc, q[p]);
    row[tid] = acc;
  }
  __syncthreads();
  const int outs[2] = {out0, out1};
  for (int k = 0; k < nout; ++k) {
    // merged launches (several batches' nodes): per-node output offsets
    const int64_t base = out_node ? out_node[node * nout + k] : out_base[k] + node * (outs[k] == 0 ? N : 1);
    if (outs[k] == 0) {
      for (int j = tid; j < N; j += 256) arena[base + j] = row[j];
    } else if (tid == 0) {
      int best = 0;
      for (int i = 1; i < N; ++i)
        if (row[i] > row[best]) best = i;
      arena[base] = static_cast<float>(best);
    }
  }
}

size_t dense_argmax_smem(int K, int N) {
  return size_t(((K * N + 3) & ~3) + ((K + 3) & ~3) + N * ((K + 7) & ~3) + N) * sizeof(float);
}

cudaError_t launch_dense_argmax(float* arena, const int64_t* shared_off, const int64_t* batched_off, int b, int nb,
                                int a_batched, int a_idx, int w_idx, int K, int N, const int64_t* out_base,
                                const int64_t* out_node, int nout, int out0, int out1, int pdl, cudaStream_t stream) {
  const size_t smem = dense_argmax_smem(K, N);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(dense_argmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(b));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, dense_argmax_kernel, arena, shared_off, batched_off, nb, a_batched, a_idx, w_idx, K, N,
                            out_base, out_node, nout, out0, out1, pdl);
}

cudaError_t launch_plan_vm(const VmLaunch& L, cudaStream_t stream) {
  // The attribute is per device: set once per device, safely from concurrent pool workers.
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t attr = cudaSuccess;
  std::call_once(once[dev & 63], [&] {
    attr = cudaFuncSetAttribute(plan_vm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr != cudaSuccess) return attr;
  dim3 grid((L.b + L.tm - 1) / L.tm, L.nsplit);
  plan_vm_kernel<<<grid, L.threads, L.smem_bytes, stream>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_concat_rows(float* arena, const ConcatLaunch& L, cudaStream_t stream) {
  concat_rows_kernel<<<L.b, 128, 0, stream>>>(arena, L);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(float* arena, const int64_t* src_off, int64_t dst_off, int b, int size,
                               cudaStream_t stream) {
  int64_t total = int64_t(b) * size;
  int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 8));
  gather_rows_kernel<<<blocks, 256, 0, stream>>>(arena, src_off, dst_off, b, size);
  return cudaGetLastError();
}

cudaError_t launch_scatter_ranges(const float* src, const int64_t* ranges, int n, float* arena, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  scatter_ranges_kernel<<<std::min((n + 7) / 8, 148 * 8), 256, 0, stream>>>(src, ranges, n, arena);
  return cudaGetLastError();
}

cudaError_t launch_pack_ranges(const float* arena, const int64_t* ranges, int n, float* dst,
                               cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  pack_ranges_kernel<<<std::min((n + 7) / 8, 148 * 8), 256, 0, stream>>>(arena, ranges, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_primop(float* arena, int op, int64_t a_off, int ar, int ac, int64_t b_off, int br, int bc,
                          int64_t out_off, int orows, int ocols, cudaStream_t stream) {
  const int64_t n = int64_t(orows) * ocols;
  int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
  primop_kernel<<<blocks, 256, 0, stream>>>(arena, op, a_off, ar, ac, b_off, br, bc, out_off, orows, ocols);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* arena, int64_t off, int64_t n, float v, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 8));
  fill_kernel<<<blocks, 256, 0, stream>>>(arena, off, n, v);
  return cudaGetLastError();
}

}  // namespace mbx
