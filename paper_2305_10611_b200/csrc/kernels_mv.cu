// kernels_mv.cu — the MV-RNN combine cell, FP32 and bit-identical to the reference.
//
// Plan (proj/src/zoo.cpp:124-136, lowered by kernelgen into one ExecutablePlan):
//   T0 = x0 . M0        x0 (1 x K) and M0 (K x N) both per-instance (batched): lres.0 . rres.1
//   T1 = x1 . M1        rres.0 . lres.1
//   T2 = concat(T0, T1)                      (1 x 2N)
//   T3 = T2 . W         W (2N x U) shared    (v_wt)
//   T4 = chain(T3)      e.g. + vbias, tanh   (shared rows / unaries)
// and, one depth later in the same flush, the matrix add M = M1 + M0 of the same nodes (zoo.cpp:
// 135, its own batch in the schedule).  Both read the same two per-instance matrices, so when the
// flush holds the two batches back to back over the same nodes (backend.cpp: mv_pair) one launch
// streams each matrix from HBM once and writes both batches' outputs: 2 x K x N floats read and
// K x N written per node, against 4 x K x N read + K x N written for the two batches separately.
//
// Mapping: a cluster of CS CTAs per node (CS column slices of NC = N / CS columns, 32 at H=128),
// 256 threads each.  A CTA issues its whole slice at once — NC columns of every row of both
// matrices, the two rows, and its U / CS rows of W^T (transposed once per parameter upload by the
// host, launch_mv_transpose) — as 16-byte cp.async (4-byte when the node's offsets are not 16-byte
// aligned), so a node costs one memory round trip; under PDL the W^T slice streams in before the
// previous level finishes.  The fused matrix add is written from the landed slice.  Then every
// product x[p] * M[p][j] is formed in place by all threads, and threads [0, NC) / [NC, 2 NC) add
// column j's products of T0 / T1 in row order (the reference's sequential chain acc = acc +
// x[p] * M[p][j], p ascending, separately rounded multiply and add, proj/src/backend.cpp:116-131),
// so the serial part of the chain is the adds alone.  The T0 / T1 slices go into every cluster
// peer's T2 row (DSMEM), one cluster barrier, T3's products T2[p] * W[p][j] in place over the W^T
// slice, threads [0, U / CS) add their column's in order and run the tail with the glibc-exact
// activations.
//
// Roofline: HBM (per-instance matrices; 75.5 MFLOP for 189 MB at MV-RNN-128 b64).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "devplan.h"
#include "kernels.h"
#include "libm_fp32.cuh"

namespace mbx {

using namespace mbx_libm;

namespace {

constexpr int kMvThreads = 256;
constexpr size_t kMaxCtasPerSm = 2048 / kMvThreads;

#ifdef MBX_MV_STAMPS  // tools/mv_bench.cu: globaltimer stamps of CTA 0's phases
__device__ unsigned long long g_mv_stamps[16];
__device__ unsigned long long g_mv_clk[2];
#define MV_STAMP(i)                                                                              \
  do {                                                                                           \
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {                                \
      unsigned long long t;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                                      \
      g_mv_stamps[i] = t;                                                                        \
      if (i == 0 || i == 6) g_mv_clk[i ? 1 : 0] = clock64();                                      \
    }                                                                                            \
  } while (0)
#else
#define MV_STAMP(i) \
  do {              \
  } while (0)
#endif

__host__ __device__ constexpr int mv_align4(int n) { return (n + 3) & ~3; }

__device__ __forceinline__ void mv_cp16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
__device__ __forceinline__ void mv_cp4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}

__device__ __forceinline__ float mv_apply(int op, float v, float rhs) {
  switch (op) {
    case kAdd: return fadd(v, rhs);
    case kMul: return fmul(v, rhs);
    case kSigmoid: return sigmoidf_exact(v);
    case kTanh: return tanhf_exact(v);
    case kRelu: return reluf_exact(v);
    default: return v;
  }
}

// Copies n contiguous floats into shared memory (16-byte pieces when both ends are aligned).
__device__ __forceinline__ void copy_flat(float* dst, const float* src, int n, int tid) {
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (n & 3) == 0) {
    for (int i = tid; i < (n >> 2); i += kMvThreads) mv_cp16(dst + 4 * i, src + 4 * i);
  } else {
    for (int i = tid; i < n; i += kMvThreads) mv_cp4(dst + i, src + i);
  }
}

// Copies rows x cols floats (global rows `gstride` apart) into shared memory (rows `cols` apart):
// 16-byte cp.async when both sides allow it, 4-byte otherwise.
__device__ __forceinline__ void copy_rows(float* dst, const float* src, int rows, int cols, int64_t gstride, int tid) {
  const bool v16 = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (gstride & 3) == 0 && (cols & 3) == 0;
  if (v16) {
    const int q = cols >> 2;  // 16-byte pieces per row
    if (kMvThreads % q == 0) {
      const int pc = tid % q, rstep = kMvThreads / q;
      for (int r = tid / q; r < rows; r += rstep) mv_cp16(dst + r * cols + 4 * pc, src + r * gstride + 4 * pc);
    } else {
      for (int i = tid; i < rows * q; i += kMvThreads) {
        const int r = i / q, c4 = (i - r * q) * 4;
        mv_cp16(dst + r * cols + c4, src + r * gstride + c4);
      }
    }
  } else {
    for (int i = tid; i < rows * cols; i += kMvThreads) {
      const int r = i / cols, c = i - r * cols;
      mv_cp4(dst + r * cols + c, src + r * gstride + c);
    }
  }
}

// The fused matrix add over this CTA's column slice: out = M1 + M0 (fp32 + is commutative, so
// this equals the reference's lm + rm).
__device__ __forceinline__ void mv_add_slice(const MvCellLaunch& A, const float* ms, int64_t node, int s, int K, int N,
                                             int NC, int tid, int nthr) {
  float* out = A.arena + A.add_out[0] + node * int64_t(K) * N + s * NC;
  const int64_t ob = A.add_out[0] + node * int64_t(K) * N + s * NC;
  if ((ob & 3) == 0 && (N & 3) == 0 && (NC & 3) == 0 && nthr % (NC >> 2) == 0) {
    const int q = NC >> 2, c4 = (tid % q) * 4, step = nthr / q;
#pragma unroll 4
    for (int r = tid / q; r < K; r += step) {
      const float4 a = *reinterpret_cast<const float4*>(ms + r * NC + c4);
      const float4 b = *reinterpret_cast<const float4*>(ms + (K + r) * NC + c4);
      *reinterpret_cast<float4*>(out + int64_t(r) * N + c4) =
          make_float4(fadd(b.x, a.x), fadd(b.y, a.y), fadd(b.z, a.z), fadd(b.w, a.w));
    }
  } else {
    for (int i = tid; i < K * NC; i += nthr) {
      const int r = i / NC, c = i - r * NC;
      out[int64_t(r) * N + c] = fadd(ms[(K + r) * NC + c], ms[r * NC + c]);
    }
  }
}

// acc = 0; acc = acc + x[r] * m[r * stride] for r = 0 .. n-1: the reference's sequential chain.
// Products of a block of 16 steps are formed first (independent loads and multiplies), then added
// in order, so the chain waits on the adds, not on every shared-memory load.
__device__ __forceinline__ float chain_dot(const float* x, const float* m, int stride, int n) {
  float acc = 0.0f;
  int r = 0;
  for (; r + 16 <= n; r += 16) {
    float p[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) p[k] = fmul(x[r + k], m[(r + k) * stride]);
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fadd(acc, p[k]);
  }
  for (; r < n; ++r) acc = fadd(acc, fmul(x[r], m[r * stride]));
  return acc;
}

// The same chain over a contiguous, 16-byte aligned m and x: 16-byte loads.
__device__ __forceinline__ float chain_dot4(const float* x, const float* m, int n) {
  float acc = 0.0f;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* m4 = reinterpret_cast<const float4*>(m);
  int r = 0;
  for (; r + 16 <= n; r += 16) {
    float p[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 a = x4[(r >> 2) + k], b = m4[(r >> 2) + k];
      p[4 * k] = fmul(a.x, b.x);
      p[4 * k + 1] = fmul(a.y, b.y);
      p[4 * k + 2] = fmul(a.z, b.z);
      p[4 * k + 3] = fmul(a.w, b.w);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fadd(acc, p[k]);
  }
  for (; r < n; ++r) acc = fadd(acc, fmul(x[r], m[r]));
  return acc;
}

// W (2N x U, row-major) -> W^T rows of 2N + 4 floats (column j contiguous, 16-byte aligned).
__global__ void mv_transpose_kernel(const float* w, float* wt, int R, int U) {
  const int64_t n = int64_t(R) * U;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / U), j = int(i - int64_t(r) * U);
    wt[int64_t(j) * (R + 4) + r] = w[i];
  }
}

__global__ void __launch_bounds__(kMvThreads) mv_cell_kernel(const __grid_constant__ MvCellLaunch A) {
  extern __shared__ __align__(16) float sm[];
  const int K = A.K, N = A.N, U = A.U, CS = A.cs;
  const int NC = N / CS, UC = U / CS;
  const int tid = threadIdx.x;
  const int s = blockIdx.x;            // column slice (= rank in the cluster)
  const int64_t node = blockIdx.y;
  // late_wt (levels too large for one wave of CTAs): W^T's slice reuses the matrices' space once
  // they are consumed (a third less shared memory, twice the CTAs per SM).
  const int mreg = mv_align4(2 * K * NC), wreg = (2 * N + 4) * UC;
  float* ms = sm;                                  // [2][K][NC]: this slice of M0, M1
  float* ws = A.late_wt ? sm : ms + mreg;          // [UC][2N + 4]: this slice of W, transposed
  float* xs = A.late_wt ? sm + max(mreg, wreg) : ws + wreg;  // [2][K]
  float* t2 = xs + mv_align4(2 * K);               // [2N]
  MV_STAMP(0);
  if (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // peers started (DSMEM)
  const int64_t* bo = A.batched_off + node * A.nb;
  // This slice of W^T (the host's transposed copy of W): UC contiguous rows of 2N + 4 floats.  It
  // does not depend on the previous kernel (the host enables PDL only then), so it streams in
  // while that kernel, which produces this level's rows and matrices, finishes.
  if (!A.late_wt) copy_flat(ws, A.wt + int64_t(s) * UC * (2 * N + 4), UC * (2 * N + 4), tid);
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  copy_rows(ms, A.arena + bo[A.m[0]] + s * NC, K, NC, N, tid);
  copy_rows(ms + K * NC, A.arena + bo[A.m[1]] + s * NC, K, NC, N, tid);
  copy_flat(xs, A.arena + bo[A.x[0]], K, tid);
  copy_flat(xs + K, A.arena + bo[A.x[1]], K, tid);
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (A.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  MV_STAMP(1);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  MV_STAMP(2);
  if (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer runs: DSMEM is live
  // ---- T0 / T1 chains (warps holding threads [0, 2 NC)) and, beside them on the other warps,
  // the fused matrix add ----
  const int cthr = (2 * NC + 31) & ~31;  // threads of the chain warps
  const bool add_beside = A.add_out && kMvThreads - cthr >= 32;
  if (A.add_out && add_beside && tid >= cthr) mv_add_slice(A, ms, node, s, K, N, NC, tid - cthr, kMvThreads - cthr);
  if (tid < 2 * NC) {
    const int g = tid / NC, j = tid - g * NC;
    // The reference zero-fills the dense output, then accumulates in row order.
    const float acc = chain_dot(xs + g * K, ms + g * K * NC + j, NC, K);
    const int pos = (g == 0 ? A.first : 1 - A.first) * N + s * NC + j;  // column of T2
    if (CS > 1) {
      const unsigned local = unsigned(__cvta_generic_to_shared(t2 + pos));
      for (int q = 0; q < CS; ++q) {
        unsigned remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(q));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(acc) : "memory");
      }
    } else {
      t2[pos] = acc;
    }
  }
  MV_STAMP(3);
  if (A.add_out && !add_beside) {
    __syncthreads();
    mv_add_slice(A, ms, node, s, K, N, NC, tid, kMvThreads);
  }
  if (A.late_wt) {  // the matrices are consumed: W^T's slice into their space
    __syncthreads();
    copy_flat(ws, A.wt + int64_t(s) * UC * (2 * N + 4), UC * (2 * N + 4), tid);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (CS > 1) {
    // Every slice of T2 is in every peer's shared memory (release / acquire at cluster scope).
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (A.late_wt) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  MV_STAMP(5);
  // ---- T3 = T2 . W (this CTA's UC columns, W^T rows contiguous) and the chain ----
  if (tid < UC) {
    const float* wr = ws + tid * (2 * N + 4);
    float v = (N & 1) == 0 ? chain_dot4(t2, wr, 2 * N) : chain_dot(t2, wr, 1, 2 * N);
    const int col = s * UC + tid;
    for (int l = 0; l < A.nlinks; ++l) {
      const float rhs = A.link_rhs[l] >= 0 ? A.arena[A.shared_off[A.link_rhs[l]] + col] : 0.0f;
      v = mv_apply(A.link_op[l], v, rhs);
    }
    A.arena[A.cell_out[0] + node * U + col] = v;
  }
  MV_STAMP(6);
}

}  // namespace

// Column slices per node: 32-column slices where N and U split evenly (a cluster of <= 8).
int mv_cell_slices(int N, int U) {
  for (int cs = std::min(8, std::max(1, N / 32)); cs > 1; cs >>= 1)
    if (N % cs == 0 && U % cs == 0) return cs;
  return 1;
}

size_t mv_cell_smem(int K, int N, int U, bool late_wt = false) {
  const int cs = mv_cell_slices(N, U);
  const int mreg = mv_align4(2 * K * (N / cs)), wreg = (2 * N + 4) * (U / cs);
  return size_t((late_wt ? std::max(mreg, wreg) : mreg + wreg) + mv_align4(2 * K) + 2 * N) * sizeof(float);
}

bool mv_cell_supported(int K, int N, int U) {
  const int cs = mv_cell_slices(N, U);
  return K >= 1 && N >= 1 && U >= 1 && 2 * (N / cs) <= kMvThreads && U / cs <= kMvThreads &&
         mv_cell_smem(K, N, U) <= 227 * 1024;
}

size_t mv_wt_floats(int N, int U) { return size_t(U) * (2 * N + 4); }

cudaError_t launch_mv_transpose(const float* w, float* wt, int N, int U, cudaStream_t stream) {
  const int64_t n = int64_t(2 * N) * U;
  mv_transpose_kernel<<<int(std::min<int64_t>((n + 255) / 256, 148 * 4)), 256, 0, stream>>>(w, wt, 2 * N, U);
  return cudaGetLastError();
}

cudaError_t launch_mv_cell(const MvCellLaunch& L0, cudaStream_t stream) {
  MvCellLaunch L = L0;
  L.cs = mv_cell_slices(L.N, L.U);
  // A level with more node clusters than one wave holds at the full layout (W^T staged up front)
  // takes the late-W^T layout: two-thirds of the shared memory, more CTAs per SM.
  auto nodes_per_wave = [&](size_t smem) {
    const int per_sm = int(std::min<size_t>(kMaxCtasPerSm, (228 * 1024) / (smem + 1024)));
    return 148 * per_sm / L.cs;
  };
  L.late_wt = L.b > nodes_per_wave(mv_cell_smem(L.K, L.N, L.U)) ? 1 : 0;
  const size_t smem = mv_cell_smem(L.K, L.N, L.U, L.late_wt != 0);
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t attr = cudaSuccess;
  std::call_once(once[dev & 63], [&] {
    attr = cudaFuncSetAttribute(mv_cell_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(L.cs), unsigned(L.b), 1);
  cfg.blockDim = dim3(kMvThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(L.cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = L.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, mv_cell_kernel, L);
}

}  // namespace mbx
