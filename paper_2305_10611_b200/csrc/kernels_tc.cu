// kernels_tc.cu — tcgen05 tensor-core kernel for the gate-GEMM cells of the batched plans.
//
// Applies to every plan of the shape
//     [concat(p0, p1)] -> dense / FusedDense(row, W_1..W_G  shared) -> column-local elementwise tail
// i.e. the TreeLSTM internal cell (add_mul_sigmoid_bias: concat(lh,rh) . [W_i|W_fl|W_fr|W_u],
// gates, c, tanh(c)), bias_dense, the recurrent sigmoid_add_dense of RNN/BiRNN, NestedRNN's inner
// cell, ... (kernelgen.cpp:100-132 emits the FusedDense; lower_block_to_kernel the chains).
//
// Mapping (swap-AB: the MMA M dimension is gate columns, N is DFG nodes, so ragged node counts
// waste at most 15 columns instead of up to 127 rows):
//   grid = (ceil(b / NT) node tiles) x (U / UC unit tiles); one CTA per SM (227 KB smem).
//   A (M x K, K-major)  = the unit tile's gate columns of all G weights, pre-packed once into the
//                         canonical no-swizzle UMMA layout as split bf16 (hi, lo), streamed
//                         chunk by chunk with cp.async.bulk (TMA bulk engine) on an mbarrier ring.
//   B (NT x K, K-major) = the tile's node rows, GATHERED straight from the arena through the
//                         per-node offset table (the reference's concat/gather is never
//                         materialised), converted to split bf16 in shared memory.
//   D (M x NT, fp32)    = TMEM accumulator; BF16x3: D += Wh*Xh + Wh*Xl + Wl*Xh (fp32-accurate
//                         operands, ~1e-5 relative), BF16: D += Wh*Xh.
//   epilogue            = tcgen05.ld -> smem -> per-element interpretation of the plan's
//                         elementwise tail (same libm-exact ops as the FP32 VM) -> outputs written
//                         batch-contiguously into the arena.
// One elected thread issues all tcgen05.mma / commits; every other thread gathers.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "libm_fp32.cuh"
#include "tc.h"

namespace mbx {

using namespace mbx_libm;

constexpr int kTcThreads = 256;
constexpr int kStages = 3;
constexpr int kMaxEpi = 24;

// Micro-op program of a plan's column-local tail (see compile_epilogue).
// Micro-op operands: a slot (earlier tail step), a gate of the accumulator tile, or one of the
// prefetched input rows (loads[idx], a batched or shared input + column slice).
enum : int8_t { kSrcNone = 0, kSrcSlot = 1, kSrcAcc = 2, kSrcBatched = 3, kSrcShared = 4, kSrcLoad = 5 };
constexpr int kOpCopy = 99;
constexpr int kMaxLoads = 12;
struct EpiSrc {
  int8_t type;
  int8_t pad;
  int16_t idx;  // slot / accumulator gate g / batched or shared input index / load index
  int32_t off;  // column-slice offset into the input row
};
struct EpiOp {
  int32_t op, dst;
  EpiSrc a, b;
};
struct EpiProg {
  int32_t nops, nslots, nout, nloads;
  int32_t out_slot[kMaxOut];
  EpiSrc loads[kMaxLoads];
  EpiOp ops[56];
};

struct TcArgs {
  const EpiProg* epi;
  const DPlan* plan;
  float* arena;
  const int64_t* shared_off;
  const int64_t* batched_off;
  const int64_t* out_base;
  const uint8_t* wpack;
  int b, K, KC, nchunks, U, G, UC, M, NT, npass, dstep, nb;
  int npieces;
  int piece_kind[2], piece_idx[2], piece_off[2], piece_k[2];
  uint32_t idesc;
  int x_bytes;        // per pass (hi or lo) X bytes: NT * K * 2
  int w_chunk_bytes;  // per pass W chunk bytes: M * KC * 2
  int tmem_cols;
  int ring_bytes;     // stages * (W chunk + X chunk); epilogue program, slots and D tile reuse it
  int stages;
  int bulk_x;         // 1: node rows land by bulk copy (every row offset 16-byte aligned)
  int ksplit;         // K-split ranks per tile (= cluster size along grid z)
  int epi_nslots, epi_nloads;
  int debug;          // MBX_TC_DEBUG bits (profiling only): 1 skip MMAs, 2 skip W copies
  unsigned long long* ts;  // MBX_TC_DEBUG & 16: %globaltimer phase stamps of CTA (0,0)
};

__device__ __forceinline__ void stamp(const TcArgs& P, int i) {
  if (P.ts && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.ts[i] = t;
    if (i == 0 || i == 4) P.ts[62 + (i == 4)] = clock64();
  }
}

__host__ __device__ inline int npass_x(const TcArgs& P) { return P.x_bytes * (P.npass > 1 ? 2 : 1); }

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Spin on the non-blocking test_wait: try_wait may park the warp for a scheduler quantum, which
// costs microseconds per hand-off in a ring that turns over every few hundred cycles.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// Canonical K-major, no-swizzle smem matrix descriptor: 8-row x 16-byte core matrices, K-adjacent
// core matrices LBO = 128 B apart, 8-row groups SBO bytes apart (cute UMMA::make_umma_desc<K>,
// LayoutType::INTERLEAVE; version 1 for sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((128u >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

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

// Offset of element (row r, k) inside one K-chunk of the canonical layout (bytes).
__device__ __forceinline__ uint32_t canon_off(int r, int kk, int KC) {
  return uint32_t((r >> 3) * (KC * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// One CTA = (node tile of NT nodes) x (unit tile of UC units = M gate rows) x (K-split rank).
// The S K-split ranks of a tile form a thread-block cluster; their partial accumulators are
// reduced through distributed shared memory and each rank finishes NT/S of the nodes.
__global__ void __launch_bounds__(kTcThreads, 1) tc_gate_kernel(TcArgs P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int node0 = blockIdx.x * P.NT;
  const int tile_u = blockIdx.y;
  const int nn = min(P.NT, P.b - node0);
  const int KC = P.KC;
  const int npass = P.npass;
  const int S = P.stages;
  const int ksplit = P.ksplit;
  uint32_t rank = 0;
  if (ksplit > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cpr = P.nchunks / ksplit;  // chunks per rank
  const int c_begin = int(rank) * cpr;
  if (tid == 0) stamp(P, 0);

  const int wstage = P.w_chunk_bytes * (npass > 1 ? 2 : 1);
  const int xchunk = P.NT * KC * 2;
  const int xstage = xchunk * (npass > 1 ? 2 : 1);
  const int rawbytes = P.bulk_x ? P.NT * KC * 4 : 0;
  const int stage_bytes = wstage + rawbytes + xstage;
  uint8_t* ring = smem;
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem + P.ring_bytes);
  uint64_t* full_x = full_w + S;
  uint64_t* empty = full_x + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int64_t* rowbase = reinterpret_cast<int64_t*>(done + 2);  // [NT][2] arena offset of each piece row
  float* dsm = reinterpret_cast<float*>(smem + P.ring_bytes - P.NT * P.M * 4);  // [NT][M] partial D

  for (int i = tid; i < P.NT * 2; i += kTcThreads) {
    const int n = i >> 1, pc = i & 1;
    int64_t base = 0;
    if (n < nn && pc < P.npieces)
      base = (P.piece_kind[pc] == kRefShared ? P.shared_off[P.piece_idx[pc]]
                                             : P.batched_off[int64_t(node0 + n) * P.nb + P.piece_idx[pc]]) +
             P.piece_off[pc];
    rowbase[i] = base;
  }

  constexpr int kGatherWarps = 6;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_w[s], 1);
      mbar_init(&full_x[s], kGatherWarps * 32);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) stamp(P, 1);

  if (warp == 0) {
    // ---- Producer warp: the weight chunk (one bulk copy) and, with bulk_x, one bulk copy per
    // node row segment, all on the bulk-copy (TMA) engine, up to S stages ahead of the MMAs.
    const uint8_t* wtile = P.wpack + size_t(tile_u) * P.nchunks * wstage;
    for (int i = 0; i < cpr; ++i) {
      const int c = c_begin + i, s = i % S;
      if (lane == 0) {
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        const int wb = (P.debug & 2) ? 0 : wstage;
        mbar_expect_tx(&full_w[s], wb + ((P.bulk_x && !(P.debug & 64)) ? nn * KC * 4 : 0));
        if (wb) bulk_g2s(ring + s * stage_bytes, wtile + size_t(c) * wstage, wstage, &full_w[s]);
      }
      __syncwarp();
      if (P.bulk_x && !(P.debug & 64)) {
        uint8_t* raw = ring + s * stage_bytes + wstage;
        const int k0 = c * KC, k1 = k0 + KC;
        for (int n = lane; n < nn; n += 32) {
          for (int pc = 0; pc < P.npieces; ++pc) {
            const int p0 = pc ? P.piece_k[0] : 0, p1 = P.piece_k[pc];
            const int a = max(k0, p0), b = min(k1, p1);
            if (a >= b) continue;
            bulk_g2s(raw + (n * KC + (a - k0)) * 4, P.arena + rowbase[2 * n + pc] + (a - p0), uint32_t(b - a) * 4,
                     &full_w[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: one thread issues every tcgen05.mma and commit ----
    if (lane == 0) {
      const uint32_t ra = smem_u32(ring);
      const uint32_t sbo = uint32_t(KC * 16);
      for (int i = 0; i < cpr; ++i) {
        const int s = i % S;
        mbar_wait(&full_w[s], (i / S) & 1);
        mbar_wait(&full_x[s], (i / S) & 1);
        tc_fence_after();
        const uint32_t wa = ra + s * stage_bytes;
        const uint32_t xa = wa + wstage + rawbytes;
        const uint64_t a_hi = make_desc(wa, sbo), b_hi = make_desc(xa, sbo);
        const uint64_t a_lo = make_desc(wa + P.w_chunk_bytes, sbo), b_lo = make_desc(xa + xchunk, sbo);
        const int nks = (P.debug & 1) ? 0 : KC / 16;
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t step = uint64_t(ks * 16);  // +256 B in the 16-byte-unit address field
          mma_bf16(tmem, a_hi + step, b_hi + step, P.idesc, (i | ks) ? 1u : 0u);
          if (npass > 1) {
            mma_bf16(tmem, a_hi + step, b_lo + step, P.idesc, 1u);
            mma_bf16(tmem, a_lo + step, b_hi + step, P.idesc, 1u);
          }
        }
        mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
      }
      mma_commit(done);
    }
  } else {
    // ---- X producers: the tile's node rows chunk by chunk (from the bulk-landed fp32 rows, or
    // gathered with loads through the per-node offset table), split into bf16 hi / lo in the
    // canonical layout.  One unit = 8 consecutive K of one node.
    const int gt = tid - 64;
    const int kb = KC >> 3;
    const int units = P.NT * kb;
    for (int i = 0; i < cpr; ++i) {
      const int c = c_begin + i, s = i % S;
      if (P.bulk_x) mbar_wait(&full_w[s], (i / S) & 1);
      else if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      const float* raw = reinterpret_cast<const float*>(ring + s * stage_bytes + wstage);
      uint8_t* xs = ring + s * stage_bytes + wstage + rawbytes;
      for (int idx = gt; idx < units; idx += kGatherWarps * 32) {
        const int n = idx / kb;
        const int kk = (idx - n * kb) << 3;
        const int k = c * KC + kk;
        float v[8];
        if (n < nn && P.bulk_x) {
          const float4 a = *reinterpret_cast<const float4*>(raw + n * KC + kk);
          const float4 bq = *reinterpret_cast<const float4*>(raw + n * KC + kk + 4);
          v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = bq.x; v[5] = bq.y; v[6] = bq.z; v[7] = bq.w;
        } else if (n < nn) {
          const int pc = (P.npieces > 1 && k >= P.piece_k[0]) ? 1 : 0;
          const int kin = k - (pc ? P.piece_k[0] : 0);
          const float* src = P.arena + rowbase[2 * n + pc] + kin;
          if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(src));
            const float4 bq = __ldg(reinterpret_cast<const float4*>(src) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = bq.x; v[5] = bq.y; v[6] = bq.z; v[7] = bq.w;
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(src + q);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = 0.0f;
        }
        const uint32_t off = canon_off(n, kk, KC);
        float h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) h[q] = __bfloat162float(__float2bfloat16_rn(v[q]));
        uint4 hi;
        hi.x = pack_bf16(h[0], h[1]); hi.y = pack_bf16(h[2], h[3]); hi.z = pack_bf16(h[4], h[5]); hi.w = pack_bf16(h[6], h[7]);
        *reinterpret_cast<uint4*>(xs + off) = hi;
        if (npass > 1) {
          uint4 lo;
          lo.x = pack_bf16(v[0] - h[0], v[1] - h[1]);
          lo.y = pack_bf16(v[2] - h[2], v[3] - h[3]);
          lo.z = pack_bf16(v[4] - h[4], v[5] - h[5]);
          lo.w = pack_bf16(v[6] - h[6], v[7] - h[7]);
          *reinterpret_cast<uint4*>(xs + xchunk + off) = lo;
        }
      }
      fence_async_smem();  // make the generic-proxy stores visible to the tensor core (async proxy)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full_x[s])) : "memory");
    }
  }
  // Accumulator complete once every MMA has retired.
  mbar_wait(done, 0);
  if (tid == 0) stamp(P, 2);
  tc_fence_after();

  // TMEM -> smem: warp w reads lanes 32*(w%4).. (gate rows) for half of the node columns.
  {
    const int q = warp & 3, half = warp >> 2;
    const int row = q * 32 + lane;
    const int cols = P.NT / 2;
    for (int c0 = half * cols; c0 < (half + 1) * cols; c0 += 8) {
      float v[8];
      tmem_ld8(tmem + (uint32_t(q * 32) << 16) + uint32_t(c0), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) dsm[(c0 + k) * P.M + row] = v[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
  if (tid == 0) stamp(P, 3);

  // Epilogue scratch (the ring is free now): program | slots | prefetched operands | D rows.
  const int ntr = P.NT / ksplit;        // nodes this rank finishes
  const int nloc0 = int(rank) * ntr;    // first of them, within the tile
  const int nloc = max(0, min(ntr, nn - nloc0));
  const int E = ntr * P.UC;
  EpiProg* prog = reinterpret_cast<EpiProg*>(smem);
  float* slots = reinterpret_cast<float*>(smem + sizeof(EpiProg));
  float* srcbuf = slots + P.epi_nslots * kTcThreads;
  float* red = srcbuf + P.epi_nloads * E;
  for (int i = tid; i < int(sizeof(EpiProg) / 4); i += kTcThreads)
    reinterpret_cast<int*>(prog)[i] = reinterpret_cast<const int*>(P.epi)[i];

  // Split-K: every rank's partial D is complete in its smem; rank r sums node columns
  // [r*ntr, (r+1)*ntr) over the cluster in rank order (deterministic) via DSMEM.
  if (ksplit > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (tid == 0) stamp(P, 5);
    const uint32_t dsm_local = smem_u32(dsm);
    for (int i = tid; i < ntr * P.M; i += kTcThreads) {
      const int n = nloc0 + i / P.M, row = i % P.M;
      const uint32_t off = uint32_t((n * P.M + row) * 4);
      float acc = 0.0f;
      for (int q = 0; q < ksplit; ++q) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(dsm_local + off), "r"(q));
        float v;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
        acc += v;
      }
      red[i] = acc;
    }
    // Peers may still be reading this CTA's partial: keep it alive until everyone is done.
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
    red = dsm;
  }
  __syncthreads();
  if (tid == 0) stamp(P, 6);

  // Prefetch every batched / shared operand the tail reads, all elements at once (one round of
  // independent loads instead of a dependent chain per element).
  const int nops = prog->nops;
  for (int i = tid; i < prog->nloads * E; i += kTcThreads) {
    const int j = i / E, e = i - j * E;
    const int n = e / P.UC, u = e - n * P.UC;
    float v = 0.0f;
    if (n < nloc) {
      const EpiSrc& s = prog->loads[j];
      const int ug = tile_u * P.UC + u;
      const int64_t node = node0 + nloc0 + n;
      v = s.type == kSrcBatched ? P.arena[P.batched_off[node * P.nb + s.idx] + s.off + ug]
                                : P.arena[P.shared_off[s.idx] + s.off + ug];
    }
    srcbuf[i] = v;
  }
  __syncthreads();
  if (tid == 0) stamp(P, 7);

  // Elementwise tail as a micro-op program per (node, unit) element.
  for (int e = tid; e < nloc * P.UC; e += kTcThreads) {
    const int n = e / P.UC, u = e - n * P.UC;
    const int ug = tile_u * P.UC + u;
    const int64_t node = node0 + nloc0 + n;
    auto fetch = [&](const EpiSrc& s) -> float {
      switch (s.type) {
        case kSrcSlot: return slots[s.idx * kTcThreads + tid];
        case kSrcAcc: return red[n * P.M + s.idx * P.UC + u];
        case kSrcLoad: return srcbuf[s.idx * E + e];
        default: return 0.0f;
      }
    };
    for (int i = 0; i < nops; ++i) {
      const EpiOp& o = prog->ops[i];
      const float a = fetch(o.a);
      const float bv = fetch(o.b);
      float r;
      switch (o.op) {
        case kAdd: r = a + bv; break;
        case kMul: r = a * bv; break;
        case kSigmoid: r = 1.0f / (1.0f + __expf(-a)); break;
        case kTanh: r = 1.0f - 2.0f / (__expf(2.0f * a) + 1.0f); break;
        case kRelu: r = a > 0.0f ? a : 0.0f; break;
        default: r = a; break;  // copy
      }
      slots[o.dst * kTcThreads + tid] = r;
    }
    for (int k = 0; k < prog->nout; ++k)
      P.arena[P.out_base[k] + node * P.U + ug] = slots[prog->out_slot[k] * kTcThreads + tid];
  }
  if (P.ts) {
    __syncthreads();
    if (tid == 0) stamp(P, 4);
  }
}

struct PwArgs {
  const EpiProg* epi;
  float* arena;
  const int64_t* shared_off;
  const int64_t* batched_off;
  const int64_t* out_base;
  int b, E, nb, nslots;
};

// One thread per (node, element) of a pointwise plan; slots in shared memory, one column per
// thread; glibc-exact activations (bit-identical to the reference).
__global__ void __launch_bounds__(256) pointwise_kernel(PwArgs P) {
  extern __shared__ float pw_slots[];
  __shared__ EpiProg prog;
  for (int i = threadIdx.x; i < int(sizeof(EpiProg) / 4); i += blockDim.x)
    reinterpret_cast<int*>(&prog)[i] = reinterpret_cast<const int*>(P.epi)[i];
  __syncthreads();
  const int tid = threadIdx.x;
  const int64_t total = int64_t(P.b) * P.E;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + tid; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t node = idx / P.E;
    const int e = int(idx - node * P.E);
    auto fetch = [&](const EpiSrc& s) -> float {
      if (s.type == kSrcSlot) return pw_slots[s.idx * 256 + tid];
      if (s.type != kSrcLoad) return 0.0f;
      const EpiSrc& l = prog.loads[s.idx];
      const int64_t base = l.type == kSrcBatched ? P.batched_off[node * P.nb + l.idx] : P.shared_off[l.idx];
      return P.arena[base + l.off + e];
    };
    for (int i = 0; i < prog.nops; ++i) {
      const EpiOp& o = prog.ops[i];
      const float a = fetch(o.a);
      const float bv = fetch(o.b);
      pw_slots[o.dst * 256 + tid] = o.op == kOpCopy ? a : apply_op(o.op, a, bv);
    }
    for (int k = 0; k < prog.nout; ++k) P.arena[P.out_base[k] + node * P.E + e] = pw_slots[prog.out_slot[k] * 256 + tid];
  }
}

// Packs G weights (each K x U fp32, row-major, in the arena) into per-unit-tile, per-chunk
// canonical K-major bf16 blocks: [tile][chunk][pass][M x KC].  Rows g*UC + j of tile t hold column
// t*UC + j of weight g; rows >= G*UC are zero.
__global__ void tc_pack_kernel(const float* arena, const int64_t* w_off, int G, int K, int U, int UC, int M, int KC,
                               int npass, uint8_t* out) {
  const int nchunks = K / KC;
  const int ntiles = U / UC;
  const int64_t total = int64_t(ntiles) * nchunks * M * KC;
  const int64_t chunk_bytes = int64_t(M) * KC * 2;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int kk = int(idx % KC);
    int64_t r1 = idx / KC;
    const int r = int(r1 % M);
    r1 /= M;
    const int c = int(r1 % nchunks);
    const int t = int(r1 / nchunks);
    float v = 0.0f;
    if (r < G * UC) {
      const int g = r / UC, col = t * UC + r % UC, k = c * KC + kk;
      v = arena[w_off[g] + int64_t(k) * U + col];
    }
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const float lo = v - __bfloat162float(h);
    uint8_t* blk = out + ((int64_t(t) * nchunks + c) * (npass > 1 ? 2 : 1)) * chunk_bytes;
    const uint32_t off = uint32_t((r >> 3) * (KC * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
    *reinterpret_cast<__nv_bfloat16*>(blk + off) = h;
    if (npass > 1) *reinterpret_cast<__nv_bfloat16*>(blk + chunk_bytes + off) = __float2bfloat16_rn(lo);
  }
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Host side

namespace {

struct TcState {
  int K = 0, KC = 0, nchunks = 0, U = 0, G = 0, UC = 0, M = 0, dstep = 0;
  int npieces = 0;
  int piece_kind[2] = {0, 0}, piece_idx[2] = {0, 0}, piece_off[2] = {0, 0}, piece_k[2] = {0, 0};
  std::vector<int> w_shared;  // shared-input index of each weight
  EpiProg prog{};
  EpiProg* dprog = nullptr;   // device copy
  // packed-weight cache: (weight offsets, precision) -> device buffer
  struct Packed {
    std::vector<int64_t> offs;
    int npass = 0;
    uint64_t epoch = 0;
    uint8_t* buf = nullptr;
  };
  std::vector<Packed> packs;
};

// Compiles the plan's steps after the contraction into micro-ops over per-element slots.  A step
// s gets slot s - dstep - 1; the contraction's own columns are read from the accumulator tile.
bool compile_epilogue(const mbatch::backend::ExecutablePlan& p, TcState& st) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  EpiProg& pr = st.prog;
  pr = EpiProg{};
  const int dstep = st.dstep;
  auto src = [&](const PlanRef& r) {
    EpiSrc s{};
    const int slice = r.cols >= 0 ? r.col_off : 0;
    if (r.kind == PlanRef::Kind::kTemp) {
      if (r.index == dstep) {
        s.type = kSrcAcc;
        s.idx = int16_t(slice / st.U);
      } else {
        s.type = kSrcSlot;
        s.idx = int16_t(r.index - dstep - 1);
      }
    } else {
      // Input rows are prefetched once per element: dedupe them into the load table.
      EpiSrc l{};
      l.type = r.kind == PlanRef::Kind::kBatched ? kSrcBatched : kSrcShared;
      l.idx = int16_t(r.index);
      l.off = slice;
      int j = 0;
      while (j < pr.nloads && !(pr.loads[j].type == l.type && pr.loads[j].idx == l.idx && pr.loads[j].off == l.off)) ++j;
      if (j == pr.nloads) {
        if (pr.nloads >= kMaxLoads) {
          s.type = kSrcNone;  // too many distinct inputs: rejected below
          return s;
        }
        pr.loads[pr.nloads++] = l;
      }
      s.type = kSrcLoad;
      s.idx = int16_t(j);
    }
    return s;
  };
  auto push = [&](int op, int dst, EpiSrc a, EpiSrc b) {
    if (pr.nops >= int(sizeof(pr.ops) / sizeof(pr.ops[0]))) return false;
    pr.ops[pr.nops++] = EpiOp{op, dst, a, b};
    return true;
  };
  const int nsteps = int(p.steps.size());
  pr.nslots = nsteps - dstep - 1;
  for (int s = dstep + 1; s < nsteps; ++s) {
    const PlanStep& ps = p.steps[s];
    const int dst = s - dstep - 1;
    if (ps.kind == PlanStep::Kind::kChain) {
      if (ps.chain.empty()) {
        if (!push(kOpCopy, dst, src(ps.ins[0]), EpiSrc{})) return false;
        continue;
      }
      for (size_t l = 0; l < ps.chain.size(); ++l) {
        EpiSrc a = l == 0 ? src(ps.ins[0]) : EpiSrc{kSrcSlot, 0, int16_t(dst), 0};
        EpiSrc b = ps.chain[l].rhs ? src(*ps.chain[l].rhs) : EpiSrc{};
        if (!push(int(ps.chain[l].op), dst, a, b)) return false;
      }
    } else {
      if (!push(int(ps.op), dst, src(ps.ins[0]), ps.ins.size() > 1 ? src(ps.ins[1]) : EpiSrc{})) return false;
    }
  }
  pr.nout = int(p.outputs.size());
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& o = p.outputs[k];
    if (o.kind != PlanRef::Kind::kTemp) return false;
    if (o.index == dstep) {  // the contraction itself is an output: copy it into a fresh slot
      const int dst = pr.nslots++;
      if (!push(kOpCopy, dst, src(o), EpiSrc{})) return false;
      pr.out_slot[k] = dst;
    } else {
      pr.out_slot[k] = o.index - dstep - 1;
    }
  }
  for (int i = 0; i < pr.nops; ++i)
    if (pr.ops[i].a.type == kSrcNone && pr.ops[i].op != kOpCopy) return false;
  return pr.nslots <= 32 && pr.nloads < kMaxLoads;
}

bool analyse(const mbatch::backend::ExecutablePlan& p, const DPlan& d, TcState& st) {
  using mbatch::backend::OpCode;
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  if (p.ghost || d.unit <= 0 || p.steps.empty()) return false;
  int dstep = -1;
  for (size_t s = 0; s < p.steps.size(); ++s) {
    const PlanStep& ps = p.steps[s];
    const bool dense = ps.kind == PlanStep::Kind::kFusedDense || (ps.kind == PlanStep::Kind::kOp && ps.op == OpCode::kDense);
    if (dense) {
      if (dstep >= 0) return false;  // one contraction per plan
      dstep = int(s);
    }
  }
  if (dstep < 0 || dstep > 1) return false;
  const PlanStep& D = p.steps[dstep];
  if (!d.steps[dstep].split || D.out_shape.rows != 1) return false;
  // A row: either a direct S/B ref or step 0 = concat of two S/B refs.
  const PlanRef& a = D.ins[0];
  auto width = [&](const PlanRef& r) {
    if (r.cols >= 0) return r.cols;
    return r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index].cols : p.batched_shapes[r.index].cols;
  };
  auto rows_of = [&](const PlanRef& r) {
    return r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index].rows : p.batched_shapes[r.index].rows;
  };
  std::vector<PlanRef> pieces;
  if (dstep == 1) {
    const PlanStep& c = p.steps[0];
    if (!(c.kind == PlanStep::Kind::kOp && c.op == OpCode::kConcat)) return false;
    if (!(a.kind == PlanRef::Kind::kTemp && a.index == 0 && a.cols < 0)) return false;
    pieces = {c.ins[0], c.ins[1]};
  } else {
    if (a.kind == PlanRef::Kind::kTemp) return false;
    pieces = {a};
  }
  bool any_batched = false;
  int k0 = 0;
  st.npieces = int(pieces.size());
  for (size_t i = 0; i < pieces.size(); ++i) {
    const PlanRef& r = pieces[i];
    if (r.kind == PlanRef::Kind::kTemp || rows_of(r) != 1) return false;
    any_batched = any_batched || r.kind == PlanRef::Kind::kBatched;
    const int w = width(r);
    if (w % 8 != 0 || (r.cols >= 0 && r.col_off % 4 != 0)) return false;
    st.piece_kind[i] = r.kind == PlanRef::Kind::kShared ? kRefShared : kRefBatched;
    st.piece_idx[i] = r.index;
    st.piece_off[i] = r.cols >= 0 ? r.col_off : 0;
    k0 += w;
    st.piece_k[i] = k0;
  }
  if (!any_batched) return false;  // all-shared contractions are hoisted, not batched
  st.K = k0;
  const int U = d.unit;
  st.U = U;
  st.w_shared.clear();
  for (size_t w = 1; w < D.ins.size(); ++w) {
    if (D.ins[w].kind != PlanRef::Kind::kShared || D.ins[w].cols >= 0) return false;
    const auto& sh = p.shared_shapes[D.ins[w].index];
    if (sh.rows != st.K || sh.cols != U) return false;
    st.w_shared.push_back(D.ins[w].index);
  }
  st.G = int(st.w_shared.size());
  if (st.G < 1 || st.G > 4) return false;
  st.UC = std::min(U, 128 / st.G);
  if (U % st.UC != 0 || st.UC % 8 != 0 || st.G * st.UC < 64) return false;
  // Always M = 128 (rows past G*UC are zero-padded): with M = 128 accumulator row r sits in TMEM
  // lane r, which the epilogue relies on (M = 64 uses a different lane map).
  st.M = 128;
  st.KC = st.K % 64 == 0 ? 64 : st.K % 32 == 0 ? 32 : st.K % 16 == 0 ? 16 : 0;
  if (!st.KC) return false;
  st.nchunks = st.K / st.KC;
  // Tail: every step after the contraction must be a split elementwise step that never reads
  // steps before the contraction; at most kMaxEpi of them.
  if (int(p.steps.size()) - dstep - 1 > kMaxEpi) return false;
  for (size_t s = dstep + 1; s < p.steps.size(); ++s) {
    if (!d.steps[s].split) return false;
    const PlanStep& ps = p.steps[s];
    std::vector<PlanRef> refs = ps.ins;
    for (auto& l : ps.chain)
      if (l.rhs) refs.push_back(*l.rhs);
    for (auto& r : refs)
      if (r.kind == PlanRef::Kind::kTemp && r.index < dstep) return false;
  }
  for (int k = 0; k < d.nout; ++k)
    if (!d.out_split[k]) return false;
  st.dstep = dstep;
  return compile_epilogue(p, st);
}

// Tiling of one launch: NT nodes per CTA (the MMA N) and S K-split ranks per tile.  Each CTA
// ingests W_tile/S of weights (+ its node rows) through a per-SM pipe measured at ~110 GB/s
// (tools/bench_bulk.cu), node tiles multiply the L2 weight traffic, and S > 1 adds a DSMEM
// reduction.  A small cost model picks the cheapest tiling that fits one wave of 148 SMs.
// MBX_TC_NT / MBX_TC_KSPLIT force a choice (tuning).
struct Tiling {
  int NT = 16, S = 1;
};

Tiling pick_tiling(int b, int utiles, int nchunks, int K, int KC, int npass) {
  static const int forced_nt = [] {
    const char* e = std::getenv("MBX_TC_NT");
    return e ? std::atoi(e) : 0;
  }();
  static const int forced_s = [] {
    const char* e = std::getenv("MBX_TC_KSPLIT");
    return e ? std::atoi(e) : 0;
  }();
  const double wpass = npass > 1 ? 2 : 1;
  const double w_tile_bytes = 128.0 * K * 2 * wpass;  // one unit tile's weights
  Tiling best;
  double best_t = 1e30;
  for (int nt : {16, 32, 64, 128}) {
    if (forced_nt && nt != forced_nt) continue;
    if (nt > 16 && nt / 2 >= b) continue;  // do not over-pad small batches
    for (int s : {1, 2, 4, 8}) {
      if (forced_s && s != forced_s) continue;
      if (nchunks % s != 0 || nt % s != 0) continue;
      const int tiles = (b + nt - 1) / nt;
      const int ctas = tiles * utiles * s;
      if (ctas > 148 && !(forced_nt || forced_s)) continue;
      const double ingest_us = (w_tile_bytes / s + double(nt) * K / s * 4) / 110e3;
      const double mma_us = double(nchunks / s) * (KC / 16) * npass * std::max(16, nt / 2) / 1.9e3;
      const double l2_us = tiles * w_tile_bytes * utiles / 16e6;
      const double red_us = s > 1 ? (s - 1) * double(nt / s) * 128 * 4 / 20.0 / 1.9e3 : 0.0;
      const double epi_us = double(nt / s) * 32 / 256 * 0.05;
      const double t = 2.0 + std::max(std::max(ingest_us, mma_us), l2_us) + red_us + epi_us;
      if (t < best_t) {
        best_t = t;
        best.NT = nt;
        best.S = s;
      }
    }
  }
  return best;
}

}  // namespace

// Pointwise plans: every step elementwise over one common shape (the hoisted TreeLSTM leaf cell,
// MV-RNN's matrix add, ...).  They run one thread per (node, element) through the micro-op
// program with the glibc-exact activations, so they stay bit-identical to the reference.
bool analyse_pointwise(const mbatch::backend::ExecutablePlan& p, TcState& st) {
  using mbatch::backend::OpCode;
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  using mbatch::backend::Shape;
  if (p.ghost || p.steps.empty() || p.outputs.empty()) return false;
  const Shape sh = p.steps[0].out_shape;
  for (const auto& ps : p.steps) {
    if (ps.out_shape != sh) return false;
    if (ps.kind == PlanStep::Kind::kFusedDense) return false;
    if (ps.kind == PlanStep::Kind::kOp && !mbatch::backend::is_elementwise(ps.op)) return false;
    std::vector<PlanRef> refs = ps.ins;
    for (auto& l : ps.chain)
      if (l.rhs) refs.push_back(*l.rhs);
    for (auto& r : refs) {
      if (r.kind == PlanRef::Kind::kTemp) {
        if (r.cols >= 0) return false;
        continue;
      }
      const Shape in = r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index] : p.batched_shapes[r.index];
      if (r.cols >= 0 ? !(sh.rows == 1 && r.cols == sh.cols) : !(in == sh)) return false;
    }
  }
  for (auto& o : p.outputs)
    if (o.kind != PlanRef::Kind::kTemp || o.cols >= 0) return false;
  st.dstep = -1;
  st.U = sh.size();
  st.K = 0;
  return compile_epilogue(p, st);
}

void tc_prepare(mbx_ctx* c, PlanEntry& pe) {
  pe.tc_kind = -1;
  auto st = std::make_unique<TcState>();
  if (!analyse(pe.exec_plan, pe.hplan, *st)) {
    *st = TcState{};
    if (!analyse_pointwise(pe.exec_plan, *st)) return;
    pe.tc_kind = 2;
    if (!c->dry) {
      cuda_check(cudaMalloc(&st->dprog, sizeof(EpiProg)), "pointwise program");
      cuda_check(cudaMemcpy(st->dprog, &st->prog, sizeof(EpiProg), cudaMemcpyHostToDevice), "pointwise program");
    }
    pe.tc_state = st.release();
    return;
  }
  if (!c->dry) {
    cuda_check(cudaMalloc(&st->dprog, sizeof(EpiProg)), "epilogue program");
    cuda_check(cudaMemcpy(st->dprog, &st->prog, sizeof(EpiProg), cudaMemcpyHostToDevice), "epilogue program");
  }
  pe.tc_kind = 1;
  pe.tc_state = st.release();
}

void tc_release(PlanEntry& pe) {
  auto* st = static_cast<TcState*>(pe.tc_state);
  if (!st) return;
  for (auto& p : st->packs) cudaFree(p.buf);
  if (st->dprog) cudaFree(st->dprog);
  delete st;
  pe.tc_state = nullptr;
}

cudaError_t tc_launch(mbx_ctx* c, const PlanEntry& pe, const BatchLaunch& L) {
  auto* st = static_cast<TcState*>(pe.tc_state);
  if (pe.tc_kind == 2) {
    PwArgs a{};
    a.epi = st->dprog;
    a.arena = arena_ptr(c);
    a.shared_off = meta_dev<int64_t>(c, L.shared_meta);
    a.batched_off = meta_dev<int64_t>(c, L.batched_meta);
    a.out_base = meta_dev<int64_t>(c, L.out_meta);
    a.b = L.b;
    a.E = st->U;
    a.nb = int(pe.exec_plan.batched_shapes.size());
    a.nslots = st->prog.nslots;
    const int64_t total = int64_t(L.b) * a.E;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8)));
    const int smem = a.nslots * 256 * 4;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(pointwise_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    pointwise_kernel<<<blocks, 256, smem, c->stream>>>(a);
    return cudaGetLastError();
  }
  const int npass = c->precision == MBX_PREC_BF16 ? 1 : 3;
  const int wpass = npass > 1 ? 2 : 1;
  // Resolve the shared offsets of the weights (host copy of the staged shared table).
  const int64_t* shared_host = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
  std::vector<int64_t> offs;
  for (int w : st->w_shared) offs.push_back(shared_host[w]);
  TcState::Packed* pk = nullptr;
  for (auto& p : st->packs)
    if (p.offs == offs && p.npass == npass && p.epoch == c->upload_epoch) pk = &p;
  const int ntiles = st->U / st->UC;
  const size_t chunk_bytes = size_t(st->M) * st->KC * 2;
  const size_t pack_bytes = size_t(ntiles) * st->nchunks * wpass * chunk_bytes;
  if (!pk) {
    // (Re)pack: weights changed (new offsets or a host upload since the last pack).
    for (auto it = st->packs.begin(); it != st->packs.end(); ++it)
      if (it->offs == offs && it->npass == npass) {
        cudaFree(it->buf);
        st->packs.erase(it);
        break;
      }
    TcState::Packed p;
    p.offs = offs;
    p.npass = npass;
    p.epoch = c->upload_epoch;
    cudaError_t e = cudaMalloc(&p.buf, pack_bytes);
    if (e != cudaSuccess) return e;
    int64_t* d_off = nullptr;
    e = cudaMallocAsync(&d_off, offs.size() * 8, c->stream);
    if (e != cudaSuccess) return e;
    cudaMemcpyAsync(d_off, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, c->stream);
    const int64_t total = int64_t(ntiles) * st->nchunks * st->M * st->KC;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
    tc_pack_kernel<<<blocks, 256, 0, c->stream>>>(arena_ptr(c), d_off, st->G, st->K, st->U, st->UC, st->M, st->KC,
                                                   npass, p.buf);
    cudaFreeAsync(d_off, c->stream);
    ++c->launches;
    st->packs.push_back(p);
    pk = &st->packs.back();
  }
  TcArgs a{};
  a.epi = st->dprog;
  a.plan = pe.dplan;
  a.arena = arena_ptr(c);
  a.shared_off = meta_dev<int64_t>(c, L.shared_meta);
  a.batched_off = meta_dev<int64_t>(c, L.batched_meta);
  a.out_base = meta_dev<int64_t>(c, L.out_meta);
  a.wpack = pk->buf;
  a.b = L.b;
  a.K = st->K;
  a.KC = st->KC;
  a.nchunks = st->nchunks;
  a.U = st->U;
  a.G = st->G;
  a.UC = st->UC;
  a.M = st->M;
  const Tiling tl = pick_tiling(L.b, ntiles, st->nchunks, st->K, st->KC, npass);
  a.NT = tl.NT;
  a.ksplit = tl.S;
  a.epi_nslots = st->prog.nslots;
  a.epi_nloads = st->prog.nloads;
  a.npass = npass;
  a.dstep = st->dstep;
  a.nb = int(pe.plan.batched_shapes.size());
  a.npieces = st->npieces;
  for (int i = 0; i < 2; ++i) {
    a.piece_kind[i] = st->piece_kind[i];
    a.piece_idx[i] = st->piece_idx[i];
    a.piece_off[i] = st->piece_off[i];
    a.piece_k[i] = st->piece_k[i];
  }
  // Instruction descriptor: kind::f16, A = B = BF16 (1), D = F32 (1), both K-major, N>>3, M>>4.
  a.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a.NT >> 3) << 17) | (uint32_t(a.M >> 4) << 24);
  a.x_bytes = a.NT * a.K * 2;
  a.w_chunk_bytes = int(chunk_bytes);
  a.tmem_cols = a.NT < 32 ? 32 : a.NT;
  const int wstage = a.w_chunk_bytes * wpass;
  const int dsm_bytes = a.NT * a.M * 4;
  // Row gather by bulk copy needs every row segment 16-byte aligned.
  {
    bool ok = true;
    const int64_t* bat = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
    const int nb = int(pe.exec_plan.batched_shapes.size());
    for (int pc = 0; pc < st->npieces; ++pc) {
      ok = ok && st->piece_off[pc] % 4 == 0 && st->piece_k[pc] % 4 == 0;
      if (st->piece_kind[pc] == kRefShared) ok = ok && shared_host[st->piece_idx[pc]] % 4 == 0;
      else
        for (int i = 0; i < L.b && ok; ++i) ok = bat[int64_t(i) * nb + st->piece_idx[pc]] % 4 == 0;
    }
    a.bulk_x = ok ? 1 : 0;
    static const int dbg = [] {
      const char* e = std::getenv("MBX_TC_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    a.debug = dbg;
    if (dbg & 4) a.bulk_x = 0;
    static unsigned long long* ts = nullptr;
    if (dbg & 16) {
      static unsigned long long* dts = nullptr;
      if (!ts) {
        ts = static_cast<unsigned long long*>(std::calloc(64, 8));
        cudaMalloc(&dts, 64 * 8);
        cudaMemset(dts, 0, 64 * 8);
      }
      a.ts = dts;
      // Print the previous launch's phase stamps (this call is serialized behind it anyway).
      cudaStreamSynchronize(c->stream);
      cudaMemcpy(ts, dts, 64 * 8, cudaMemcpyDeviceToHost);
      std::fprintf(stderr,
                   "tc phases us: alloc %.2f mainloop %.2f tmem %.2f epilogue %.2f [cluster-wait %.2f reduce %.2f "
                   "prefetch %.2f tail %.2f] sm %.0f MHz\n",
                   (ts[1] - ts[0]) / 1e3, (ts[2] - ts[1]) / 1e3, (ts[3] - ts[2]) / 1e3, (ts[4] - ts[3]) / 1e3,
                   ts[5] ? (double(ts[5]) - ts[3]) / 1e3 : 0.0, ts[5] ? (double(ts[6]) - ts[5]) / 1e3 : 0.0,
                   (double(ts[7]) - ts[6]) / 1e3, (double(ts[4]) - ts[7]) / 1e3,
                   ts[4] > ts[0] ? double(ts[63] - ts[62]) / double(ts[4] - ts[0]) * 1e3 : 0.0);
      ts[5] = 0;
      cudaMemcpy(dts, ts, 64 * 8, cudaMemcpyHostToDevice);
      std::fprintf(stderr, "  chunk: W+raw landed / X converted / MMAs issued (us from start)\n");
      for (int k = 0; k < 16; ++k)
        std::fprintf(stderr, "  %2d %8.2f %8.2f %8.2f\n", k, (double(ts[24 + k]) - ts[0]) / 1e3,
                     (double(ts[40 + k]) - ts[0]) / 1e3, (double(ts[8 + k]) - ts[0]) / 1e3);
    }
  }
  const int xstage = a.NT * a.KC * 2 * wpass + (a.bulk_x ? a.NT * a.KC * 4 : 0);
  const int stage_bytes = wstage + xstage;
  const int ntr = a.NT / a.ksplit;
  const int epi_bytes = int(sizeof(EpiProg)) + st->prog.nslots * kTcThreads * 4 +
                        st->prog.nloads * ntr * st->UC * 4 + ntr * a.M * 4 + dsm_bytes;
  const int budget = 218 * 1024;
  const int cpr = st->nchunks / a.ksplit;
  a.stages = std::min(6, std::max(2, budget / stage_bytes));
  a.stages = std::min(a.stages, std::max(2, cpr));
  a.ring_bytes = std::max(a.stages * stage_bytes, (epi_bytes + 127) / 128 * 128);
  const int smem = a.ring_bytes + (3 * a.stages + 2) * 8 + a.NT * 2 * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_gate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(tc_gate_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((L.b + a.NT - 1) / a.NT, ntiles, a.ksplit);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = c->stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 1;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = unsigned(a.ksplit);
  cfg.attrs = attrs;
  cfg.numAttrs = a.ksplit > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, tc_gate_kernel, a);
}

}  // namespace mbx
