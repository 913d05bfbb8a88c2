// berxit.cu — the Berxit early-exit encoder on B200 (BASELINE configs[4]; ABI:
// include/mbx_berxit.h).  Parity unpinned: the reference has no Berxit (proj/src/zoo.cpp:305-317);
// the checker is oracle/berxit_oracle.cpp (the paper's model).
//
// ACRoBat batches this model per layer over the instances that have not exited.  Here that batch
// never leaves the device: `alive` (instance ids in instance order) and `count` live in HBM, the
// exit kernel of layer l writes layer l+1's list, and every kernel of a layer reads its tiles from
// that list (a gather by index array: an exited instance's rows stay where they are, nothing is
// compacted or copied).  One mini-batch = 2 + 7 L launches captured once per batch size as a CUDA
// graph; the host sees the results only.
//
// Per layer (all on one stream; instance rows [S = 128][.] stay at x[inst], the operand images at
// x_img[inst] etc.):
//   bx_gemm<QKV>     q/8, k, v^T images = x Wqkv^T + b        (tcgen05, A = x_img)
//   bx_attention     ctx_img = softmax(q k^T / 8) v per head  (tcgen05 on bulk-copied images)
//   bx_gemm<RESID>   y    = x + ctx Wo^T + b
//   bx_layernorm     x, x_img = LN1(y)
//   bx_gemm<GELU>    f_img = GELU(x W1^T + b)                 (the epilogue writes the A image)
//   bx_gemm<RESID>   y    = x + f W2^T + b
//   bx_layernorm     x, x_img = LN2(y); CLS rows: LTE certainty, logits of the exiting instances;
//                    the last CTA writes the next layer's running list (exit head fused)
//
// Operand images: every GEMM operand is stored by its producer as split bf16 (hi = rn(v),
// lo = rn(v - hi); one part in BF16 precision) in the canonical no-swizzle K-major UMMA layout,
// one 64-wide K chunk of one 128-row instance tile (16 KB per part) or of one 256-row weight tile
// (32 KB per part) contiguous, so a pipeline stage is two cp.async.bulk copies (A tile + W tile).
//
// bx_gemm: persistent (one CTA per SM, 192 KB of stages), tiles = (running instance, 256-column
// tile), M = 128 tokens x N = 256 x K chunk 64; warp 0 issues the bulk copies into a stage ring,
// warp 1 (one thread) issues tcgen05.mma (3 per K step in BF16X3: hi*hi + hi*lo + lo*hi) into one
// of two 256-column TMEM accumulators, warps 2-5 drain the other accumulator (tcgen05.ld) through
// the fused epilogue while the next tile's MMAs run.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "mbx.h"
#include "mbx_berxit.h"

namespace mbx {
extern std::atomic<int64_t> g_launches;
}

namespace bx {

typedef unsigned short bf16_t;

constexpr int kSeq = 128;       // rows of one instance tile (MMA M)
constexpr int kNT = 256;        // MMA N per tile
constexpr int kKC = 64;         // K chunk (elements)
constexpr int kABlock = kSeq * kKC;  // bf16 elements of one A chunk part (16 KB)
constexpr int kWBlock = kNT * kKC;   // bf16 elements of one W chunk part (32 KB)
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter, each draining half of a tile's columns
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kStageSmem = 192 * 1024;

enum Epi { EPI_PLAIN = 0, EPI_RESID = 1, EPI_GELU = 2, EPI_QKV = 3 };

// ---- device helpers ----------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Programmatic dependent launch: every kernel after the first of a mini-batch is launched while
// its predecessor runs; it sets up shared memory / TMEM, then waits here for the predecessor's
// completion (and memory) before touching anything in HBM, and lets its own successor launch.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// Canonical K-major no-swizzle descriptor: LBO 128 B (K-adjacent core matrices), SBO 1024 B
// (8-row groups of a 64-wide chunk), version 1.
__device__ __forceinline__ unsigned long long make_desc(unsigned saddr) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3FFF);
  d |= (unsigned long long)((128u >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((1024u >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  return d;
}
__device__ __forceinline__ void mma_bf16(unsigned tmem_d, unsigned long long a, unsigned long long b, unsigned idesc,
                                         unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(unsigned addr, float* v) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ unsigned short to_bf16(float x) {
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(x));
  return h;
}
__device__ __forceinline__ float from_bf16(unsigned short h) { return __uint_as_float(unsigned(h) << 16); }
// hi = rn(x), lo = rn(x - hi)
__device__ __forceinline__ void split2(float x, unsigned short& hi, unsigned short& lo) {
  hi = to_bf16(x);
  lo = to_bf16(x - from_bf16(hi));
}

// Element offset of (row r, k within the 64-wide chunk) in the canonical layout.
__device__ __forceinline__ int canon(int r, int kk) { return (r >> 3) * 512 + (kk >> 3) * 64 + (r & 7) * 8 + (kk & 7); }

// Writes n8 consecutive groups of 8 values (k = k0 .. k0 + 8 n8, k0 % 8 == 0) of row r of
// instance `inst` into an A image with kch chunks and P parts.
template <int N8>
__device__ __forceinline__ void store_img_row(bf16_t* img, int kch, int P, int inst, int r, int k0, const float* v) {
#pragma unroll
  for (int g = 0; g < N8; ++g) {
    const int k = k0 + 8 * g;
    unsigned hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      unsigned short h0, l0, h1, l1;
      split2(v[8 * g + 2 * e], h0, l0);
      split2(v[8 * g + 2 * e + 1], h1, l1);
      hi[e] = unsigned(h0) | (unsigned(h1) << 16);
      lo[e] = unsigned(l0) | (unsigned(l1) << 16);
    }
    const size_t base = ((size_t)inst * kch + (k >> 6)) * P * kABlock + canon(r, k & 63);
    *reinterpret_cast<uint4*>(img + base) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    if (P > 1) *reinterpret_cast<uint4*>(img + base + kABlock) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// ---- GEMM ---------------------------------------------------------------------------------------
struct GemmArgs {
  const bf16_t* a_img;  // [inst][kch][P][128 x 64]
  const bf16_t* w_img;  // [ntile][kch][P][256 x 64]
  const float* bias;    // [N]
  const float* resid;   // EPI_RESID: [inst][128][N]
  float* out;           // EPI_PLAIN / EPI_RESID: [inst][128][N]
  bf16_t* out_img;      // EPI_GELU: [inst][N/64][P][128 x 64]
  const int* alive;
  const int* count;
  int kch, N, P;
  int nt;  // tile width chosen on the host for the batch size (256, 128 or 64)
  // EPI_QKV: out_img = Q image (scaled by 1/8), k_img = K image ([inst][head][part][128 x 64],
  // i.e. A images with one chunk per head), vt_img = V^T image ([inst][head][key chunk][part][64 x 64])
  bf16_t* k_img;
  bf16_t* vt_img;
  int H;
};

// Fused epilogue of one accumulator tile: row r of instance `inst`, columns n0 .. n0 + NT; tm is
// the TMEM address of this warp's lane quarter at the tile's first column.
template <int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& g, unsigned tm, int inst, int n0, int NT, int r,
                                              int half) {
  const int P = g.P;
  const int ncc = NT / 64;  // 32-column groups per epilogue warp
#pragma unroll 1
  for (int cc = half * ncc; cc < (half + 1) * ncc; ++cc) {
    float v[32];
    tmem_ld32(tm + unsigned(cc * 32), v);
    const int col0 = n0 + cc * 32;
    const float4* b4 = reinterpret_cast<const float4*>(g.bias + col0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 b = __ldg(b4 + j);
      v[4 * j] += b.x;
      v[4 * j + 1] += b.y;
      v[4 * j + 2] += b.z;
      v[4 * j + 3] += b.w;
    }
    const size_t row = ((size_t)inst * kSeq + r) * g.N + col0;
    if (EPI == EPI_GELU) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu(v[j]);
      store_img_row<4>(g.out_img, g.N / kKC, P, inst, r, col0, v);
    } else if (EPI == EPI_QKV) {
      const int H = g.H, sec = col0 / H, c = col0 - sec * H;
      if (sec == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= 0.125f;  // 1 / sqrt(64), exact
        store_img_row<4>(g.out_img, H / kKC, P, inst, r, c, v);
      } else if (sec == 1) {
        store_img_row<4>(g.k_img, H / kKC, P, inst, r, c, v);
      } else {
        const int h = c >> 6, d0 = c & 63;
        bf16_t* vb = g.vt_img + (((size_t)inst * (H / 64) + h) * 2 + (r >> 6)) * P * 4096;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          unsigned short hi, lo;
          split2(v[j], hi, lo);
          const int e = canon(d0 + j, r & 63);
          vb[e] = hi;
          if (P > 1) vb[e + 4096] = lo;
        }
      }
    } else {
      if (EPI == EPI_RESID) {
        const float4* r4 = reinterpret_cast<const float4*>(g.resid + row);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 x = r4[j];
          v[4 * j] = x.x + v[4 * j];
          v[4 * j + 1] = x.y + v[4 * j + 1];
          v[4 * j + 2] = x.z + v[4 * j + 2];
          v[4 * j + 3] = x.w + v[4 * j + 3];
        }
      }
      float4* o4 = reinterpret_cast<float4*>(g.out + row);
#pragma unroll
      for (int j = 0; j < 8; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  }
}

template <int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1) bx_gemm(GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int P = g.P;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + kStageSmem);
  unsigned long long* full = bars;          // [S <= 8]
  unsigned long long* empty = bars + 8;     // [S <= 8]
  unsigned long long* acc_full = bars + 16; // [2]
  unsigned long long* acc_empty = bars + 18;  // [2]
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 32 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  pdl_wait_and_release();
  const int count = *g.count;
  // Tile width (MMA N: 256, 128 or 64, a row range of the weight image's 256-row tiles) for THIS
  // layer's running count, known only here: the smallest modelled makespan, ceil(tiles / CTAs) x
  // (width + per-tile cost) + the last tile's exposed epilogue (~3/4 width).  The width never
  // changes a column's accumulation order, only the parallelism.
  int NT = g.nt;
  if (count * (g.N / NT) < int(gridDim.x) / 2) {  // most CTAs idle at the host's width: narrow it
    int best = -1;
    for (int w = 256; w >= 64; w >>= 1) {
      const int tiles = count * (g.N / w), rounds = (tiles + gridDim.x - 1) / gridDim.x, cost = rounds * (w + 48) + 3 * w / 4;
      if (best < 0 || cost < best) best = cost, NT = w;
    }
  }
  const int ntiles = g.N / NT;
  const unsigned a_bytes = unsigned(P) * kABlock * 2, w_part = unsigned(NT) * 128, w_bytes = unsigned(P) * w_part;
  const unsigned stage_bytes = a_bytes + w_bytes;
  const int S = kStageSmem / int(stage_bytes);
  const int ntile_total = count * ntiles;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x) {
        const int inst = g.alive[t / ntiles], n0 = (t % ntiles) * NT;
        const bf16_t* a = g.a_img + (size_t)inst * g.kch * P * kABlock;
        // rows n0 .. n0 + NT of the 256-row image tile: a contiguous range of each part block
        const bf16_t* w = g.w_img + (size_t)(n0 / kNT) * g.kch * P * kWBlock + (n0 % kNT) * kKC;
        for (int c = 0; c < g.kch; ++c, ++it) {
          const int s = it % S;
          if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
          unsigned char* st = smem + s * stage_bytes;
          mbar_expect_tx(&full[s], stage_bytes);
          bulk_g2s(st, a + (size_t)c * P * kABlock, a_bytes, &full[s]);
          for (int p = 0; p < P; ++p)
            bulk_g2s(st + a_bytes + p * w_part, w + ((size_t)c * P + p) * kWBlock, w_part, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::f16: A = B = BF16, D = F32, both K-major, N = 256, M = 128.
      const unsigned idesc = (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(NT >> 3) << 17) | (unsigned(kSeq >> 4) << 24);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tc) {
        const int acc = tc & 1;
        if (tc >= 2) mbar_wait(&acc_empty[acc], ((tc >> 1) - 1) & 1);
        tc_fence_after();
        const unsigned d = tmem + unsigned(acc * kNT);
        for (int c = 0; c < g.kch; ++c, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const unsigned sa = smem_u32(smem + s * stage_bytes), sb = sa + a_bytes;
#pragma unroll
          for (int ks = 0; ks < kKC / 16; ++ks) {
            const unsigned long long ah = make_desc(sa + ks * 256), bh = make_desc(sb + ks * 256);
            mma_bf16(d, ah, bh, idesc, (c | ks) ? 1u : 0u);
            if (P > 1) {
              const unsigned long long al = make_desc(sa + kABlock * 2 + ks * 256);
              const unsigned long long bl = make_desc(sb + w_part + ks * 256);
              mma_bf16(d, ah, bl, idesc, 1u);
              mma_bf16(d, al, bh, idesc, 1u);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[acc]);
      }
    }
  } else {
    // ---- epilogue: warps 2..5, TMEM lane quarter q = warp % 4, row r = 32 q + lane ----
    const int q = warp & 3, r = 32 * q + lane;
    int tc = 0;
    for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tc) {
      const int acc = tc & 1;
      const int inst = g.alive[t / ntiles], n0 = (t % ntiles) * NT;
      mbar_wait(&acc_full[acc], (tc >> 1) & 1);
      tc_fence_after();
      epilogue_tile<EPI>(g, tmem + (unsigned(32 * q) << 16) + unsigned(acc * kNT), inst, n0, NT, r, (warp - 2) >> 2);
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---- attention: one CTA per (head, running instance) on tcgen05 ---------------------------------
// S = Q K^T (M = 128 queries, N = 128 keys, K = 64) and O = P V (M = 128, N = 64, K = 128 keys),
// split bf16 (3 products per K step in BF16X3) with fp32 TMEM accumulation; the softmax is fp32
// per query row (thread = row = TMEM lane).  Q (scaled by 1/8, exact), K and V^T are converted
// from qkv's fp32 rows straight into the canonical K-major layouts; P is written back as the A
// operand of the second product, over Q and K (dead once S is in TMEM).  Shared memory (bytes):
// Q [part] 16 K | K [part] 16 K (later P [key chunk][part] 16 K) | V^T [key chunk][part] 8 K
// = 96 K: two CTAs per SM.
constexpr int kAttSmem = 96 * 1024 + 64;

__device__ __forceinline__ void st_split4(unsigned char* base_hi, int lo_off, int e_off, float a, float b, float c,
                                          float d, int P) {
  unsigned short h[4], l[4];
  split2(a, h[0], l[0]);
  split2(b, h[1], l[1]);
  split2(c, h[2], l[2]);
  split2(d, h[3], l[3]);
  *reinterpret_cast<uint2*>(base_hi + 2 * e_off) =
      make_uint2(unsigned(h[0]) | (unsigned(h[1]) << 16), unsigned(h[2]) | (unsigned(h[3]) << 16));
  if (P > 1)
    *reinterpret_cast<uint2*>(base_hi + lo_off + 2 * e_off) =
        make_uint2(unsigned(l[0]) | (unsigned(l[1]) << 16), unsigned(l[2]) | (unsigned(l[3]) << 16));
}

__global__ void __launch_bounds__(128, 2) bx_attention(const bf16_t* q_img, const bf16_t* k_img,
                                                       const bf16_t* vt_img, bf16_t* ctx_img, const int* alive,
                                                       const int* count, int H, int P) {
  extern __shared__ __align__(1024) unsigned char asmem[];
  unsigned char* sQ = asmem;
  unsigned char* sK = asmem + 32768;
  unsigned char* sVT = asmem + 65536;
  unsigned char* sP = asmem;  // over Q and K
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(asmem + 98304);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(asmem + 98304 + 32);
  const int m = blockIdx.y, h = blockIdx.x;
  pdl_wait_and_release();
  if (m >= *count) return;
  const int inst = alive[m];
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // Q, K and V^T arrive MMA-ready from the QKV GEMM's epilogue: three bulk copies.
  if (t == 0) {
    const size_t qk = ((size_t)inst * (H / 64) + h) * P * 8192;  // elements
    const unsigned qb = unsigned(P) * 16384;
    mbar_expect_tx(&bar[2], 3 * qb);
    bulk_g2s(sQ, q_img + qk, qb, &bar[2]);
    bulk_g2s(sK, k_img + qk, qb, &bar[2]);
    bulk_g2s(sVT, vt_img + qk, qb, &bar[2]);
  }
  mbar_wait(&bar[2], 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  const unsigned idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(128 >> 3) << 17) | (unsigned(kSeq >> 4) << 24);
  const unsigned idesc_o = (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(64 >> 3) << 17) | (unsigned(kSeq >> 4) << 24);
  if (t == 0) {
    const unsigned q0 = smem_u32(sQ), k0 = smem_u32(sK);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const unsigned long long qh = make_desc(q0 + ks * 256), kh = make_desc(k0 + ks * 256);
      mma_bf16(tmem, qh, kh, idesc_s, ks ? 1u : 0u);
      if (P > 1) {
        mma_bf16(tmem, qh, make_desc(k0 + 16384 + ks * 256), idesc_s, 1u);
        mma_bf16(tmem, make_desc(q0 + 16384 + ks * 256), kh, idesc_s, 1u);
      }
    }
    mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  tc_fence_after();
  // softmax of row t: lanes 32 warp .. of TMEM = rows
  const unsigned lane_base = tmem + (unsigned(32 * warp) << 16);
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    float v[32];
    tmem_ld32(lane_base + unsigned(c * 32), v);
#pragma unroll
    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, v[j]);
  }
  float l = 0.f;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    float v[32];
    tmem_ld32(lane_base + unsigned(c * 32), v);
    unsigned char* pb = sP + (c >> 1) * 32768;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = expf(v[j] - mx);
      l += v[j];
    }
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      st_split4(pb, 16384, canon(t, (c & 1) * 32 + j), v[j], v[j + 1], v[j + 2], v[j + 3], P);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const unsigned p0 = smem_u32(sP), v0 = smem_u32(sVT);
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const unsigned pa = p0 + c * 32768 + ks * 256, vb = v0 + c * 16384 + ks * 256;
        const unsigned long long ph = make_desc(pa), vh = make_desc(vb);
        mma_bf16(tmem + 128, ph, vh, idesc_o, (c | ks) ? 1u : 0u);
        if (P > 1) {
          mma_bf16(tmem + 128, ph, make_desc(vb + 8192), idesc_o, 1u);
          mma_bf16(tmem + 128, make_desc(pa + 16384), vh, idesc_o, 1u);
        }
      }
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const float inv = 1.0f / l;
  float o[64];
  tmem_ld32(lane_base + 128, o);
  tmem_ld32(lane_base + 160, o + 32);
#pragma unroll
  for (int d = 0; d < 64; ++d) o[d] *= inv;
  store_img_row<8>(ctx_img, H / kKC, P, inst, t, h * 64, o);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
  }
}

// ---- layer norm: one warp per row; y -> x (fp32) and x_img ----------------------------------------
// With `ex.on` (LN2) the warp of each running instance's first row (CLS) also runs the exit head
// on the normalised row it holds in registers: certainty u = sigmoid(w_lte . h + b_lte); an exiting
// instance writes its logits and exit layer.  The last CTA to finish (counter) compacts the running
// list in instance order for the next layer and records this layer's batch in the schedule.
struct ExitArgs {
  int on;
  const float *w_lte, *b_lte, *wc, *bc;
  float* logits;
  int *exit_layer, *sched, *keep;
  unsigned* done;
  int* alive_w;  // == alive (written by the last CTA only)
  int* count_w;
  int C, layer, L, bmax;
  float tau;
};

__global__ void __launch_bounds__(256) bx_layernorm(const float* y, float* x, bf16_t* x_img, const float* gam,
                                                    const float* bet, const int* alive, const int* count, int H,
                                                    int P, float eps, ExitArgs ex) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int m = row / kSeq, r = row % kSeq;
  pdl_wait_and_release();
  const int n = *count;
  if (m < n) {
    const int inst = alive[m];
    const size_t off = ((size_t)inst * kSeq + r) * H;
    const int nv = H / 128;  // float4 per lane
    float4 v[8];
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nv) {
        v[j] = reinterpret_cast<const float4*>(y + off)[lane + 32 * j];
        sum += (v[j].x + v[j].y) + (v[j].z + v[j].w);
      }
#pragma unroll
    for (int s = 16; s; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
    const float mean = sum / float(H);
    float var = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nv) {
        const float a = v[j].x - mean, b = v[j].y - mean, c = v[j].z - mean, d = v[j].w - mean;
        var += (a * a + b * b) + (c * c + d * d);
      }
#pragma unroll
    for (int s = 16; s; s >>= 1) var += __shfl_xor_sync(0xffffffffu, var, s);
    const float inv = 1.0f / sqrtf(var / float(H) + eps);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nv) {
        const int k = 4 * (lane + 32 * j);
        const float4 g = __ldg(reinterpret_cast<const float4*>(gam + k));
        const float4 b = __ldg(reinterpret_cast<const float4*>(bet + k));
        float o[4] = {(v[j].x - mean) * inv * g.x + b.x, (v[j].y - mean) * inv * g.y + b.y,
                      (v[j].z - mean) * inv * g.z + b.z, (v[j].w - mean) * inv * g.w + b.w};
        v[j] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(x + off)[lane + 32 * j] = v[j];
        unsigned short hh[4], ll[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split2(o[e], hh[e], ll[e]);
        const size_t base = ((size_t)inst * (H / kKC) + (k >> 6)) * P * kABlock + canon(r, k & 63);
        *reinterpret_cast<uint2*>(x_img + base) =
            make_uint2(unsigned(hh[0]) | (unsigned(hh[1]) << 16), unsigned(hh[2]) | (unsigned(hh[3]) << 16));
        if (P > 1)
          *reinterpret_cast<uint2*>(x_img + base + kABlock) =
              make_uint2(unsigned(ll[0]) | (unsigned(ll[1]) << 16), unsigned(ll[2]) | (unsigned(ll[3]) << 16));
      }
    if (ex.on && r == 0) {
      auto wdot = [&](const float* w) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < nv) {
            const float4 c = __ldg(reinterpret_cast<const float4*>(w) + lane + 32 * j);
            a = fmaf(c.x, v[j].x, a);
            a = fmaf(c.y, v[j].y, a);
            a = fmaf(c.z, v[j].z, a);
            a = fmaf(c.w, v[j].w, a);
          }
#pragma unroll
        for (int s = 16; s; s >>= 1) a += __shfl_xor_sync(0xffffffffu, a, s);
        return a;
      };
      const float z = wdot(ex.w_lte) + ex.b_lte[0];
      const float u = 1.0f / (1.0f + expf(-z));
      const bool out = (u >= ex.tau) || ex.layer == ex.L - 1;
      if (out) {
        for (int c = 0; c < ex.C; ++c) {
          const float a = wdot(ex.wc + (size_t)c * H);
          if (lane == 0) ex.logits[(size_t)inst * ex.C + c] = a + ex.bc[c];
        }
        if (lane == 0) ex.exit_layer[inst] = ex.layer;
      }
      if (lane == 0) ex.keep[m] = out ? 0 : 1;
    }
  }
  if (!ex.on) return;
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ex.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    const volatile int* keep = ex.keep;
    int k = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int mm = b0 + lane;
      const int id = mm < n ? alive[mm] : -1;
      const bool kp = mm < n && keep[mm];
      if (mm < n) ex.sched[(size_t)ex.layer * ex.bmax + mm] = id;
      const unsigned bal = __ballot_sync(0xffffffffu, kp);
      if (kp) ex.alive_w[k + __popc(bal & ((1u << lane) - 1))] = id;
      k += __popc(bal);
    }
    if (lane == 0) {
      *ex.count_w = k;
      *ex.done = 0;
    }
  }
}

// ---- mini-batch start: alive = 0..b-1, count = b, schedule / exits reset; x -> x_img ---------
__global__ void bx_begin(int* alive, int* count, int* exit_layer, int* sched, int b, int bmax, int L) {
  for (int i = threadIdx.x; i < bmax; i += blockDim.x) {
    alive[i] = i;
    exit_layer[i] = -1;
  }
  for (int i = threadIdx.x; i < bmax * L; i += blockDim.x) sched[i] = -1;
  if (threadIdx.x == 0) *count = b;
}

__global__ void __launch_bounds__(256) bx_to_image(const float* x, bf16_t* x_img, int H, int P, int b) {
  // one thread per (instance, row, 8-column group)
  pdl_wait_and_release();
  const size_t g8 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t per_inst = (size_t)kSeq * (H / 8);
  if (g8 >= per_inst * b) return;
  const int inst = int(g8 / per_inst);
  const int rem = int(g8 % per_inst), r = rem / (H / 8), k0 = 8 * (rem % (H / 8));
  const float* src = x + ((size_t)inst * kSeq + r) * H + k0;
  float v[8];
  const float4 a = reinterpret_cast<const float4*>(src)[0], c = reinterpret_cast<const float4*>(src)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
  store_img_row<1>(x_img, H / kKC, P, inst, r, k0, v);
}

// Weight W [N][K] fp32 -> image [N/256][K/64][P][256 x 64] split bf16.
__global__ void bx_weight_image(const float* W, bf16_t* img, int N, int K, int P) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * K) return;
  const int n = int(e / K), k = int(e % K);
  const int kch = K / kKC;
  unsigned short hi, lo;
  split2(W[e], hi, lo);
  const size_t base = ((size_t)(n / kNT) * kch + k / kKC) * P * kWBlock + canon(n % kNT, k % kKC);
  img[base] = hi;
  if (P > 1) img[base + kWBlock] = lo;
}

// ---- host ----------------------------------------------------------------------------------------
void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda error in ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace bx

struct mbx_berxit {
  int device = 0, precision = MBX_PREC_BF16X3, P = 2, bmax = 0, sms = 148;
  mbx_berxit_config c{};
  cudaStream_t stream = nullptr;
  float* params = nullptr;  // flat fp32 parameters (device)
  bx::bf16_t *wqkv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;
  float *x = nullptr, *y = nullptr, *logits = nullptr;
  bx::bf16_t *q_img = nullptr, *k_img = nullptr, *vt_img = nullptr;
  bx::bf16_t *x_img = nullptr, *ctx_img = nullptr, *f_img = nullptr;
  int *alive = nullptr, *count = nullptr, *exit_layer = nullptr, *sched = nullptr, *keep = nullptr;
  float* wc_al = nullptr;    // 16-byte aligned copy of Wc
  unsigned* done = nullptr;  // CTA counter of the exit-fused layer norm (self-resetting)
  bool params_set = false;
  std::map<int, cudaGraphExec_t> graphs;
  std::string err;
  // parameter views (device)
  const float *bqkv, *bo, *g1, *be1, *b1, *b2, *g2, *be2, *wl, *bl, *wc, *bc;
};

namespace {

thread_local std::string g_bx_err;

template <class F>
int guarded(mbx_berxit* m, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    (m ? m->err : g_bx_err) = e.what();
  }
  return 1;
}

void validate(const mbx_berxit_config* c) {
  if (!c) throw std::runtime_error("null config");
  if (c->hidden <= 0 || c->heads <= 0 || c->ffn <= 0 || c->layers <= 0 || c->seq <= 0 || c->classes <= 0)
    throw std::runtime_error("berxit: sizes must be positive");
  if (c->hidden % c->heads) throw std::runtime_error("berxit: hidden must be a multiple of heads");
}

void validate_device(const mbx_berxit_config* c) {
  validate(c);
  if (c->seq != bx::kSeq) throw std::runtime_error("berxit: the device path needs seq == 128");
  if (c->hidden / c->heads != 64) throw std::runtime_error("berxit: the device path needs hidden / heads == 64");
  if (c->hidden % bx::kNT || c->ffn % bx::kNT) throw std::runtime_error("berxit: hidden and ffn must be multiples of 256");
  if (c->hidden > 1024) throw std::runtime_error("berxit: hidden > 1024 not supported by the layer-norm kernel");
}

inline float uni(std::mt19937& g, float lo, float hi) {
  return lo + (hi - lo) * (float(g() >> 8) * (1.0f / 16777216.0f));
}

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  bx::check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

// Launch with programmatic stream serialization (the kernel's pdl_wait_and_release orders it
// after its predecessor); captured into the mini-batch graph as programmatic edges.
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, int threads, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  bx::check(cudaLaunchKernelEx(&cfg, kernel, args...), "berxit launch");
}

void launch_gemm(mbx_berxit* m, int b, int epi, const bx::bf16_t* a_img, const bx::bf16_t* w_img, int K, int N,
                 const float* bias, const float* resid, float* out, bx::bf16_t* out_img) {
  // Tile width for a batch of b running instances: the smallest makespan ceil(tiles / SMs) x
  // (width + fixed per-tile cost) (BERT-base b64: 256 for QKV / W1, 128 for Wo / W2).  The kernel
  // narrows it when the layer's running count (known only on the device) leaves most CTAs idle.
  int nt = 256;
  long best = -1;
  for (int w : {256, 128, 64}) {
    const long tiles = (long)b * (N / w), rounds = (tiles + m->sms - 1) / m->sms, cost = rounds * (w + 48);
    if (best < 0 || cost < best) best = cost, nt = w;
  }
  bx::GemmArgs g{a_img, w_img, bias, resid, out, out_img, m->alive, m->count, K / bx::kKC, N, m->P, nt,
                 m->k_img, m->vt_img, m->c.hidden};
  const int grid = (int)std::min<long>(m->sms, (long)b * (N / 64));
  const size_t smem = bx::kStageSmem + 256;
  switch (epi) {
    case bx::EPI_PLAIN: launch_pdl(bx::bx_gemm<bx::EPI_PLAIN>, grid, bx::kGemmThreads, smem, m->stream, g); break;
    case bx::EPI_RESID: launch_pdl(bx::bx_gemm<bx::EPI_RESID>, grid, bx::kGemmThreads, smem, m->stream, g); break;
    case bx::EPI_GELU: launch_pdl(bx::bx_gemm<bx::EPI_GELU>, grid, bx::kGemmThreads, smem, m->stream, g); break;
    default: launch_pdl(bx::bx_gemm<bx::EPI_QKV>, grid, bx::kGemmThreads, smem, m->stream, g); break;
  }
  bx::check(cudaGetLastError(), "bx_gemm launch");
}

// Enqueues one mini-batch of b instances whose inputs are already in m->x.
void enqueue(mbx_berxit* m, int b) {
  const auto& c = m->c;
  const int H = c.hidden, F = c.ffn, L = c.layers, P = m->P;
  const size_t wp = 3 * (size_t)H * H;
  bx::bx_begin<<<1, 256, 0, m->stream>>>(m->alive, m->count, m->exit_layer, m->sched, b, m->bmax, L);
  const size_t groups = (size_t)b * bx::kSeq * (H / 8);
  launch_pdl(bx::bx_to_image, dim3(unsigned((groups + 255) / 256)), 256, 0, m->stream, (const float*)m->x, m->x_img, H,
             P, b);
  (void)wp;
  for (int l = 0; l < L; ++l) {
    launch_gemm(m, b, bx::EPI_QKV, m->x_img, m->wqkv, H, 3 * H, m->bqkv, nullptr, nullptr, m->q_img);
    launch_pdl(bx::bx_attention, dim3(c.heads, m->bmax), 128, bx::kAttSmem, m->stream, (const bx::bf16_t*)m->q_img,
               (const bx::bf16_t*)m->k_img, (const bx::bf16_t*)m->vt_img, m->ctx_img, (const int*)m->alive,
               (const int*)m->count, H, P);
    launch_gemm(m, b, bx::EPI_RESID, m->ctx_img, m->wo, H, H, m->bo, m->x, m->y, nullptr);
    bx::ExitArgs off{};
    launch_pdl(bx::bx_layernorm, dim3(m->bmax * bx::kSeq / 8), 256, 0, m->stream, (const float*)m->y, m->x, m->x_img,
               m->g1, m->be1, (const int*)m->alive, (const int*)m->count, H, P, c.ln_eps, off);
    launch_gemm(m, b, bx::EPI_GELU, m->x_img, m->w1, H, F, m->b1, nullptr, nullptr, m->f_img);
    launch_gemm(m, b, bx::EPI_RESID, m->f_img, m->w2, F, H, m->b2, m->x, m->y, nullptr);
    bx::ExitArgs ex{1, m->wl, m->bl, m->wc, m->bc, m->logits, m->exit_layer, m->sched, m->keep, m->done,
                    m->alive, m->count, c.classes, l, L, m->bmax, c.exit_threshold};
    launch_pdl(bx::bx_layernorm, dim3(m->bmax * bx::kSeq / 8), 256, 0, m->stream, (const float*)m->y, m->x, m->x_img,
               m->g2, m->be2, (const int*)m->alive, (const int*)m->count, H, P, c.ln_eps, ex);
    bx::check(cudaGetLastError(), "berxit layer launch");
  }
}

void run_graph(mbx_berxit* m, int b) {
  auto it = m->graphs.find(b);
  if (it == m->graphs.end()) {
    cudaGraph_t graph;
    bx::check(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      enqueue(m, b);
    } catch (...) {
      cudaStreamEndCapture(m->stream, &graph);
      throw;
    }
    bx::check(cudaStreamEndCapture(m->stream, &graph), "end capture");
    cudaGraphExec_t exec;
    bx::check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    it = m->graphs.emplace(b, exec).first;
  }
  bx::check(cudaGraphLaunch(it->second, m->stream), "graph launch");
  mbx::g_launches += 2 + 7 * m->c.layers;
}

}  // namespace

extern "C" {

void mbx_berxit_config_default(mbx_berxit_config* c) {
  c->hidden = 768;
  c->heads = 12;
  c->ffn = 3072;
  c->layers = 12;
  c->seq = 128;
  c->classes = 8;
  c->exit_threshold = 0.6f;
  c->ln_eps = 1e-12f;
}

int64_t mbx_berxit_param_count(const mbx_berxit_config* c) {
  const int64_t H = c->hidden, F = c->ffn;
  return 3 * H * H + 3 * H + H * H + H + 2 * H + F * H + F + H * F + H + 2 * H + H + 1 + c->classes * H + c->classes;
}

int mbx_berxit_make_params(const mbx_berxit_config* c, unsigned seed, float* out) {
  return guarded(nullptr, [&] {
    validate(c);
    std::mt19937 g(seed * 7919u + 17u);
    const int64_t h = c->hidden, f = c->ffn, C = c->classes;
    auto fill = [&](int64_t n, float lo, float hi) {
      for (int64_t k = 0; k < n; ++k) *out++ = uni(g, lo, hi);
    };
    const float a = 0.05f, bb = 0.02f;
    fill(3 * h * h, -a, a); fill(3 * h, -bb, bb);
    fill(h * h, -a, a); fill(h, -bb, bb);
    fill(h, 0.9f, 1.1f); fill(h, -0.1f, 0.1f);
    fill(f * h, -a, a); fill(f, -bb, bb);
    fill(h * f, -a, a); fill(h, -bb, bb);
    fill(h, 0.9f, 1.1f); fill(h, -0.1f, 0.1f);
    fill(h, -0.1f, 0.1f); fill(1, -0.1f, 0.1f);
    fill(C * h, -a, a); fill(C, -bb, bb);
  });
}

int mbx_berxit_make_input(const mbx_berxit_config* c, unsigned seed, int instance, float* out) {
  return guarded(nullptr, [&] {
    validate(c);
    std::mt19937 g(seed * 104729u + 31u * unsigned(instance) + 7u);
    for (int64_t k = 0; k < (int64_t)c->seq * c->hidden; ++k) out[k] = uni(g, -1.0f, 1.0f);
  });
}

int mbx_berxit_create(int device, int precision, const mbx_berxit_config* c, int max_batch, mbx_berxit** out) {
  *out = nullptr;
  auto m = new mbx_berxit();
  const int rc = guarded(m, [&] {
    validate_device(c);
    if (precision != MBX_PREC_BF16X3 && precision != MBX_PREC_BF16)
      throw std::runtime_error("berxit: precision must be bf16x3 or bf16");
    if (max_batch <= 0 || max_batch > 4096) throw std::runtime_error("berxit: max_batch out of range");
    m->device = device;
    m->precision = precision;
    m->P = precision == MBX_PREC_BF16X3 ? 2 : 1;
    m->c = *c;
    m->bmax = max_batch;
    bx::check(cudaSetDevice(device), "cudaSetDevice");
    bx::check(cudaDeviceGetAttribute(&m->sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    bx::check(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking), "stream");
    const size_t H = c->hidden, F = c->ffn, B = max_batch, S = bx::kSeq, P = m->P;
    m->params = dalloc<float>(mbx_berxit_param_count(c));
    m->wqkv = dalloc<bx::bf16_t>(3 * H * H * P);
    m->wo = dalloc<bx::bf16_t>(H * H * P);
    m->w1 = dalloc<bx::bf16_t>(F * H * P);
    m->w2 = dalloc<bx::bf16_t>(H * F * P);
    m->x = dalloc<float>(B * S * H);
    m->y = dalloc<float>(B * S * H);
    m->q_img = dalloc<bx::bf16_t>(B * S * H * P);
    m->k_img = dalloc<bx::bf16_t>(B * S * H * P);
    m->vt_img = dalloc<bx::bf16_t>(B * S * H * P);
    m->x_img = dalloc<bx::bf16_t>(B * S * H * P);
    m->ctx_img = dalloc<bx::bf16_t>(B * S * H * P);
    m->f_img = dalloc<bx::bf16_t>(B * S * F * P);
    m->logits = dalloc<float>(B * c->classes);
    m->alive = dalloc<int>(B);
    m->count = dalloc<int>(1);
    m->exit_layer = dalloc<int>(B);
    m->sched = dalloc<int>(B * c->layers);
    m->keep = dalloc<int>(B);
    m->wc_al = dalloc<float>((size_t)c->classes * H);
    m->done = dalloc<unsigned>(1);
    bx::check(cudaMemset(m->done, 0, sizeof(unsigned)), "memset");
    const size_t smem = bx::kStageSmem + 256;
    bx::check(cudaFuncSetAttribute(bx::bx_gemm<bx::EPI_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
    bx::check(cudaFuncSetAttribute(bx::bx_gemm<bx::EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
    bx::check(cudaFuncSetAttribute(bx::bx_gemm<bx::EPI_GELU>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
    bx::check(cudaFuncSetAttribute(bx::bx_gemm<bx::EPI_QKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");

    bx::check(cudaFuncSetAttribute(bx::bx_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, bx::kAttSmem), "attr");
  });
  if (rc) {
    g_bx_err = m->err;
    mbx_berxit_destroy(m);
    return rc;
  }
  *out = m;
  return 0;
}

void mbx_berxit_destroy(mbx_berxit* m) {
  if (!m) return;
  for (auto& kv : m->graphs) cudaGraphExecDestroy(kv.second);
  void* bufs[] = {m->params, m->wqkv, m->wo, m->w1, m->w2, m->x, m->y, m->q_img, m->k_img, m->vt_img, m->x_img, m->ctx_img,
                  m->f_img, m->logits, m->alive, m->count, m->exit_layer, m->sched, m->keep, m->done, m->wc_al};
  for (void* p : bufs)
    if (p) cudaFree(p);
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
}

const char* mbx_berxit_last_error(const mbx_berxit* m) { return m ? m->err.c_str() : g_bx_err.c_str(); }

int mbx_berxit_set_params(mbx_berxit* m, const float* params, int64_t n) {
  return guarded(m, [&] {
    if (n != mbx_berxit_param_count(&m->c)) throw std::runtime_error("berxit: parameter count mismatch");
    bx::check(cudaSetDevice(m->device), "cudaSetDevice");
    bx::check(cudaMemcpyAsync(m->params, params, n * sizeof(float), cudaMemcpyHostToDevice, m->stream), "params H2D");
    const int64_t H = m->c.hidden, F = m->c.ffn;
    const float* p = m->params;
    const float* wqkv = p; p += 3 * H * H;
    m->bqkv = p; p += 3 * H;
    const float* wo = p; p += H * H;
    m->bo = p; p += H;
    m->g1 = p; p += H;
    m->be1 = p; p += H;
    const float* w1 = p; p += F * H;
    m->b1 = p; p += F;
    const float* w2 = p; p += H * F;
    m->b2 = p; p += H;
    m->g2 = p; p += H;
    m->be2 = p; p += H;
    m->wl = p; p += H;
    m->bl = p; p += 1;
    // Wc follows the single b_lte float: an aligned copy for the exit head's float4 loads.
    bx::check(cudaMemcpyAsync(m->wc_al, p, sizeof(float) * m->c.classes * H, cudaMemcpyDeviceToDevice, m->stream),
              "Wc copy");
    m->wc = m->wc_al; p += m->c.classes * H;
    m->bc = p;
    auto img = [&](const float* W, bx::bf16_t* out, int64_t N, int64_t K) {
      const int64_t e = N * K;
      bx::bx_weight_image<<<unsigned((e + 255) / 256), 256, 0, m->stream>>>(W, out, int(N), int(K), m->P);
      bx::check(cudaGetLastError(), "weight image");
      ++mbx::g_launches;
    };
    img(wqkv, m->wqkv, 3 * H, H);
    img(wo, m->wo, H, H);
    img(w1, m->w1, F, H);
    img(w2, m->w2, H, F);
    bx::check(cudaStreamSynchronize(m->stream), "params sync");
    m->params_set = true;
  });
}

int mbx_berxit_run_device(mbx_berxit* m, int batch, const float* x_dev) {
  return guarded(m, [&] {
    if (!m->params_set) throw std::runtime_error("berxit: parameters not set");
    if (batch <= 0 || batch > m->bmax) throw std::runtime_error("berxit: batch out of range");
    bx::check(cudaSetDevice(m->device), "cudaSetDevice");
    const size_t n = (size_t)batch * bx::kSeq * m->c.hidden;
    if (x_dev != m->x)
      bx::check(cudaMemcpyAsync(m->x, x_dev, n * sizeof(float), cudaMemcpyDeviceToDevice, m->stream), "inputs D2D");
    run_graph(m, batch);
  });
}

int mbx_berxit_read(mbx_berxit* m, int batch, float* logits, int32_t* exit_layer, int32_t* schedule) {
  return guarded(m, [&] {
    if (batch <= 0 || batch > m->bmax) throw std::runtime_error("berxit: batch out of range");
    const int C = m->c.classes, L = m->c.layers;
    if (logits)
      bx::check(cudaMemcpyAsync(logits, m->logits, sizeof(float) * batch * C, cudaMemcpyDeviceToHost, m->stream), "D2H");
    if (exit_layer)
      bx::check(cudaMemcpyAsync(exit_layer, m->exit_layer, sizeof(int) * batch, cudaMemcpyDeviceToHost, m->stream), "D2H");
    if (schedule)
      for (int l = 0; l < L; ++l)
        bx::check(cudaMemcpyAsync(schedule + (size_t)l * batch, m->sched + (size_t)l * m->bmax, sizeof(int) * batch,
                                  cudaMemcpyDeviceToHost, m->stream),
                  "D2H");
    bx::check(cudaStreamSynchronize(m->stream), "berxit sync");
  });
}

int mbx_berxit_run(mbx_berxit* m, int batch, const float* x, float* logits, int32_t* exit_layer, int32_t* schedule) {
  return guarded(m, [&] {
    if (!m->params_set) throw std::runtime_error("berxit: parameters not set");
    if (batch <= 0 || batch > m->bmax) throw std::runtime_error("berxit: batch out of range");
    bx::check(cudaSetDevice(m->device), "cudaSetDevice");
    const size_t n = (size_t)batch * bx::kSeq * m->c.hidden;
    bx::check(cudaMemcpyAsync(m->x, x, n * sizeof(float), cudaMemcpyHostToDevice, m->stream), "inputs H2D");
    run_graph(m, batch);
    if (mbx_berxit_read(m, batch, logits, exit_layer, schedule)) throw std::runtime_error(m->err);
  });
}

void* mbx_berxit_stream(mbx_berxit* m) { return m ? m->stream : nullptr; }

int mbx_berxit_launches_per_batch(const mbx_berxit* m, int) { return 2 + 7 * m->c.layers; }

}  // extern "C"
