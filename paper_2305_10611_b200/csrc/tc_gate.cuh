// tc_gate.cuh — device source of the per-plan tensor-core and pointwise kernels.
//
// This file is not compiled on its own.  At plan registration (kernels_tc.cu: tc_prepare) the
// host generates a prelude with the plan's compile-time shape (MBX_KC, MBX_U, MBX_G, MBX_UC, ...)
// and its column-local elementwise tail as straight-line code (mbx_tail / mbx_pw_tail), then
// compiles prelude + libm_fp32.cuh + tc_abi.h + this file for sm_100a with NVRTC (jit.cpp).  The
// reference equally generates one kernel per signature (kernelgen.cpp:212-292 lowers each block
// into a plan; ACRoBat emits a specialised batched kernel per plan).
//
// mbx_tc_gate — plans  [concat(p0, p1)] -> dense / FusedDense(row, shared W_1..W_G) -> tail:
//   swap-AB tcgen05: MMA M = 128 gate rows of one unit tile (G gates x UC units, zero padded),
//   N = NT nodes of one node tile, K in chunks of MBX_KC; fp32 accumulator in TMEM.
//   grid = (node tiles, unit tiles, K-split ranks); the ranks of a tile form a cluster.
//   warp 0      : weight producer — one cp.async.bulk per stage (TMA bulk engine), mbarrier ring
//   warp 1      : MMA issuer — one thread issues tcgen05.mma / tcgen05.commit
//   warps 2..7  : node-row gatherers — cp.async (16 B, or 4 B when rows are unaligned) straight
//                 from the arena through the per-node offset table into an fp32 staging ring,
//                 converted to split bf16 (hi, lo) in the canonical no-swizzle K-major layout;
//                 afterwards they prefetch the tail's input rows while the MMAs drain.
//   epilogue    : tcgen05.ld -> each rank pushes its partial accumulator for the nodes rank r
//                 finishes straight into rank r's shared memory (st.shared::cluster), one cluster
//                 barrier, then every thread sums the S partials in rank order (deterministic),
//                 runs the generated tail and writes the outputs batch-contiguously.
//   PDL: the weight stream starts before griddepcontrol.wait, everything that reads activations
//   after it, so a launch overlaps its predecessor's tail when launched programmatically.
//
// mbx_pointwise — purely elementwise plans: one thread per (node, element), generated tail with
//   the glibc-exact activations (bit-identical to the reference).

#define MBX_M 128

#define MBX_THREADS 256

namespace mbx_gen {

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

__device__ __forceinline__ void mbar_arrive_cnt(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Operand images (mbx_tc_levels): a consumer level whose every gathered row has exactly one
// producer row gets an image of its B operands, [tile][K rank][chunk][hi | lo][canonical
// no-swizzle K-major nt x KC], which the producers fill as they write the rows (split bf16) and
// the consumer loads with a few bulk copies.  d = {base lo, base hi, p | nt << 16,
// k0 | log2 KC << 12 | log2 kslice << 16 | parts << 20}: the tile's image (byte offset), the
// consumer column, the consumer's tile width, the piece's first K index, the consumer's K chunk and
// K slice per rank (both powers of two: shifts, no divisions in the producers' store loop), and the
// split-bf16 parts (2: hi, lo; 3: hi, mid, lo).
// Returns the byte offset of column u's hi part; part q is q * *part_off bytes further.
__device__ __forceinline__ long long img_addr(const int4 d, int u, int* part_off) {
  const long long base = (long long)(((unsigned long long)(unsigned)d.y << 32) | (unsigned)d.x);
  const int p = d.z & 0xffff, nt = d.z >> 16;
  const int k0 = d.w & 0xfff, lkc = (d.w >> 12) & 0xf, lks = (d.w >> 16) & 0xf, parts = (d.w >> 20) & 0xf;
  const int k = k0 + u, r = k >> lks, kr = k & ((1 << lks) - 1), j = kr >> lkc, kk = kr & ((1 << lkc) - 1);
  *part_off = nt << (lkc + 1);
  return base + (long long)((r << (lks - lkc)) + j) * parts * (nt << (lkc + 1)) + (p >> 3) * (16 << lkc) +
         (kk >> 3) * 128 + (p & 7) * 16 + (kk & 7) * 2;
}
__device__ __forceinline__ int img_parts(const int4 d) { return (d.w >> 20) & 0xf; }
// x = sum of `parts` bf16 values (successive residuals, round to nearest): hi, [mid,] lo.
__device__ __forceinline__ void split_bf16(float x, int parts, unsigned short* out) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (q >= parts) {
      out[q] = 0;
      continue;
    }
    unsigned short h;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(x));
    out[q] = h;
    x = x - __uint_as_float(unsigned(h) << 16);
  }
}

// Spin on test_wait (try_wait may park the warp for a scheduler quantum).
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
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

// Weight tiles are re-read by every level of a phase: keep them in L2 (evict_last).
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Canonical K-major, no-swizzle UMMA shared-memory descriptor: 8-row x 16-byte core matrices,
// K-adjacent core matrices 128 B apart (LBO), 8-row groups SBO bytes apart; version 1 (sm_100).
__device__ __forceinline__ unsigned long long make_desc(unsigned saddr, unsigned sbo) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3FFF);
  d |= (unsigned long long)((128u >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
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

__device__ __forceinline__ void tmem_ld8(unsigned addr, float* v) {
  unsigned r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive accumulator columns of this warp's 32 lanes, one wait.
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

__device__ __forceinline__ unsigned pack_bf16x2(float lo_elem, float hi_elem) {
  unsigned r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}
__device__ __forceinline__ float bf16_round(float x) {
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(x));
  return __uint_as_float(unsigned(h) << 16);
}

// Byte offset of element (row r, k) inside one K-chunk of the canonical layout.
__device__ __forceinline__ unsigned canon_off(int r, int kk) {
  return unsigned((r >> 3) * (MBX_KC * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}

}  // namespace mbx_gen

#ifdef MBX_STAMPS
#define MBX_STAMP(who, i)                                                                        \
  do {                                                                                           \
    if (threadIdx.x == (who)) {                                                                  \
      unsigned long long t_;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
      P.stamps[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + (i)] = t_; \
    }                                                                                            \
  } while (0)
#define MBX_CSTAMP(i)                                                                                   \
  do {                                                                                                  \
    if (threadIdx.x == 64 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64) {     \
      unsigned long long t_ = clock64();                                                                \
      P.stamps[gridDim.x * gridDim.y * gridDim.z * 8 + (i)] = t_;                                       \
    }                                                                                                   \
  } while (0)
#define MBX_MSTAMP(i)                                                                                   \
  do {                                                                                                  \
    if (threadIdx.x == 32 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 30) {      \
      unsigned long long t_ = clock64();                                                                \
      P.stamps[gridDim.x * gridDim.y * gridDim.z * 8 + 32 + (i)] = t_;                                  \
    }                                                                                                   \
  } while (0)
#else
#define MBX_MSTAMP(i) \
  do {                \
  } while (0)
#define MBX_CSTAMP(i) \
  do {                \
  } while (0)
#define MBX_STAMP(who, i) \
  do {                    \
  } while (0)
#endif

#ifdef MBX_GATE_KERNEL
// Roles (256 threads): warp 0 lane 0 = weight producer, warp 1 = TMEM owner + MMA issuer, warps
// 2-7 = node-row gather (cp.async straight into the MMA stage, completion counted on an mbarrier
// by cp.async.mbarrier.arrive) and in-place fp32 -> split bf16 conversion.
#define MBX_GATHER 192
#define MBX_STAGES 4
#ifndef MBX_LOOKAHEAD
#define MBX_LOOKAHEAD 2
#endif
extern "C" __global__ void __launch_bounds__(MBX_THREADS, 1) mbx_tc_gate(const __grid_constant__ TcGateArgs P) {
  using namespace mbx_gen;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = P.NT;
  const int node0 = blockIdx.x * NT;
  const int tile_u = blockIdx.y;
  const int nn = min(NT, P.b - node0);
  MBX_STAMP(0, 0);
  MBX_CSTAMP(63);
  const int npass = P.npass;
  constexpr int S = MBX_STAGES;  // power of two: stage / phase arithmetic is shifts and masks
  const int ksplit = P.ksplit;
  unsigned rank = 0;
  if (ksplit > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cpr = MBX_NCHUNKS / ksplit;  // chunks per rank
  const int c_begin = int(rank) * cpr;
  // Unit tiles read the same node rows: start each at a different chunk so concurrent requests
  // spread over different L2 lines.  Chunk of pipeline step i: c_begin + (i + rot) mod cpr.
  const int rot = (tile_u * 3) % cpr;
  auto chunk_of = [&](int i) {
    const int j = i + rot;
    return c_begin + (j >= cpr ? j - cpr : j);
  };
  const int ntr = NT / ksplit;           // nodes this rank finishes
  const int nloc0 = int(rank) * ntr;     // first of them within the tile
  const int nloc = max(0, min(ntr, nn - nloc0));
  const int E = ntr * MBX_UC;

  const int wpass = npass > 1 ? 2 : 1;
  const int wchunk = MBX_M * MBX_KC * 2;  // one pass of one weight chunk (bytes)
  const int xchunk = NT * MBX_KC * 2;     // one pass of one node chunk
  const int wstage = wchunk * wpass;
  const int stage_bytes = wstage + 2 * xchunk;  // X part doubles as the fp32 landing zone
  unsigned char* ring = smem + P.ring_off;
  float* recv = reinterpret_cast<float*>(smem + P.recv_off);  // [S-1][ntr][128] peers' partials
  float* srcbuf = reinterpret_cast<float*>(smem + P.src_off);
  unsigned long long* full_w = reinterpret_cast<unsigned long long*>(smem + P.bar_off);
  unsigned long long* full_x = full_w + S;
  unsigned long long* xraw = full_x + S;
  unsigned long long* empty = xraw + S;
  unsigned long long* done = empty + S;
  unsigned long long* rbar = done + 1;
  unsigned long long* tready = rbar + 1;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(rbar + 2);
  long long* rowbase = reinterpret_cast<long long*>(rbar + 3);  // [NT][2]

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_w[s], 1);
      mbar_init(&full_x[s], MBX_GATHER / 32);
      mbar_init(&xraw[s], MBX_GATHER);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(rbar, 1);
    mbar_init(tready, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ksplit > 1) mbar_expect_tx(rbar, unsigned((ksplit - 1) * ntr * MBX_M * 4));
  }
  __syncthreads();
  // Peers may push partials into this CTA's receive buffer once its mbarrier is armed.
  if (ksplit > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  pdl_launch_dependents();
  MBX_STAMP(0, 1);

  if (warp == 0) {
    // ---- weight producer (weights are static: no dependency on the previous launch) ----
    if (lane == 0) {
      const unsigned char* wtile = P.wpack + (size_t)tile_u * MBX_NCHUNKS * wstage;
      const unsigned long long keep = policy_evict_last();
      for (int i = 0; i < cpr; ++i) {
        const int c = chunk_of(i), s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        mbar_expect_tx(&full_w[s], wstage);
        bulk_g2s_keep(ring + s * stage_bytes, wtile + (size_t)c * wstage, wstage, &full_w[s], keep);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (also owns the TMEM allocation; the epilogue learns the address through
    // the tready mbarrier) ----
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    tc_fence_before();
    mbar_arrive(tready);
    mbar_wait(tready, 0);
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    if (lane == 0) {
      // kind::f16, A = B = BF16, D = F32, both K-major, N = NT, M = 128.
      const unsigned idesc = (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(NT >> 3) << 17) | (unsigned(MBX_M >> 4) << 24);
      const unsigned ra = smem_u32(ring);
      const unsigned sbo = unsigned(MBX_KC * 16);
      for (int i = 0; i < cpr; ++i) {
        const int s = i % S;
        mbar_wait(&full_w[s], (i / S) & 1);
        MBX_MSTAMP(3 * i);
        mbar_wait(&full_x[s], (i / S) & 1);
        MBX_MSTAMP(3 * i + 1);
        tc_fence_after();
        const unsigned wa = ra + s * stage_bytes;
        const unsigned xa = wa + wstage;
        const unsigned long long a_hi = make_desc(wa, sbo), b_hi = make_desc(xa, sbo);
        const unsigned long long a_lo = make_desc(wa + wchunk, sbo), b_lo = make_desc(xa + xchunk, sbo);
#pragma unroll
        for (int ks = 0; ks < MBX_KC / 16; ++ks) {
          const unsigned long long step = (unsigned long long)(ks * 16);  // +256 B in 16-byte units
          mma_bf16(tmem, a_hi + step, b_hi + step, idesc, (i | ks) ? 1u : 0u);
          if (npass > 1) {
            mma_bf16(tmem, a_hi + step, b_lo + step, idesc, 1u);
            mma_bf16(tmem, a_lo + step, b_hi + step, idesc, 1u);
          }
        }
        mma_commit(&empty[s]);
        MBX_MSTAMP(3 * i + 2);
      }
      mma_commit(done);
      MBX_STAMP(32, 4);
    }
  } else {
    // ---- node rows (warps 2-7): cp.async 16 B quads (4 B when rows are unaligned) straight into
    // the stage's landing zone, LOOKAHEAD chunks ahead; arrival of everyone's quads is counted
    // on xraw[s] by cp.async.mbarrier.arrive; then each thread converts its share of the landed
    // chunk to split bf16 in place. ----
    const int gt = tid - 64;
    pdl_wait();  // activations and offset tables of this launch are ready
    for (int i = gt; i < NT * 2; i += MBX_GATHER) {
      const int n = i >> 1, pc = i & 1;
      long long base = 0;
      if (n < nn && pc < MBX_NPIECES)
        base = (P.piece_kind[pc] == 0 ? P.shared_off[P.piece_idx[pc]]
                                      : P.batched_off[(long long)(node0 + n) * P.nb + P.piece_idx[pc]]) +
               P.piece_off[pc];
      rowbase[i] = base;
    }
    named_sync(1, MBX_GATHER);
    // Lane mapping: each group of 8 lanes handles one quad position of 8 consecutive nodes, so its
    // shared-memory writes cover one contiguous 128-byte core matrix (no bank conflicts); quad qq
    // of a node row lands where its 8-element group's hi (even qq) or lo (odd qq) operand will
    // live, so the conversion rewrites it in place.
    constexpr int kq = MBX_KC / 4;  // 16-byte quads per node row per chunk
    const int l8 = gt & 7;
    const int g0 = gt >> 3;          // 0..23
    const int ngroups = (NT >> 3) * kq;
    const float* arena = P.arena;
    auto issue = [&](int i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      const int k = chunk_of(i) * MBX_KC;
      const int p1 = (MBX_NPIECES > 1 && k >= MBX_PK0) ? 1 : 0;  // chunks never straddle the pieces
      const int kin = k - (p1 ? MBX_PK0 : 0);
      unsigned char* xs = ring + s * stage_bytes + wstage;
      for (int g = g0; g < ngroups; g += MBX_GATHER / 8) {
        const int qq = g % kq, nb8 = g / kq;
        const int n = nb8 * 8 + l8;
        const bool valid = n < nn;
        const float* src = arena + (valid ? rowbase[2 * n + p1] + kin + qq * 4 : 0);
        float* dst = reinterpret_cast<float*>(xs + nb8 * (MBX_KC * 16) + l8 * 16 + ((qq >> 1) << 7) +
                                              ((qq & 1) ? xchunk : 0));
        if (P.vec16) {
          cp_async16(dst, src, valid);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) cp_async4(dst + e, src + e, valid);
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&xraw[s])) : "memory");
    };
    auto prefetch_tail_inputs = [&]() {
      // The tail's input rows for the nodes this rank finishes: one row = UC consecutive floats.
      for (int r = gt; r < P.nloads * ntr; r += MBX_GATHER) {
        const int j = r / ntr, n = r - j * ntr;
        float* dst = srcbuf + j * E + n * MBX_UC;
        const bool valid = n < nloc;
        long long base = 0;
        if (valid) {
          const TcLoad& l = P.loads[j];
          const long long node = node0 + nloc0 + n;
          base = (l.kind == 1 ? P.batched_off[node * P.nb + l.idx] : P.shared_off[l.idx]) + l.off + tile_u * MBX_UC;
        }
        const float* src = arena + base;
#pragma unroll 8
        for (int u = 0; u < MBX_UC; ++u) cp_async4(dst + u, src + u, valid);
      }
    };
    const int look = min(MBX_LOOKAHEAD, S - 1);
    for (int j = 0; j < min(look, cpr); ++j) issue(j);
    if (look >= cpr) prefetch_tail_inputs();
    constexpr int kb = MBX_KC / 8;
    const int ngroups8 = (NT >> 3) * kb;
    for (int i = 0; i < cpr; ++i) {
      if (i + look < cpr) {
        issue(i + look);
        if (i + look == cpr - 1) prefetch_tail_inputs();
      }
      const int s = i % S;
      mbar_wait(&xraw[s], (i / S) & 1);
      MBX_CSTAMP(2 * i);
      unsigned char* xs = ring + s * stage_bytes + wstage;
      for (int g = g0; g < ngroups8; g += MBX_GATHER / 8) {
        const int m = g % kb, nb8 = g / kb;  // 8 lanes = one core matrix (8 nodes x 8 k)
        const unsigned off = unsigned(nb8 * (MBX_KC * 16) + m * 128 + l8 * 16);
        const float4 a = *reinterpret_cast<const float4*>(xs + off);
        const float4 bq = *reinterpret_cast<const float4*>(xs + xchunk + off);
        const float v[8] = {a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w};
        unsigned hp[4], lp[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hp[q] = pack_bf16x2(v[2 * q], v[2 * q + 1]);  // low half = element 2q
          const float h0 = __uint_as_float(hp[q] << 16), h1 = __uint_as_float(hp[q] & 0xffff0000u);
          lp[q] = pack_bf16x2(v[2 * q] - h0, v[2 * q + 1] - h1);
        }
        const uint4 hi = make_uint4(hp[0], hp[1], hp[2], hp[3]);
        const uint4 lo = make_uint4(lp[0], lp[1], lp[2], lp[3]);
        // All of a group's quads were read above by this thread, so in-place is safe.
        *reinterpret_cast<uint4*>(xs + off) = hi;
        if (npass > 1) *reinterpret_cast<uint4*>(xs + xchunk + off) = lo;
      }
      fence_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_x[s]);
      MBX_CSTAMP(2 * i + 1);
    }
    cp_async_wait<0>();
  }

  // ---- epilogue ----
  pdl_wait();
  mbar_wait(tready, 0);
  mbar_wait(done, 0);
  MBX_STAMP(0, 5);
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  // TMEM lane = gate row; warp w reads lanes 32*(w%4).. for half of the node columns into the
  // drained ring: stg[node][row].
  float* stg = reinterpret_cast<float*>(ring);
  {
    const int q = warp & 3, half = warp >> 2;
    const int row = q * 32 + lane;
    const int cols = NT / 2;
    for (int c0 = half * cols; c0 < (half + 1) * cols; c0 += 8) {
      float v[8];
      tmem_ld8(tmem + (unsigned(q * 32) << 16) + unsigned(c0), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) stg[(c0 + k) * MBX_M + row] = v[k];
    }
  }
  tc_fence_before();
  if (ksplit > 1) {
    fence_async_smem();  // staged partials -> visible to the bulk-copy engine
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' barriers armed
  }
  __syncthreads();
  MBX_STAMP(0, 2);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
  if (ksplit > 1) {
    // Split-K: push the partial rows of the nodes rank r finishes to rank r (DSMEM bulk copies,
    // completion counted on r's receive mbarrier), then wait for the S-1 incoming slices.
    if (tid == 0) {
      const unsigned bytes = unsigned(ntr * MBX_M * 4);
      for (int r = 0; r < ksplit; ++r) {
        if (r == int(rank)) continue;
        const int slot = int(rank) < r ? int(rank) : int(rank) - 1;
        unsigned dst, bar;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(dst)
                     : "r"(smem_u32(recv + (size_t)slot * ntr * MBX_M)), "r"(r));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(rbar)), "r"(r));
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "r"(smem_u32(stg + (size_t)r * ntr * MBX_M)), "r"(bytes), "r"(bar)
            : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    mbar_wait(rbar, 0);
  }
  MBX_STAMP(0, 6);

  // Sum the partials in rank order (deterministic) and run the plan's tail per (node, unit).
  for (int e = tid; e < nloc * MBX_UC; e += MBX_THREADS) {
    const int n = e / MBX_UC, u = e - n * MBX_UC;
    float g[MBX_G];
#pragma unroll
    for (int gi = 0; gi < MBX_G; ++gi) {
      const int col = gi * MBX_UC + u;
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q >= ksplit) break;
        const float v = q == int(rank) ? stg[(nloc0 + n) * MBX_M + col]
                                       : recv[((q < int(rank) ? q : q - 1) * ntr + n) * MBX_M + col];
        acc = q == 0 ? v : acc + v;
      }
      g[gi] = acc;
    }
    float l[MBX_NLOADS > 0 ? MBX_NLOADS : 1];
#pragma unroll
    for (int j = 0; j < MBX_NLOADS; ++j) l[j] = srcbuf[j * E + e];
    float o[MBX_NOUT];
    mbx_tail(g, l, o);
    const long long node = node0 + nloc0 + n;
    const int ug = tile_u * MBX_UC + u;
#pragma unroll
    for (int k = 0; k < MBX_NOUT; ++k) P.arena[P.out_base[k] + node * MBX_U + ug] = o[k];
  }
  if (ksplit > 1 && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#ifdef MBX_STAMPS
  __syncthreads();
  MBX_STAMP(0, 7);
#endif
}
#endif  // MBX_GATE_KERNEL


#ifdef MBX_LEVELS_KERNEL
// mbx_tc_levels — one persistent launch for a run of consecutive batches ("levels") of the same
// gate plan, e.g. every internal-node depth of a TreeLSTM flush.
//   grid = (node-tile groups, unit tiles, MBX_LS K-split ranks), all CTAs co-resident (one per
//   SM); group x takes node tiles x, x + gridDim.x, ... of every level.
//   * The CTA's weight slice (128 gate rows x K/MBX_LS, split bf16) is bulk-copied into shared
//     memory ONCE and reused by every level: per level only the node rows move.
//   * Per node tile: 16-byte cp.async gathers the rows of this rank's K slice through the level's
//     offset table straight into the canonical no-swizzle K-major UMMA layout.  Rows whose
//     producer wrote their split-bf16 shadow (TcLevel::shadow: [8 x bf16 hi | 8 x bf16 lo] per
//     8-float group at the row's own offset) arrive MMA-ready; otherwise the fp32 rows are
//     converted to split bf16 in place.  tcgen05.mma into TMEM, partial accumulators exchanged
//     between the K ranks of the unit tile, summed in rank order (deterministic), the generated
//     tail, outputs (and, where a later level gathers them, their shadows) written
//     batch-contiguously.
//     MBX_LXCH 0: the ranks form a cluster; partials move by DSMEM bulk copies.
//     MBX_LXCH 1: no cluster (any grid that fits on the SMs); partials move through an
//                 L2-resident buffer, completion signalled by per-(group, unit tile, rank) release
//                 counters, which each owner resets when the launch is done with them.
//   * Between levels, per-unit-tile readiness counters instead of a grid barrier: a CTA releases
//     its unit tile's counter when it finished a level; before the next level it acquires only
//     the counters of the unit tiles that produce the columns its K slice (and its tail) reads
//     (TcLevelsArgs::dep_mask), so it never waits for the rest of the grid.  Every read of
//     activations bypasses L1 (.cg): L1 is not coherent.
#define MBX_LGATHER 192
#define MBX_LCPR (MBX_NCHUNKS / MBX_LS)
#if MBX_LXCH == 0
#define MBX_LLOC (MBX_LNT / MBX_LS)  // nodes a rank finishes per tile: a contiguous slice
#else
#define MBX_LLOC (((MBX_LNT / 8 + MBX_LS - 1) / MBX_LS) * 8)  // 8-node chunks c with c % S == rank
#endif
#define MBX_LEPT ((MBX_LLOC * MBX_UC + MBX_THREADS - 1) / MBX_THREADS)
// Elements are handed out in pairs of consecutive units of one node when the tile allows it, so
// the partial sums load 8 bytes per (gate, rank) (half the load instructions) while every thread
// still gets a share of the tail.
#if MBX_UC % 2 == 0 && MBX_LEPT % 2 == 0
#define MBX_LQ 2
#else
#define MBX_LQ 1
#endif
#define MBX_READY_STRIDE 32  // readiness counters one 128-byte line apart
#ifdef MBX_STAMPS
#define MBX_LSTAMP_T(t, lv, i)                                                                      \
  do {                                                                                              \
    if (threadIdx.x == (t) && (lv) < 64) {                                                          \
      P.stamps[(((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 64 + (lv)) * 16 + \
               (i)] = clock64();                                                                      \
    }                                                                                               \
  } while (0)
#else
#define MBX_LSTAMP_T(t, lv, i) \
  do {                         \
  } while (0)
#endif
#define MBX_LSTAMP(lv, i) MBX_LSTAMP_T(0, lv, i)

namespace mbx_gen {
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// One thread spins until *ctr reaches target (modular); a wait that cannot complete (it never
// should: every CTA is co-resident) traps after ~2 s instead of hanging the GPU.
__device__ __forceinline__ void spin_until(const unsigned* ctr, unsigned target) {
  if (int(ld_acquire_u32(ctr) - target) >= 0) return;
  const unsigned long long t0 = global_ns();
  while (int(ld_acquire_u32(ctr) - target) < 0)
    if (global_ns() - t0 > 2000000000ull) __trap();
}
// Partials: shared memory (exchange through DSMEM) or L2 (.cg: written by other SMs this launch).
__device__ __forceinline__ float ld_partial(const float* p) {
#if MBX_LXCH == 0
  return *p;
#else
  return __ldcg(p);
#endif
}
__device__ __forceinline__ float2 ld_partial2(const float* p) {
#if MBX_LXCH == 0
  return *reinterpret_cast<const float2*>(p);
#else
  return __ldcg(reinterpret_cast<const float2*>(p));
#endif
}
// Split-bf16 shadow of one output element at arena float offset o: bytes [4g, 4g + 16) of the
// shadow hold the 8 bf16 "hi" parts of the 8-float group g = o & ~7, bytes [4g + 16, 4g + 32)
// the "lo" parts (hi = bf16(x), lo = bf16(x - hi), exactly the gather's in-place conversion).
__device__ __forceinline__ void store_shadow(unsigned char* shadow, long long o, float x) {
  unsigned short h, l;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(x));
  const float rest = x - __uint_as_float(unsigned(h) << 16);
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(l) : "f"(rest));
  unsigned char* p = shadow + 4 * o - 2 * (o & 7);
  *reinterpret_cast<unsigned short*>(p) = h;
  *reinterpret_cast<unsigned short*>(p + 16) = l;
}
}  // namespace mbx_gen

extern "C" __global__ void __launch_bounds__(MBX_THREADS, 1) mbx_tc_levels(const __grid_constant__ TcLevelsArgs P) {
  using namespace mbx_gen;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ TcLevel slv[64];  // the first 64 entries of the level table
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  MBX_LSTAMP(0, 14);  // kernel entry
  const int tile_u = blockIdx.y;
  constexpr int S = MBX_LS;
  for (int i = tid; i < min(P.nlevels, 64); i += MBX_THREADS) slv[i] = P.levels[i];
  constexpr int CPR = MBX_LCPR;
  unsigned rank = 0;
#if MBX_LXCH == 0
  if (S > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
#else
  rank = blockIdx.z;
#endif
  const int c_begin = int(rank) * CPR;
  const int npass = P.npass;
  // Split-bf16 parts of each operand: 1 (bf16), 2 (bf16x3: hi, lo), 3 (bf16x6: hi, mid, lo);
  // the shared-memory layout holds MBX_LPARTS.
  // (A bf16x6 context registers its plans with MBX_LPARTS 3, the others with 2: compile-time
  // bounds for the MMA and image loops.)
  const int parts = npass == 1 ? 1 : MBX_LPARTS;
  const int wpass = parts;
  const int wchunk = MBX_M * MBX_KC * 2;
  const int wstage = wchunk * wpass;
  constexpr int xchunk = MBX_LNT * MBX_KC * 2;  // one part of one node chunk at the maximal tile
  // Part q sits q * (xchunk + 64) into the chunk: the lo part 64 B past the hi part modulo 128, so
  // the gather's 16-byte writes of a row's even and odd quads fall in different banks; chunks are
  // xstride apart.
  constexpr int xlo = xchunk + 64;
  constexpr int xstride = MBX_LPARTS * (xchunk + 64);
  unsigned char* wsm = smem + P.w_off;          // [CPR][wstage], resident for the whole launch
  unsigned char* xsm = smem + P.x_off;          // [CPR][xstride]; after the MMAs: stg (LXCH 0)
  float* stg = reinterpret_cast<float*>(xsm);   // [nt][128] this rank's partials (LXCH 0)
  float* recv = reinterpret_cast<float*>(smem + P.recv_off);  // [S-1][nt/S][128] peers' partials
  unsigned long long* wfull = reinterpret_cast<unsigned long long*>(smem + P.bar_off);
  unsigned long long* xraw = wfull + 1;
  unsigned long long* xfull = xraw + CPR;
  unsigned long long* done = xfull + CPR;
  unsigned long long* rbar = done + 1;
  unsigned long long* tready = rbar + 1;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tready + 1);
  long long* rowbase = reinterpret_cast<long long*>(tready + 2);  // [MBX_LNT][2]
  (void)recv;
  (void)stg;

  if (tid == 0) {
    mbar_init(wfull, 1);
    for (int j = 0; j < CPR; ++j) {
      mbar_init(&xraw[j], MBX_LGATHER);
      mbar_init(&xfull[j], MBX_LGATHER / 32);
    }
    mbar_init(done, 1);
    mbar_init(rbar, 1);
    mbar_init(tready, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // The weight slice: static, so it streams in before the previous kernel finishes (PDL).
    mbar_expect_tx(wfull, unsigned(CPR * wstage));
    const unsigned char* wtile = P.wpack + (size_t)tile_u * MBX_NCHUNKS * wstage;
    const unsigned long long keep = policy_evict_last();
    for (int j = 0; j < CPR; ++j)
      bulk_g2s_keep(wsm + j * wstage, wtile + (size_t)(c_begin + j) * wstage, wstage, wfull, keep);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
#if MBX_LXCH == 0
  if (S > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
  else __syncthreads();
#else
  __syncthreads();
#endif
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  const int grp = blockIdx.x, ngrp = gridDim.x;
  const int gt = tid - 64;  // gather thread index (warps 2-7)
  // Readiness counters this CTA acquires before a level: the unit tiles its K slice reads (per
  // rank, from the host) and those its tail's batched loads read.
  unsigned long long deps = P.dep_mask[rank];
  for (int j = 0; j < MBX_NLOADS; ++j)
    if (P.loads[j].kind == 1) {
      const int c0 = P.loads[j].off + tile_u * MBX_UC;
      if (c0 + MBX_UC <= MBX_U) {
        for (int t = c0 / MBX_UC; t <= (c0 + MBX_UC - 1) / MBX_UC; ++t) deps |= 1ull << t;
      } else {
        deps = ~0ull;
      }
    }
  // Its own unit tile always: then a counter reaching per_level * lv proves every CTA of that tile
  // finished level lv - 1 (each increments once per level, only after its own wait at that level,
  // which includes its own counter), however unevenly the CTAs progress.
  deps |= 1ull << tile_u;
  deps &= gridDim.y >= 64 ? ~0ull : ((1ull << gridDim.y) - 1ull);
  const unsigned per_level = unsigned(ngrp * S);  // increments of one counter per completed level
  // Offset-table lookups of one tile's node rows (static: known before the producers finish).
  auto fill_rowbase = [&](const TcLevel L, int node0, int nt) {
    const int nn = min(nt, L.b - node0);
    for (int i = gt; i < nt * 2; i += MBX_LGATHER) {
      const int n = i >> 1, pc = i & 1;
      long long base = 0;
      if (n < nn && pc < MBX_NPIECES)
        base = (P.piece_kind[pc] == 0 ? __ldg(L.shared_off + P.piece_idx[pc])
                                      : __ldg(L.batched_off + (long long)(node0 + n) * P.nb + P.piece_idx[pc])) +
               P.piece_off[pc];
      rowbase[i] = base;
    }
  };
  bool have_rb = false;  // gather threads: rowbase already holds the next tile's rows
  auto lvl = [&](int i) -> TcLevel { return i < 64 ? slv[i] : P.levels[i]; };
  if (warp >= 2 && grp * slv[0].nt < slv[0].b) {
    fill_rowbase(slv[0], grp * slv[0].nt, slv[0].nt);
    have_rb = true;
  }
  pdl_wait();  // the first level's inputs come from earlier launches

  unsigned it = 0;  // node tiles processed by this CTA: parity of every per-tile mbarrier
  for (int lv = 0; lv < P.nlevels; ++lv) {
    // By value: the compiler cannot prove the arena stores leave the table alone, and a reference
    // would re-read it from global memory inside every loop.
    const TcLevel L = lvl(lv);
    long long obase[MBX_NOUT];
#pragma unroll
    for (int k = 0; k < MBX_NOUT; ++k) obase[k] = __ldg(L.out_base + k);
    const int b = L.b, nt = L.nt;
    const int ntr = nt / S;
    MBX_LSTAMP(lv, 0);
    if (lv + 1 == P.nlevels) pdl_launch_dependents();
    if (lv > 0) {
      // Levels 0..lv-1 of every unit tile this CTA reads are complete once their counters reach
      // per_level * lv (each of the tile's CTAs adds 1 per finished level).  CTAs with no tile at
      // this level wait too: an early increment would stand in for a missing one.
      if (tid < 64 && ((deps >> tid) & 1ull))
        spin_until(P.ready + tid * MBX_READY_STRIDE, P.ready_base + per_level * unsigned(lv));
      __syncthreads();
    }
    MBX_LSTAMP(lv, 6);
    for (int node0 = grp * nt; node0 < b; node0 += ngrp * nt, ++it) {
      const unsigned par = it & 1u;
      const int nn = min(nt, b - node0);
#if MBX_LXCH == 0
      const int nloc0 = int(rank) * ntr;
      const int nloc = max(0, min(ntr, nn - nloc0));
      auto loc_col = [&](int m) { return nloc0 + m; };  // tile column of the rank's m-th node
      if (S > 1 && tid == 0) mbar_expect_tx(rbar, unsigned((S - 1) * ntr * MBX_M * 4));
#else
      // Rank r finishes the 8-node chunks c of the tile with c % S == r (lane-aligned slices).
      const int nloc = ((nt / 8 + S - 1) / S) * 8;  // this tile's node slots of the rank (<= MBX_LLOC)
      auto loc_col = [&](int m) { return (((m >> 3) * S + int(rank)) << 3) + (m & 7); };
#endif
      // Element t of this thread: node n (of the rank's slots) and unit u; its linear index
      // n * UC + u is quad * LQ + t % LQ with quad = tid + (t / LQ) * THREADS.
      auto elem = [&](int t, int& n, int& u) {
        constexpr int w = MBX_UC / MBX_LQ;
        const int qd = tid + (t / MBX_LQ) * MBX_THREADS;
        n = qd / w;
        u = (qd - n * w) * MBX_LQ + t % MBX_LQ;
      };
      // Whether element block t / LQ holds any element of this tile (warp-uniform).
      auto any_elem = [&](int t) { return (t / MBX_LQ) * MBX_THREADS * MBX_LQ < nloc * MBX_UC; };
      // ---- tail operands of the nodes this rank finishes: into registers, in flight during the
      // gather and the MMAs (warps 0-1 now, the gather warps once their copies are issued) ----
      float lreg[MBX_LEPT][MBX_NLOADS > 0 ? MBX_NLOADS : 1];
      int4 dreg[MBX_LEPT];  // image destinations of the element's row (L.img_slot >= 0)
      auto load_tail_operands = [&]() {
#pragma unroll
        for (int t = 0; t < MBX_LEPT; ++t) {
          int n, u;
          elem(t, n, u);
          const bool valid = n < nloc && loc_col(n) < nn;
          const long long node = node0 + loc_col(n);
          if (!any_elem(t)) break;  // warp-uniform: no element of this tile
#pragma unroll
          for (int j = 0; j < MBX_NLOADS; ++j) {
            const TcLoad& l = P.loads[j];
            float v = 0.0f;
            if (valid) {
              const long long base = (l.kind == 1 ? __ldg(L.batched_off + node * P.nb + l.idx) : __ldg(L.shared_off + l.idx)) +
                                     l.off + tile_u * MBX_UC + u;
              v = __ldcg(P.arena + base);
            }
            lreg[t][j] = v;
          }
          dreg[t] = make_int4(0, -1, 0, 0);
          if (L.img_slot >= 0 && valid) dreg[t] = __ldg(L.img_dst + node);
        }
      };
      if (warp < 2) load_tail_operands();
      if (warp >= 2) {
        // ---- gather (+ conversion of fp32 rows) on warps 2-7; rowbase is normally filled during
        // the previous tile ----
        if (!have_rb) fill_rowbase(L, node0, nt);
        have_rb = false;
        named_sync(1, MBX_LGATHER);
        MBX_LSTAMP_T(64, lv, 8);
        if (L.img >= 0) {
          // Operand image: this rank's K slice of the tile, already split bf16 in the canonical
          // layout — 2 bulk copies per chunk (hi, lo); the MMA issuer waits on xraw[j] itself.
          if (gt == 0) {
            // The image was written by other SMs' generic-proxy stores, released to this CTA
            // through the readiness counters; the bulk copies read it through the async proxy.
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const int cb = nt * MBX_KC * 2;
            const unsigned char* src = P.img + L.img + (long long)(node0 / nt) * nt * (MBX_NCHUNKS * MBX_KC) * 2 * parts +
                                       (long long)rank * CPR * parts * cb;
#pragma unroll 1
            for (int j = 0; j < CPR; ++j) {
              mbar_expect_tx(&xraw[j], unsigned(parts * cb));
              mbar_arrive_cnt(&xraw[j], MBX_LGATHER - 1);
              unsigned char* xs = xsm + j * xstride;
              for (int q = 0; q < parts; ++q)
                bulk_g2s(xs + q * xlo, src + (long long)(j * parts + q) * cb, unsigned(cb), &xraw[j]);
            }
          }
        } else {
        // Lane mapping: consecutive lanes take consecutive 16-byte quads of one node row, so a
        // warp reads whole 128-byte row segments (coalesced); quad qq of node n lands where its
        // 8-element group's hi (even qq) or lo (odd qq) operand lives — for shadow rows that is
        // exactly where the shadow already keeps it, for fp32 rows it is converted in place.
        constexpr int kq = MBX_KC / 4;
        const int nq = ((nn + 7) & ~7) * kq;  // columns past the last valid 8-group are never read
        const unsigned char* src_base = L.shadow ? P.shadow : reinterpret_cast<const unsigned char*>(P.arena);
#pragma unroll 1
        for (int j = 0; j < CPR; ++j) {
          const int k = (c_begin + j) * MBX_KC;
          const int p1 = (MBX_NPIECES > 1 && k >= MBX_PK0) ? 1 : 0;
          const int kin = k - (p1 ? MBX_PK0 : 0);
          unsigned char* xs = xsm + j * xstride;
          for (int g = gt; g < nq; g += MBX_LGATHER) {
            const int n = g / kq, qq = g - n * kq;
            const bool valid = n < nn;
            const unsigned char* src = src_base + (valid ? 4 * (rowbase[2 * n + p1] + kin + qq * 4) : 0);
            unsigned char* dst = xs + (n >> 3) * (MBX_KC * 16) + (n & 7) * 16 + ((qq >> 1) << 7) + ((qq & 1) ? xlo : 0);
            if (L.vec16) {
              cp_async16(dst, src, valid);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) cp_async4(dst + 4 * e, src + 4 * e, valid);
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&xraw[j])) : "memory");
        }
        }
        // Every row address of this tile is issued: look up the next tile's rows now (its
        // offset tables are static), off the critical path of the next gather.
        MBX_LSTAMP_T(64, lv, 9);
        named_sync(1, MBX_LGATHER);
        if (node0 + ngrp * nt < b) {
          fill_rowbase(L, node0 + ngrp * nt, nt);
          have_rb = true;
        } else if (lv + 1 < P.nlevels && grp * lvl(lv + 1).nt < lvl(lv + 1).b) {
          const TcLevel Ln = lvl(lv + 1);
          fill_rowbase(Ln, grp * Ln.nt, Ln.nt);
          have_rb = true;
        }
        constexpr int kb = MBX_KC / 8;
        const int ngroups8 = ((nn + 7) >> 3) * kb;
        const int l8 = gt & 7, g0 = gt >> 3;
#pragma unroll 1
        for (int j = 0; j < CPR; ++j) {
          if (L.img >= 0) {  // every barrier completes once per tile: pass xfull on
            __syncwarp();
            if (lane == 0) mbar_arrive(&xfull[j]);
            continue;
          }
          mbar_wait(&xraw[j], par);

          if (!L.shadow) {
            unsigned char* xs = xsm + j * xstride;
            for (int g = g0; g < ngroups8; g += MBX_LGATHER / 8) {
              const int m = g % kb, nb8 = g / kb;
              const unsigned off = unsigned(nb8 * (MBX_KC * 16) + m * 128 + l8 * 16);
              const float4 a = *reinterpret_cast<const float4*>(xs + off);
              const float4 bq = *reinterpret_cast<const float4*>(xs + xlo + off);
              const float v[8] = {a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w};
              unsigned short sp[8][3];
#pragma unroll
              for (int e = 0; e < 8; ++e) split_bf16(v[e], parts, sp[e]);
#pragma unroll
              for (int q = 0; q < 3; ++q) {
                if (q >= parts) break;
                uint4 w;  // low half of each word = the even element
                w.x = unsigned(sp[0][q]) | (unsigned(sp[1][q]) << 16);
                w.y = unsigned(sp[2][q]) | (unsigned(sp[3][q]) << 16);
                w.z = unsigned(sp[4][q]) | (unsigned(sp[5][q]) << 16);
                w.w = unsigned(sp[6][q]) | (unsigned(sp[7][q]) << 16);
                *reinterpret_cast<uint4*>(xs + q * xlo + off) = w;
              }
            }
          }
          // Chunk j is ready for the tensor core (async proxy): its MMAs overlap the next chunk.
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xfull[j]);
        }
        MBX_LSTAMP_T(64, lv, 7);
        // The tail's operands: off the gather -> MMA critical path, in flight during the MMAs and
        // the exchange.
        load_tail_operands();
      } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ----
        if (it == 0) mbar_wait(wfull, 0);
        const unsigned idesc =
            (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(nt >> 3) << 17) | (unsigned(MBX_M >> 4) << 24);
        const unsigned sbo = unsigned(MBX_KC * 16);
#pragma unroll 1
        for (int j = 0; j < CPR; ++j) {
          mbar_wait(L.img >= 0 ? &xraw[j] : &xfull[j], par);  // image chunks land by TMA (async proxy)
          tc_fence_after();
          const unsigned wa = smem_u32(wsm + j * wstage);
          const unsigned xa = smem_u32(xsm + j * xstride);
          const unsigned long long a0 = make_desc(wa, sbo), b0 = make_desc(xa, sbo);
          const unsigned long long a1 = make_desc(wa + wchunk, sbo), b1 = make_desc(xa + xlo, sbo);
          const unsigned long long a2 = make_desc(wa + 2 * wchunk, sbo), b2 = make_desc(xa + 2 * xlo, sbo);
#pragma unroll
          for (int ks = 0; ks < MBX_KC / 16; ++ks) {
            const unsigned long long step = (unsigned long long)(ks * 16);
            mma_bf16(tmem, a0 + step, b0 + step, idesc, (j | ks) ? 1u : 0u);
            if (parts > 1) {  // bf16x3: + hi.lo + lo.hi
              mma_bf16(tmem, a0 + step, b1 + step, idesc, 1u);
              mma_bf16(tmem, a1 + step, b0 + step, idesc, 1u);
            }
            if (parts > 2) {  // bf16x6: + hi.lo' + mid.mid + lo'.hi (the terms down to 2^-24)
              mma_bf16(tmem, a0 + step, b2 + step, idesc, 1u);
              mma_bf16(tmem, a1 + step, b1 + step, idesc, 1u);
              mma_bf16(tmem, a2 + step, b0 + step, idesc, 1u);
            }
          }
        }
        mma_commit(done);
        MBX_LSTAMP_T(32, lv, 11);
      }
      MBX_LSTAMP(lv, 1);
      mbar_wait(done, par);
      MBX_LSTAMP(lv, 2);
      __syncwarp();
      tc_fence_after();
#if MBX_LXCH == 0
      // ---- accumulators -> shared memory (the X region is free once the MMAs completed) ----
      {
        const int q = warp & 3, half = warp >> 2;
        const int row = q * 32 + lane;
        const int cols = nt / 2;
        for (int c0 = half * cols; c0 < (half + 1) * cols; c0 += 8) {
          float v[8];
          tmem_ld8(tmem + (unsigned(q * 32) << 16) + unsigned(c0), v);
#pragma unroll
          for (int k = 0; k < 8; ++k) stg[(c0 + k) * MBX_M + row] = v[k];
        }
      }
      MBX_LSTAMP(lv, 12);
      tc_fence_before();
      if (S > 1) {
        fence_async_smem();  // staged partials -> visible to the bulk-copy engine
        cluster_sync();      // every rank staged its partials, armed rbar, consumed the last tile
        MBX_LSTAMP(lv, 3);
        if (tid == 0) {
          const unsigned bytes = unsigned(ntr * MBX_M * 4);
          for (int r = 0; r < S; ++r) {
            if (r == int(rank)) continue;
            const int slot = int(rank) < r ? int(rank) : int(rank) - 1;
            unsigned dst, bar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(dst)
                         : "r"(smem_u32(recv + (size_t)slot * ntr * MBX_M)), "r"(r));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(rbar)), "r"(r));
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst),
                "r"(smem_u32(stg + (size_t)r * ntr * MBX_M)), "r"(bytes), "r"(bar)
                : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        mbar_wait(rbar, par);
      } else {
        __syncthreads();
      }
      // Per source rank, the base of its partials of this rank's nodes (own: staging; peers: recv).
      const float* pq[S];
#pragma unroll
      for (int q = 0; q < S; ++q)
        pq[q] = q == int(rank) ? stg + nloc0 * MBX_M : recv + (q < int(rank) ? q : q - 1) * ntr * MBX_M;
      auto pptr = [&](int q, int n, int col) -> const float* { return pq[q] + n * MBX_M + col; };
#else
      // ---- accumulators -> every rank's L2 slots (the own slice too: the reduction then reads
      // all S partials the same way, uniform and branch-free, every load in flight) ----
      // part layout: [tile parity][group][unit tile][destination rank][source rank][LLOC][128]
      float* pbase = P.part + ((size_t)(par * ngrp + grp) * gridDim.y + tile_u) * S * S * MBX_LLOC * MBX_M;
      {
        // Warp w reads TMEM lanes 32*(w%4).. (gate rows), every other 32-column block in one load
        // (one wait per 4 chunks of 8 nodes).
        const int q = warp & 3, half = warp >> 2;
        const int row = q * 32 + lane;
        const int nch = (nn + 7) >> 3;
        for (int c0 = half * 32; c0 < nch * 8; c0 += 64) {
          float v[32];
          tmem_ld32(tmem + (unsigned(q * 32) << 16) + unsigned(c0), v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ch = (c0 >> 3) + i;
            if (ch < nch) {
              const int r = ch % S, m0 = (ch / S) * 8;
              float* dst = pbase + ((size_t)(r * S + int(rank)) * MBX_LLOC + m0) * MBX_M + row;
#pragma unroll
              for (int k = 0; k < 8; ++k) __stcg(dst + k * MBX_M, v[8 * i + k]);
            }
          }
        }
      }
      MBX_LSTAMP(lv, 12);
      tc_fence_before();
      __syncthreads();
      MBX_LSTAMP(lv, 13);
      if (S > 1) {
        unsigned* flags = P.xflags + (grp * gridDim.y + tile_u) * S;
        if (tid < S && tid != int(rank)) red_release_add(flags + tid, 1u);
        MBX_LSTAMP(lv, 3);
        if (tid == 0) spin_until(flags + rank, unsigned(S - 1) * (it + 1));
        __syncthreads();
      }
      auto pptr = [&](int q, int n, int col) -> const float* {
        return pbase + ((size_t)(int(rank) * S + q) * MBX_LLOC + n) * MBX_M + col;
      };
#endif
      MBX_LSTAMP(lv, 4);
      // ---- sum the partials in rank order, run the tail, write the outputs ----
      // Every partial of every element is read before the first output store: through generic
      // pointers a store would order all later loads behind it (one L2 round trip per element).
      // Branch-free: invalid elements read node 0's (in-bounds) partials and are never stored, so
      // every element's loads issue together.
      float gsum[MBX_LEPT][MBX_G];
#pragma unroll
      for (int t = 0; t < MBX_LEPT; t += MBX_LQ) {
        int n, u;
        elem(t, n, u);  // the quad's first element
        const int nv = (n < nloc && loc_col(n) < nn) ? n : 0;
#pragma unroll
        for (int gi = 0; gi < MBX_G; ++gi) {
          const int col = gi * MBX_UC + u;
#if MBX_LQ == 2
          float2 pv[S];
#pragma unroll
          for (int q = 0; q < S; ++q) pv[q] = ld_partial2(pptr(q, nv, col));
          float2 acc = pv[0];
#pragma unroll
          for (int q = 1; q < S; ++q) {
            acc.x = acc.x + pv[q].x;
            acc.y = acc.y + pv[q].y;
          }
          gsum[t][gi] = acc.x;
          gsum[t + 1][gi] = acc.y;
#else
          float pv[S];
#pragma unroll
          for (int q = 0; q < S; ++q) pv[q] = ld_partial(pptr(q, nv, col));
          float acc = pv[0];
#pragma unroll
          for (int q = 1; q < S; ++q) acc = acc + pv[q];
          gsum[t][gi] = acc;
#endif
        }
      }
      MBX_LSTAMP(lv, 15);
      // Every element's tail first (independent activation chains the scheduler can interleave),
      // then the stores: a store between two elements would keep their chains apart.
      float ov[MBX_LEPT][MBX_NOUT];
#pragma unroll
      for (int t = 0; t < MBX_LEPT; ++t)
        if (any_elem(t)) mbx_tail(gsum[t], lreg[t], ov[t]);
      MBX_LSTAMP(lv, 13);
      const unsigned smask = L.shadow_out;
      if (smask == 0 && L.img_slot < 0) {  // plain outputs (warp-uniform)
#pragma unroll
        for (int t = 0; t < MBX_LEPT; ++t) {
          int n, u;
          elem(t, n, u);
          if (n < nloc && loc_col(n) < nn) {
            const long long node = node0 + loc_col(n);
#pragma unroll
            for (int k = 0; k < MBX_NOUT; ++k) P.arena[obase[k] + node * MBX_U + tile_u * MBX_UC + u] = ov[t][k];
          }
        }
      } else {
#pragma unroll
      for (int t = 0; t < MBX_LEPT; ++t) {
        int n, u;
        elem(t, n, u);
        if (n < nloc && loc_col(n) < nn) {
          const long long node = node0 + loc_col(n);
          const int ug = tile_u * MBX_UC + u;
#pragma unroll
          for (int k = 0; k < MBX_NOUT; ++k) {
            const long long o = obase[k] + node * MBX_U + ug;
            P.arena[o] = ov[t][k];
            if ((smask >> k) & 1u) store_shadow(P.shadow, o, ov[t][k]);
            if (k == L.img_slot) {  // scattered into the consumer level's operand image
              const int4 d = dreg[t];
              if (d.y >= 0) {
                int po;
                const long long a = img_addr(d, ug, &po);
                const int np = parts;  // the consumer's image has this launch's parts
                unsigned short sp[3];
                split_bf16(ov[t][k], np, sp);
#pragma unroll
                for (int q = 0; q < 3; ++q)  // static indices: sp stays in registers
                  if (q < np) *reinterpret_cast<unsigned short*>(P.img + a + q * po) = sp[q];
              }
            }
          }
        }
      }
      }
      MBX_LSTAMP(lv, 10);
#if MBX_LXCH == 0
      if (S > 1 && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
      __syncthreads();  // stg / recv / TMEM free for the next tile
      tc_fence_after();
      MBX_LSTAMP(lv, 5);
    }
    // This CTA's part of level lv is written: release it to the level's consumers (the
    // __syncthreads orders every thread's stores before thread 0's release).
    if (lv + 1 < P.nlevels) {
      __syncthreads();
      if (tid == 0) red_release_add(P.ready + tile_u * MBX_READY_STRIDE, 1u);
    }
  }
#if MBX_LXCH == 0
  if (S > 1) cluster_sync();  // no peer still pushes into this CTA's shared memory
#else
  // Every increment of this CTA's exchange counter happened before its last wait: reset it for
  // the next launch (stream order makes launches sequential).
  if (S > 1 && tid == 0 && it > 0) P.xflags[(grp * gridDim.y + tile_u) * S + rank] = 0u;
#endif
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}
#endif  // MBX_LEVELS_KERNEL


#ifdef MBX_SMALL_KERNEL
// mbx_exact_gate — bit-exact CUDA-core path of the gate plans: the FP32 context's cells, the
// decision-feeding cells (NestedRNN's, always exact), and plans with few output columns (U x G
// <= 64, e.g. the TreeLSTM classifier relu(h . c_wt + cbias), where tensor-core tiles would be
// mostly padding) in every precision.  Every output is the reference's sequential chain
// acc = acc + x[p] * w[p][j] over p ascending with separately rounded multiply and add
// (proj/src/backend.cpp:116-131), the tail with the glibc-exact activations.
//   grid = (node tiles of MBX_SNPC nodes, unit slices of MBX_SUC units); thread = (node, unit),
//   MBX_G independent chains.  The weight slice and the nodes' rows stream through shared memory
//   in K chunks of MBX_SKB through a ring of MBX_SST cp.async stages (all of K at once when it
//   fits: the kernel is load-latency bound, each chunk in flight hides one L2 round trip), so no
//   operand is read twice from L2 by one CTA and the chains run from shared memory.
#define MBX_SNT (MBX_SNPC * MBX_SUC)
#ifndef MBX_STHREADS
#define MBX_STHREADS MBX_THREADS  // block size (narrow variants: fewer threads, more CTAs)
#endif
extern "C" __global__ void __launch_bounds__(MBX_STHREADS) mbx_small_dense(const __grid_constant__ SmallArgs P) {
  extern __shared__ __align__(16) float sms[];
  constexpr int K = MBX_K, U = MBX_U, G = MBX_G, NPC = MBX_SNPC, UC = MBX_SUC, KB = MBX_SKB;
  // Weight chunk transposed, [gate][unit][KB + 4]: a thread's column is contiguous along K, so
  // its operands load 4 at a time (rows 4 floats apart: the transposing 4-byte copies of 8
  // consecutive units land in different banks).
  constexpr int KBP = KB + 4;
  constexpr int WCH = G * UC * KBP, XCH = NPC * KB, BUF = WCH + XCH;
  static_assert(K % KB == 0 && KB % 8 == 0, "K chunking");
  const int tid = threadIdx.x;
  // Phase stamps (profiling builds of the host only: P.stamps is null on every measured path).
  auto stamp = [&](int i) {
    if (P.stamps && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.stamps[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + i] = t;
    }
  };
  stamp(0);
  const int node0 = blockIdx.x * NPC;
  const int u0 = blockIdx.y * UC;
  const int nn = min(NPC, P.b - node0);
  // PDL: every input (weights included: they may be a hoisted prefix's output) after the wait.
  mbx_gen::pdl_wait();
  mbx_gen::pdl_launch_dependents();
  stamp(1);
  __shared__ long long rowb[NPC][2];
  // Weight bases into registers first: through generic pointers the compiler cannot prove the
  // shared-memory stores leave the offset table alone and would re-read it every iteration.
  const float* wsrc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) wsrc[g] = P.arena + __ldg(P.shared_off + P.w_idx[g]) + u0;
  for (int i = tid; i < nn * 2; i += MBX_STHREADS) {
    const int n = i >> 1, pc = i & 1;
    long long base = 0;
    if (pc < MBX_NPIECES)
      base = (P.piece_kind[pc] == 0 ? P.shared_off[P.piece_idx[pc]]
                                    : P.batched_off[(long long)(node0 + n) * P.nb + P.piece_idx[pc]]) +
             P.piece_off[pc] - (pc ? MBX_PK0 : 0);
    rowb[n][pc] = base;
  }
  __syncthreads();
  // Single-chunk launches (all of K staged at once: the narrow variants, decision heads): the
  // weight slice comes in as VW-float vector loads of a row's unit run, all in flight from
  // registers, then scattered into the transposed rows; node rows with 16-byte copies where
  // aligned.  (A warp's staging is otherwise a long serial stream of 4-byte copies: with one or
  // two warps per SM that stream, not bandwidth, sets the time.)
  constexpr int NST0 = MBX_SST;
  constexpr int VW = UC % 4 == 0 ? 4 : (UC % 2 == 0 ? 2 : 1);
  constexpr int NVG = (KB * UC / VW + MBX_STHREADS - 1) / MBX_STHREADS;  // vectors per thread per gate
  constexpr bool REG_STAGE = NST0 == 1 && VW > 1 && G * NVG * VW <= 64;
  auto stage_direct = [&](float* buf) {
    float wr[G][NVG][VW];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int j = 0; j < NVG; ++j) {
        const int v = tid + j * MBX_STHREADS, r = v / (UC / VW), q = v - r * (UC / VW);
        if (v < KB * UC / VW) {
          const float* src = wsrc[g] + (long long)r * U + q * VW;
          if (VW == 4) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(src));
            wr[g][j][0] = x.x, wr[g][j][VW > 1 ? 1 : 0] = x.y, wr[g][j][VW > 2 ? 2 : 0] = x.z, wr[g][j][VW > 3 ? 3 : 0] = x.w;
          } else {
            const float2 x = __ldg(reinterpret_cast<const float2*>(src));
            wr[g][j][0] = x.x, wr[g][j][VW > 1 ? 1 : 0] = x.y;
          }
        }
      }
    for (int n = 0; n < nn; ++n)
      for (int pc = 0; pc < MBX_NPIECES; ++pc) {
        const int k0 = pc ? MBX_PK0 : 0, k1 = pc ? K : (MBX_NPIECES > 1 ? MBX_PK0 : K);
        const float* row = P.arena + rowb[n][pc];
        float* dst = buf + WCH + n * KB;
        if (((rowb[n][pc] + k0) & 3) == 0 && (k0 & 3) == 0 && (k1 & 3) == 0) {
          for (int k = k0 + 4 * tid; k < k1; k += 4 * MBX_STHREADS) mbx_gen::cp_async16(dst + k, row + k, true);
        } else {
          for (int k = k0 + tid; k < k1; k += MBX_STHREADS) mbx_gen::cp_async4(dst + k, row + k, true);
        }
      }
    mbx_gen::cp_async_commit();
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int j = 0; j < NVG; ++j) {
        const int v = tid + j * MBX_STHREADS, r = v / (UC / VW), q = v - r * (UC / VW);
        if (v < KB * UC / VW)
#pragma unroll
          for (int e = 0; e < VW; ++e) buf[(g * UC + q * VW + e) * KBP + r] = wr[g][j][e];
      }
  };
  auto stage = [&](int c, float* buf) {
    const int k0 = c * KB;
    // cp.async: every copy in flight at once (a load -> store loop through registers would be
    // serialised by the possible aliasing of the generic pointers).
#pragma unroll
    for (int g = 0; g < G; ++g)
      for (int i = tid; i < KB * UC; i += MBX_STHREADS) {
        const int r = i / UC, q = i - r * UC;
        mbx_gen::cp_async4(buf + (g * UC + q) * KBP + r, wsrc[g] + (long long)(k0 + r) * U + q, true);
      }
    for (int i = tid; i < nn * KB; i += MBX_STHREADS) {
      const int n = i / KB, k = k0 + (i - n * KB);
      const int pc = (MBX_NPIECES > 1 && k >= MBX_PK0) ? 1 : 0;
      mbx_gen::cp_async4(buf + WCH + i, P.arena + rowb[n][pc] + k, true);
    }
    mbx_gen::cp_async_commit();
  };
  // MBX_SGS = G: each gate's chain on its own thread (thread = (gate, node, unit), G x more warps
  // issuing: a thread's chain is a single instruction stream, so few threads with G chains each
  // are issue-latency bound); the tail then reads the G sums back from shared memory.
  // MBX_SGS = 1: one thread per (node, unit) with all G chains.
#ifndef MBX_SGS
#define MBX_SGS 1
#endif
  constexpr int GS = MBX_SGS, GT = G / GS;  // gates split over threads, gates per thread
  static_assert(G % GS == 0 && MBX_SNT * GS <= MBX_STHREADS, "gate split");
  const int gq = tid / MBX_SNT, tr = tid - gq * MBX_SNT;  // gate group, (node, unit) index
  const int n = tr / UC, u = tr - n * UC;
  const bool active = gq < GS && n < nn && u0 + u < U;
  float g[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) g[gi] = 0.0f;
  // The tail's other operands (e.g. the children's cell states) are loaded now, by the threads
  // that will run the tail: their latency hides under the staging and the chains.
  const long long node = node0 + n;
  const int ug = u0 + u;
  float l[MBX_NLOADS > 0 ? MBX_NLOADS : 1];
  if (active && gq == 0) {
#pragma unroll
    for (int j = 0; j < MBX_NLOADS; ++j) {
      const TcLoad& d = P.loads[j];
      const long long base = d.kind == 1 ? P.batched_off[node * P.nb + d.idx] : P.shared_off[d.idx];
      l[j] = P.arena[base + d.off + ug];
    }
  }
  constexpr int NCH = K / KB, NST = MBX_SST, D = NST - 1;  // D chunks in flight ahead
  static_assert(NST >= 1 && (NST > 1 || NCH == 1), "stages");
  // One commit group per chunk (empty past the end) so the wait count is the same every step.
  // (The vector path needs 16- / 8-byte aligned weight runs: every gate's base and U.)
  bool direct = REG_STAGE && (U % VW) == 0;
#pragma unroll
  for (int g = 0; g < G; ++g) direct = direct && (reinterpret_cast<unsigned long long>(wsrc[g]) % (VW * 4)) == 0;
  if (D == 0) {
    if (direct) stage_direct(sms);
    else stage(0, sms);
  }
#pragma unroll 1
  for (int c = 0; c < D; ++c) {
    if (c < NCH) stage(c, sms + c * BUF);
    else mbx_gen::cp_async_commit();
  }
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    float* cur = sms + (c % NST) * BUF;
    if (D > 0) {
      if (c + D < NCH) stage(c + D, sms + ((c + D) % NST) * BUF);  // the buffer computed at c - 1
      else mbx_gen::cp_async_commit();
    }
    mbx_gen::cp_async_wait<D>();
    __syncthreads();
    if (c == 0) stamp(2);
    if (active) {
      const float4* x4 = reinterpret_cast<const float4*>(cur + WCH + n * KB);
      const float* w = cur + u * KBP;
      // Blocks of 8 p: operands (16-byte loads) and products first (independent), then the 8
      // dependent adds of each chain in p order — the add chain is the only serial part.
      // Unrolled 4 blocks deep so the next blocks' loads and products overlap this block's adds.
#pragma unroll 4
      for (int p0 = 0; p0 < KB; p0 += 8) {
        const float4 xa = x4[p0 >> 2], xb = x4[(p0 >> 2) + 1];
        const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
        for (int gj = 0; gj < GT; ++gj) {
          const int gi = gq * GT + gj;
          const float4* w4 = reinterpret_cast<const float4*>(w + gi * UC * KBP + p0);
          const float4 wa = w4[0], wb = w4[1];
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
          float pr[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pr[q] = mbx_libm::fmul(xv[q], wv[q]);
#pragma unroll
          for (int q = 0; q < 8; ++q) g[gj] = mbx_libm::fadd(g[gj], pr[q]);
        }
      }
    }
    __syncthreads();  // the buffer is refilled NST chunks on
  }
  stamp(3);
  if (GS > 1) {  // gather the G sums of (node, unit) on its gate-group-0 thread
    float* gsm = sms;  // [G][MBX_SNT] (the staging buffers are free after the last chunk)
    if (active)
#pragma unroll
      for (int gj = 0; gj < GT; ++gj) gsm[(gq * GT + gj) * MBX_SNT + tr] = g[gj];
    __syncthreads();
    if (gq != 0 || !active) return;
#pragma unroll
    for (int gi = 0; gi < G; ++gi) g[gi] = gsm[gi * MBX_SNT + tr];
  }
  if (!active) return;
  float o[MBX_NOUT];
  stamp(4);
  mbx_tail_exact(g, l, o);
#pragma unroll
  for (int k = 0; k < MBX_NOUT; ++k)
    P.arena[(P.out_node ? P.out_node[node * MBX_NOUT + k] : P.out_base[k] + node * U) + ug] = o[k];
  stamp(5);
}
#endif  // MBX_SMALL_KERNEL

#ifdef MBX_POINTWISE_KERNEL
// One thread per (node, element); the offset-table lookups are shared by the E elements of a
// node.  FAST selects the fast activations (tensor-core precisions).
template <bool FAST, int V>
__device__ __forceinline__ void mbx_pointwise_body(const PwArgs& P) {
  // PDL: launched while the predecessor drains; its outputs are read only after the wait.
  mbx_gen::pdl_wait();
  mbx_gen::pdl_launch_dependents();
  // V = 4: each thread takes 4 consecutive elements with 16-byte loads and stores (the host
  // checked that every row involved is 16-byte aligned); one offset lookup per 4 elements.
  constexpr int EV = MBX_PW_E / V;
  const long long total = (long long)P.b * EV;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long node = idx / EV;
    const int e = int(idx - node * EV) * V;
    float l[V][MBX_NLOADS > 0 ? MBX_NLOADS : 1];
#pragma unroll
    for (int j = 0; j < MBX_NLOADS; ++j) {
      const TcLoad& d = P.loads[j];
      const long long base = d.kind == 1 ? P.batched_off[node * P.nb + d.idx] : P.shared_off[d.idx];
      if (V == 4) {
        const float4 v = *reinterpret_cast<const float4*>(P.arena + base + d.off + e);
        l[0][j] = v.x;
        l[V > 1 ? 1 : 0][j] = v.y;
        l[V > 2 ? 2 : 0][j] = v.z;
        l[V > 3 ? 3 : 0][j] = v.w;
      } else {
        l[0][j] = P.arena[base + d.off + e];
      }
    }
    float o[V][MBX_NOUT];
#pragma unroll
    for (int w = 0; w < V; ++w) {
      if (FAST) mbx_pw_tail_fast(l[w], o[w]);
      else mbx_pw_tail(l[w], o[w]);
    }
#pragma unroll
    for (int k = 0; k < MBX_NOUT; ++k) {
      const long long off = P.out_base[k] + node * MBX_PW_E + e;
      float* dst = P.arena + off;
      if (V == 4) {
        const float4 v = make_float4(o[0][k], o[V > 1 ? 1 : 0][k], o[V > 2 ? 2 : 0][k], o[V > 3 ? 3 : 0][k]);
        *reinterpret_cast<float4*>(dst) = v;
        // Split-bf16 shadow of the 4 values (half an 8-float group; see mbx_tc_levels): the
        // later tensor-core level that gathers this row reads it MMA-ready.
        if ((P.shadow_out >> k) & 1u) {
          const float x[4] = {v.x, v.y, v.z, v.w};
          unsigned hp[2], lp[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            hp[q] = mbx_gen::pack_bf16x2(x[2 * q], x[2 * q + 1]);
            const float h0 = __uint_as_float(hp[q] << 16), h1 = __uint_as_float(hp[q] & 0xffff0000u);
            lp[q] = mbx_gen::pack_bf16x2(x[2 * q] - h0, x[2 * q + 1] - h1);
          }
          unsigned char* sp = P.shadow + 4 * off - 2 * (off & 7);
          *reinterpret_cast<uint2*>(sp) = make_uint2(hp[0], hp[1]);
          *reinterpret_cast<uint2*>(sp + 16) = make_uint2(lp[0], lp[1]);
        }
        if (k == P.img_slot) {  // scattered into the consumer level's operand image
          const int4 d = P.img_dst[node];
          if (d.y >= 0) {
            const float x[4] = {v.x, v.y, v.z, v.w};
            const int np = mbx_gen::img_parts(d);
            unsigned short sp[4][3];
#pragma unroll
            for (int q = 0; q < 4; ++q) mbx_gen::split_bf16(x[q], np, sp[q]);
            int po;
            const long long a = mbx_gen::img_addr(d, e, &po);
#pragma unroll
            for (int q = 0; q < 3; ++q)  // static indices: sp stays in registers
              if (q < np)
                *reinterpret_cast<uint2*>(P.img + a + q * po) = make_uint2(unsigned(sp[0][q]) | (unsigned(sp[1][q]) << 16),
                                                                         unsigned(sp[2][q]) | (unsigned(sp[3][q]) << 16));
          }
        }
      } else {
        *dst = o[0][k];
      }
    }
  }
}
extern "C" __global__ void __launch_bounds__(256) mbx_pointwise(const __grid_constant__ PwArgs P) {
  mbx_pointwise_body<false, 1>(P);
}
extern "C" __global__ void __launch_bounds__(256) mbx_pointwise_fast(const __grid_constant__ PwArgs P) {
  mbx_pointwise_body<true, 1>(P);
}
#if MBX_PW_E % 4 == 0
extern "C" __global__ void __launch_bounds__(256) mbx_pointwise4(const __grid_constant__ PwArgs P) {
  mbx_pointwise_body<false, 4>(P);
}
extern "C" __global__ void __launch_bounds__(256) mbx_pointwise_fast4(const __grid_constant__ PwArgs P) {
  mbx_pointwise_body<true, 4>(P);
}
#endif
#endif  // MBX_POINTWISE_KERNEL
