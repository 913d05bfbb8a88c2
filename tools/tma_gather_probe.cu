// Microbenchmark / correctness probe: TMA tile::gather4 of arbitrary bf16 rows into the
// SWIZZLE_128B K-major layout, consumed by tcgen05.mma as the B operand (N = gathered rows),
// with A (M = 128) in the no-swizzle canonical layout the levels kernel uses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_gather_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int M = 128, KS = 128, W = 512;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ unsigned long long desc_noswz(unsigned saddr, unsigned sbo) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3FFF);
  d |= (unsigned long long)((128u >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  return d;
}
__device__ __forceinline__ unsigned long long desc_sw128(unsigned saddr) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3FFF);
  d |= (unsigned long long)(1u) << 16;               // LBO (unused for swizzled K-major)
  d |= (unsigned long long)((1024u >> 4) & 0x3FFF) << 32;  // SBO: 8 rows x 128 B
  d |= 1ull << 46;
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

struct Args {
  const unsigned char* apack;  // [KS/32 chunks][128 x 32] canonical no-swizzle bf16
  const int* idx;              // [nt] row ids
  int nt, k0;
  float* out;                  // [nt][128]
  unsigned long long* cycles;
  int issuers;
  int tile;
};

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tmap,
                                                const __grid_constant__ CUtensorMap tmap4,
                                                const __grid_constant__ Args P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* asm_ = smem;                 // 128 x 128 bf16 = 32 KB
  unsigned char* bsm = smem + 32768;          // 2 boxes x nt x 128 B
  __shared__ unsigned long long bar, done;
  __shared__ unsigned tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nt = P.nt;
  for (int i = tid; i < 32768 / 16; i += 128)
    reinterpret_cast<uint4*>(asm_)[i] = reinterpret_cast<const uint4*>(P.apack)[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tslot;
  // Three rounds (the first is cold): issuers = the first P.issuers lanes of warp 0..3 (one
  // lane per warp), each issuing every issuers-th gather4.
  unsigned long long t0 = 0;
  for (int round = 0; round < 3; ++round) {
    __syncthreads();
    t0 = clock64();
    const int nis = P.issuers;
    const int me = (tid & 31) == 0 ? warp : -1;
    if (tid == 0) {
      const unsigned bytes = unsigned(2 * nt * 128);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    }
    __syncthreads();
    if (me >= 0 && me < nis) {
      int k = 0;
      for (int b = 0; b < 2; ++b)
        for (int q = 0; q < nt / 4; ++q, ++k) {
          if (k % nis != me) continue;
          const unsigned dst = smem_u32(bsm + b * nt * 128 + q * 512);
          if (P.tile) {  // comparison: plain 2D tile load of 4 consecutive rows (not the same data)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                "l"(&tmap4), "r"(P.k0 + 64 * b), "r"(P.idx[4 * q]), "r"(smem_u32(&bar))
                : "memory");
            continue;
          }
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
              "l"(&tmap), "r"(P.k0 + 64 * b), "r"(P.idx[4 * q]), "r"(P.idx[4 * q + 1]), "r"(P.idx[4 * q + 2]),
              "r"(P.idx[4 * q + 3]), "r"(smem_u32(&bar))
              : "memory");
        }
    }
    if (tid == 0) {
      asm volatile(
          "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(
              smem_u32(&bar)), "r"(round & 1)
          : "memory");
      P.cycles[round] = clock64() - t0;
    }
  }
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned idesc = (1u << 4) | (1u << 7) | (1u << 10) | (unsigned(nt >> 3) << 17) | (unsigned(M >> 4) << 24);
    for (int kk = 0; kk < KS; kk += 16) {
      const int j = kk / 32, s = (kk % 32) / 16;
      const unsigned long long a = desc_noswz(smem_u32(asm_ + j * (128 * 32 * 2) + s * 256), 32 * 16);
      const int b = kk / 64, ks = (kk % 64) / 16;
      const unsigned long long bd = desc_sw128(smem_u32(bsm + b * nt * 128 + ks * 32));
      const unsigned acc = kk ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(a), "l"(bd), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(
          smem_u32(&done))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < nt; c0 += 8) {
    unsigned r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + (unsigned(warp * 32) << 16) + unsigned(c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 8; ++k) P.out[(c0 + k) * M + row] = __uint_as_float(r[k]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 3000;
  std::mt19937 rng(5);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<__nv_bfloat16> hrows(size_t(R) * W);
  for (auto& x : hrows) x = __float2bfloat16(U(rng));
  std::vector<float> a(M * KS);
  for (auto& x : a) x = __bfloat162float(__float2bfloat16(U(rng)));
  // canonical no-swizzle K-major A: [chunk][r>>3][k>>3 in chunk][r&7][k&7]
  std::vector<__nv_bfloat16> apack(M * KS);
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < KS; ++k) {
      const int j = k / 32, kk = k % 32;
      const size_t off = size_t(j) * (M * 32) * 2 + (r >> 3) * (32 * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2;
      apack[off / 2] = __float2bfloat16(a[r * KS + k]);
    }
  void *d_rows, *d_apack;
  CK(cudaMalloc(&d_rows, hrows.size() * 2));
  CK(cudaMemcpy(d_rows, hrows.data(), hrows.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_apack, apack.size() * 2));
  CK(cudaMemcpy(d_apack, apack.data(), apack.size() * 2, cudaMemcpyHostToDevice));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {cuuint64_t(W), cuuint64_t(R)};
  cuuint64_t gstride[1] = {cuuint64_t(W) * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d_rows, gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode: %d\n", int(cr));
  CUtensorMap tmap4;
  cuuint32_t box4[2] = {64, 4};
  cr = enc(&tmap4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d_rows, gdim, gstride, box4, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode tile4: %d\n", int(cr));
  // Overlapping-row variant (row stride 16 B < row size): does the encoder accept it?
  {
    CUtensorMap t2;
    cuuint64_t g2[2] = {64, cuuint64_t(R) * W / 8};
    cuuint64_t s2[1] = {16};
    CUresult c2 = enc(&t2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d_rows, g2, s2, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode overlapping rows (stride 16 B): %d\n", int(c2));
  }
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 2 * 256 * 128 + 1024));
  for (int tile : {0, 1}) for (int issuers : {1, 4}) for (int nt : {16, 64, 256}) {
    for (int k0 : {0}) {
      std::vector<int> idx(nt);
      for (auto& x : idx) x = int(rng() % R);
      int* d_idx;
      float* d_out;
      unsigned long long* d_cyc;
      CK(cudaMalloc(&d_idx, nt * 4));
      CK(cudaMemcpy(d_idx, idx.data(), nt * 4, cudaMemcpyHostToDevice));
      CK(cudaMalloc(&d_out, size_t(nt) * M * 4));
      CK(cudaMalloc(&d_cyc, 24));
      Args P{static_cast<unsigned char*>(d_apack), d_idx, nt, k0, d_out, d_cyc, issuers, tile};
      probe<<<1, 128, 32768 + 2 * 256 * 128 + 1024>>>(tmap, tmap4, P);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      std::vector<float> out(size_t(nt) * M);
      unsigned long long cyc[3] = {0, 0, 0};
      CK(cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(cyc, d_cyc, 24, cudaMemcpyDeviceToHost));
      double maxerr = 0;
      for (int n = 0; n < nt; ++n)
        for (int m = 0; m < M; ++m) {
          double ref = 0;
          for (int k = 0; k < KS; ++k) ref += double(a[m * KS + k]) * double(__bfloat162float(hrows[size_t(idx[n]) * W + k0 + k]));
          maxerr = std::max(maxerr, std::fabs(ref - out[size_t(n) * M + m]));
        }
      std::printf("tile=%d issuers=%d nt=%3d k0=%3d: max abs err %.3e, gather us: cold %.2f warm %.2f %.2f\n", tile, issuers, nt, k0,
                  maxerr, cyc[0] / 1965.0, cyc[1] / 1965.0, cyc[2] / 1965.0);
      cudaFree(d_idx);
      cudaFree(d_out);
      cudaFree(d_cyc);
    }
  }
  return 0;
}
