// Microbenchmark: per-SM ingest of an L2-resident buffer with cp.async.bulk (1D bulk copy,
// mbarrier ring) vs plain 16-byte loads.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void bulk_kernel(const uint8_t* src, size_t src_bytes, int chunk, int stages, int iters, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  size_t off = (size_t(blockIdx.x) * 7919 * chunk) % (src_bytes - chunk);
  off &= ~size_t(127);
  for (int i = 0; i < iters + stages; ++i) {
    const int s = i % stages;
    if (i >= stages) {
      uint32_t ph = ((i / stages) - 1) & 1;
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(s32(&bar[s])), "r"(ph));
    }
    if (i < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(sm + s * chunk)),
                   "l"(src + off), "r"(chunk), "r"(s32(&bar[s])));
      off = (off + chunk) % (src_bytes - chunk);
      off &= ~size_t(127);
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[blockIdx.x] = t1 - t0;
}

__global__ void ldg_kernel(const uint4* src, size_t n16, int iters, int per_iter16, unsigned long long* out, uint4* sink) {
  unsigned long long t0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint4 acc = make_uint4(0, 0, 0, 0);
  size_t base = (size_t(blockIdx.x) * 7919 * per_iter16) % (n16 - per_iter16);
  for (int i = 0; i < iters; ++i) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      size_t idx = base + threadIdx.x + u * blockDim.x;
      v[u] = __ldg(src + (idx % n16));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    base = (base + per_iter16) % (n16 - per_iter16);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  size_t bytes = 8 << 20;  // 8 MiB, L2-resident after the first pass
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* out;
  cudaMallocManaged(&out, 1024 * 8);
  uint4* sink;
  cudaMalloc(&sink, 64);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int grid : {1, 16, 148}) {
    for (int chunk : {4096, 16384, 32768}) {
      for (int stages : {2, 4, 6}) {
        if (chunk * stages > 200 * 1024) continue;
        int iters = 64;
        for (int rep = 0; rep < 2; ++rep) bulk_kernel<<<grid, 32, chunk * stages + 64>>>(src, bytes, chunk, stages, iters, out);
        cudaDeviceSynchronize();
        double mx = 0;
        for (int b = 0; b < grid; ++b) mx = mx > out[b] ? mx : out[b];
        printf("bulk grid %3d chunk %6d stages %d: %.2f us, per-SM %.1f GB/s, total %.2f TB/s\n", grid, chunk, stages, mx / 1e3,
               double(chunk) * iters / mx, double(chunk) * iters * grid / mx / 1e3);
      }
    }
  }
  for (int grid : {1, 16, 148}) {
    int threads = 256, per_iter16 = threads * 8;
    int iters = 64;
    for (int rep = 0; rep < 2; ++rep) ldg_kernel<<<grid, threads>>>((const uint4*)src, bytes / 16, iters, per_iter16, out, sink);
    cudaDeviceSynchronize();
    double mx = 0;
    for (int b = 0; b < grid; ++b) mx = mx > out[b] ? mx : out[b];
    printf("ldg  grid %3d 256 thr x 8 x 16B: %.2f us, per-SM %.1f GB/s, total %.2f TB/s\n", grid, mx / 1e3,
           double(per_iter16) * 16 * iters / mx, double(per_iter16) * 16 * iters * grid / mx / 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
