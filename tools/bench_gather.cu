// Microbenchmark: per-SM throughput of gathering scattered 128-byte row segments (the tensor-core
// kernels' node-row gather) from an L2-resident buffer into shared memory, three ways:
//   ldgsts : cp.async 16 B per thread (LDGSTS), completion via cp.async.wait_group
//   ldg    : ld.global.v4 into registers, st.shared
//   bulk   : cp.async.bulk (TMA bulk engine) per 128 B row, completion on an mbarrier
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_gather tools/bench_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

constexpr int kRows = 128;        // rows per chunk (NT)
constexpr int kRowBytes = 128;    // bytes per row segment (KC = 32 floats)
constexpr int kChunk = kRows * kRowBytes;

__global__ void ldgsts_kernel(const float* buf, const int* rows, int nrows_total, int iters, int threads_used,
                              unsigned long long* out, int mode) {
  // mode bits: 1 zfill form, 2 rows offset by 16 B (not line aligned), 4 all CTAs read the same rows
  __shared__ __align__(128) uint8_t sm[2 * kChunk];
  __shared__ int srow[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) srow[i] = rows[((mode & 4) ? 0 : blockIdx.x * 131 + i) % nrows_total + ((mode & 4) ? i : 0)];
  __syncthreads();
  unsigned long long c0 = clock64();
  const int shift = (mode & 2) ? 4 : 0;
  if (t < threads_used) {
    for (int i = 0; i < iters; ++i) {
      uint8_t* dst = sm + (i & 1) * kChunk;
      for (int q = t; q < kRows * 8; q += threads_used) {
        const int r = q >> 3, qq = q & 7;
        const float* src = buf + size_t(srow[(i * 17 + r) & 1023]) * 512 + qq * 4 + shift;
        if (mode & 1)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s32(dst + r * kRowBytes + qq * 16)), "l"(src), "r"(16)
                       : "memory");
        else
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(dst + r * kRowBytes + qq * 16)), "l"(src)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x] = clock64() - c0;
}

__global__ void ldg_kernel(const float* buf, const int* rows, int nrows_total, int iters, int threads_used,
                           unsigned long long* out) {
  __shared__ __align__(128) uint8_t sm[kChunk];
  __shared__ int srow[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) srow[i] = rows[(blockIdx.x * 131 + i) % nrows_total];
  __syncthreads();
  unsigned long long c0 = clock64();
  if (t < threads_used) {
    for (int i = 0; i < iters; ++i) {
      float4 v[16];
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = t + j * threads_used;
        if (q < kRows * 8) {
          const int r = q >> 3, qq = q & 7;
          v[j] = __ldcg(reinterpret_cast<const float4*>(buf + size_t(srow[(i * 17 + r) & 1023]) * 512 + qq * 4));
          ++cnt;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = t + j * threads_used;
        if (q < kRows * 8) *reinterpret_cast<float4*>(sm + (q >> 3) * kRowBytes + (q & 7) * 16) = v[j];
      }
    }
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x] = clock64() - c0;
  if (sm[t] == 123) out[1023] = 1;  // keep the stores alive
}

__global__ void bulk_kernel(const float* buf, const int* rows, int nrows_total, int iters, unsigned long long* out) {
  __shared__ __align__(128) uint8_t sm[2 * kChunk];
  __shared__ uint64_t bar[4];
  __shared__ int srow[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) srow[i] = rows[(blockIdx.x * 131 + i) % nrows_total];
  if (t == 0) {
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned long long c0 = clock64();
  if (t < 32) {
    for (int i = 0; i < iters + 4; ++i) {
      const int s = i & 3;
      if (i >= 4) {
        if (t == 0) {
          uint32_t ph = ((i >> 2) - 1) & 1;
          asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                           s32(&bar[s])),
                       "r"(ph));
        }
        __syncwarp();
      }
      if (i < iters) {
        if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(kChunk));
        __syncwarp();
        for (int r = t; r < kRows; r += 32) {
          const float* src = buf + size_t(srow[(i * 17 + r) & 1023]) * 512;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           s32(sm + (s & 1) * kChunk + r * kRowBytes)),
                       "l"(src), "r"(kRowBytes), "r"(s32(&bar[s]))
                       : "memory");
        }
      }
    }
  }
  __syncthreads();
  if (t == 0) out[blockIdx.x] = clock64() - c0;
}

int main() {
  const int nrows_total = 4096;  // 4096 rows x 2 KB = 8 MB, L2-resident
  float* buf;
  cudaMalloc(&buf, size_t(nrows_total) * 512 * 4);
  cudaMemset(buf, 0, size_t(nrows_total) * 512 * 4);
  int* rows;
  cudaMallocManaged(&rows, nrows_total * 4);
  for (int i = 0; i < nrows_total; ++i) rows[i] = (i * 2654435761u) % nrows_total;
  unsigned long long* out;
  cudaMallocManaged(&out, 1024 * 8);
  const int iters = 64;
  auto report = [&](const char* name, int grid) {
    cudaDeviceSynchronize();
    double mx = 0, sum = 0;
    for (int b = 0; b < grid; ++b) {
      mx = mx > out[b] ? mx : out[b];
      sum += out[b];
    }
    printf("%-28s grid %3d: %.1f B/clk/SM (mean), %.1f (slowest)\n", name, grid, double(kChunk) * iters / (sum / grid),
           double(kChunk) * iters / mx);
  };
  for (int mode = 0; mode < 8; ++mode) {
    for (int rep = 0; rep < 2; ++rep) ldgsts_kernel<<<148, 256>>>(buf, rows, nrows_total, iters, 192, out, mode);
    char nm[64];
    snprintf(nm, sizeof nm, "ldgsts 192 thr mode %d", mode);
    report(nm, 148);
  }
  for (int grid : {1, 148}) {
    for (int th : {64, 128, 256}) {
      for (int rep = 0; rep < 2; ++rep) ldgsts_kernel<<<grid, 256>>>(buf, rows, nrows_total, iters, th, out, 0);
      char nm[64];
      snprintf(nm, sizeof nm, "ldgsts %d thr", th);
      report(nm, grid);
      for (int rep = 0; rep < 2; ++rep) ldg_kernel<<<grid, 256>>>(buf, rows, nrows_total, iters, th, out);
      snprintf(nm, sizeof nm, "ldg.v4 %d thr", th);
      report(nm, grid);
    }
    for (int rep = 0; rep < 2; ++rep) bulk_kernel<<<grid, 256>>>(buf, rows, nrows_total, iters, out);
    report("bulk 128B rows", grid);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
