// Cycles per step of a sequential fp32 dot-product chain read from shared memory (probe).
#include "../paper_2305_10611_b200/csrc/kernels_mv.cu"
#include <cstdio>
using namespace mbx;
__global__ void probe(float* out, long long* cyc, int variant) {
  __shared__ __align__(16) float x[256];
  __shared__ __align__(16) float m[256 * 33];
  for (int i = threadIdx.x; i < 256 * 33; i += blockDim.x) m[i] = 1.0f + i * 1e-6f;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) x[i] = 0.5f + i * 1e-5f;
  __syncthreads();
  long long t0 = clock64();
  float acc = 0;
  if (variant == 0) acc = chain_dot(x, m + threadIdx.x, 32, 256);
  else if (variant == 1) {
#pragma unroll 8
    for (int r = 0; r < 256; ++r) acc = fadd(acc, fmul(x[r], m[r * 32 + threadIdx.x]));
  } else if (variant == 2) {  // products precomputed in registers, then the add chain
    float p[256 / 8];
    for (int r0 = 0; r0 < 256; r0 += 32) {
#pragma unroll
      for (int k = 0; k < 32; ++k) p[k % 32] = fmul(x[r0 + k], m[(r0 + k) * 32 + threadIdx.x]);
#pragma unroll
      for (int k = 0; k < 32; ++k) acc = fadd(acc, p[k]);
    }
  } else if (variant == 4) {  // products in smem, stride-32 scalar loads
#pragma unroll 16
    for (int r = 0; r < 256; ++r) acc = fadd(acc, m[r * 32 + threadIdx.x]);
  } else if (variant == 5) {  // products in smem, contiguous float4 loads
    const float4* mt = reinterpret_cast<const float4*>(m + threadIdx.x * 260);
#pragma unroll 8
    for (int r = 0; r < 64; ++r) {
      const float4 b = mt[r];
      acc = fadd(acc, b.x); acc = fadd(acc, b.y); acc = fadd(acc, b.z); acc = fadd(acc, b.w);
    }
  } else if (variant == 6) {  // products in smem, contiguous float4, all loaded up front in 2 halves
    const float4* mt = reinterpret_cast<const float4*>(m + threadIdx.x * 260);
    for (int h = 0; h < 2; ++h) {
      float4 b[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) b[r] = mt[h * 32 + r];
#pragma unroll
      for (int r = 0; r < 32; ++r) { acc = fadd(acc, b[r].x); acc = fadd(acc, b[r].y); acc = fadd(acc, b[r].z); acc = fadd(acc, b[r].w); }
    }
  } else {  // transposed, float4
    const float4* mt = reinterpret_cast<const float4*>(m + threadIdx.x * 260);
    const float4* xv = reinterpret_cast<const float4*>(x);
#pragma unroll 4
    for (int r = 0; r < 64; ++r) {
      const float4 a = xv[r], b = mt[r];
      acc = fadd(acc, fmul(a.x, b.x)); acc = fadd(acc, fmul(a.y, b.y));
      acc = fadd(acc, fmul(a.z, b.z)); acc = fadd(acc, fmul(a.w, b.w));
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[variant] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 7; ++v) probe<<<1, 32>>>(o, c, v);
  long long h[7]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
  for (int v = 0; v < 7; ++v) printf("variant %d: %lld cycles / 256 steps = %.1f\n", v, h[v], h[v] / 256.0);
}
