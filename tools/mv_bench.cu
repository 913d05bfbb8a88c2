// Standalone timing of the MV-RNN cell kernel on synthetic nodes (phase stamps of CTA 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -DMBX_MV_STAMPS -I../paper_2305_10611_b200/csrc
//        mv_bench.cu -o mv_bench
#include "../paper_2305_10611_b200/csrc/kernels_mv.cu"
#include <cstdio>
#include <vector>
using namespace mbx;
int main(int argc, char** argv) {
  const int H = 128, K = H, N = H, U = H;
  std::vector<int> bs = {2, 13, 61, 126, 209};
  const int64_t per = 2 * H + 2 * H * H;  // lv, rv, Rm, Lm
  const int bmax = 209;
  size_t total = 2 * H * H + H + size_t(bmax) * per + size_t(bmax) * (H + H * H) + 64;
  float* arena;
  cudaMalloc(&arena, total * 4);
  cudaMemset(arena, 0, total * 4);
  std::vector<int64_t> sh = {0, 2 * H * H};
  std::vector<int64_t> bo(size_t(bmax) * 4);
  int64_t cur = 2 * H * H + H;
  for (int i = 0; i < bmax; ++i) {
    bo[i * 4 + 0] = cur; bo[i * 4 + 1] = cur + 2 * H; bo[i * 4 + 2] = cur + H; bo[i * 4 + 3] = cur + 2 * H + H * H;
    cur += per;
  }
  int64_t outs[2] = {cur, cur + int64_t(bmax) * H};
  int64_t *dsh, *dbo, *dout;
  cudaMalloc(&dsh, 16); cudaMalloc(&dbo, bo.size() * 8); cudaMalloc(&dout, 16);
  cudaMemcpy(dsh, sh.data(), 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dbo, bo.data(), bo.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, outs, 16, cudaMemcpyHostToDevice);
  float* wt; cudaMalloc(&wt, mv_wt_floats(N, U) * 4); launch_mv_transpose(arena, wt, N, U, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int pdl = 0; pdl < 2; ++pdl)
  for (int nb : bs) {
    MvCellLaunch L{};
    L.arena = arena; L.shared_off = dsh; L.batched_off = dbo; L.b = nb; L.nb = 4;
    L.x[0] = 0; L.m[0] = 1; L.x[1] = 2; L.m[1] = 3; L.first = 0; L.w = 0; L.K = K; L.N = N; L.U = U;
    L.nlinks = 2; L.link_op[0] = kAdd; L.link_rhs[0] = 1; L.link_op[1] = kTanh; L.link_rhs[1] = -1;
    L.cell_out = dout; L.add_out = dout + 1; L.pdl = pdl; L.wt = wt;
    for (int w = 0; w < 3; ++w) launch_mv_cell(L, 0);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch_mv_cell(L, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long st[16];
    cudaMemcpyFromSymbol(st, g_mv_stamps, sizeof st);
    unsigned long long ck[2];
    cudaMemcpyFromSymbol(ck, g_mv_clk, sizeof ck);
    printf("[%.0f MHz] ", double(ck[1] - ck[0]) * 1000.0 / double(st[6] - st[0]));
    printf("pdl=%d b=%3d  %.2f us/launch  stamps(ns):", pdl, nb, ms * 1000 / 20);
    for (int i : {1, 2, 4, 7, 3, 5, 6}) printf(" %lld", (long long)(st[i] - st[0]));
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
}
