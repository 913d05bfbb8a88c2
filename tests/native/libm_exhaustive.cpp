// Exhaustive check of the device libm restatements (paper_2305_10611_b200/csrc/libm_fp32.cuh)
// against the host libm the reference links (glibc expf / tanhf), over every float bit pattern
// in [lo, hi).  Built with -ffp-contract=off by tests/test_libm_exact.py.  Prints mismatch counts.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include "../../paper_2305_10611_b200/csrc/libm_fp32.cuh"

int main(int argc, char** argv) {
  uint64_t lo = argc > 1 ? strtoull(argv[1], 0, 0) : 0, hi = argc > 2 ? strtoull(argv[2], 0, 0) : (1ull << 32);
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 4;
  std::vector<uint64_t> bad_exp(nt), bad_tanh(nt), first(nt, ~0ull);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t]() {
      for (uint64_t u = lo + t; u < hi; u += nt) {
        float x = mbx_libm::u2f((uint32_t)u);
        float a = std::exp(x), b = mbx_libm::expf_exact(x);
        float c = std::tanh(x), d = mbx_libm::tanhf_exact(x);
        bool e1 = mbx_libm::f2u(a) != mbx_libm::f2u(b) && !(std::isnan(a) && std::isnan(b));
        bool e2 = mbx_libm::f2u(c) != mbx_libm::f2u(d) && !(std::isnan(c) && std::isnan(d));
        if (e1) ++bad_exp[t];
        if (e2) ++bad_tanh[t];
        if ((e1 || e2) && first[t] == ~0ull) first[t] = u;
      }
    });
  for (auto& x : th) x.join();
  uint64_t be = 0, bt = 0, f = ~0ull;
  for (unsigned t = 0; t < nt; ++t) { be += bad_exp[t]; bt += bad_tanh[t]; if (first[t] < f) f = first[t]; }
  printf("{\"range\": [%llu, %llu], \"expf_mismatch\": %llu, \"tanhf_mismatch\": %llu, \"first_bad\": %lld}\n",
         (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)be, (unsigned long long)bt,
         f == ~0ull ? -1LL : (long long)f);
  return 0;
}
