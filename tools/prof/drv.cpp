// gprof driver: TreeLSTM-512 b64 evaluations in a dry context (host path only).
#include "mbx.h"
#include <vector>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  int iters = argc > 1 ? atoi(argv[1]) : 500;
  mbx_ctx* c; mbx_ctx_create(-1, 1, &c);
  mbx_model* m; if (mbx_model_create(c, "treelstm", 512, &m)) { printf("err %s\n", mbx_last_error(c)); return 1; }
  mbx_model_make_params(m, 1);
  int64_t nt=0, nd=0; mbx_model_make_inputs(m, 1, 64, nullptr, &nt, nullptr, &nd);
  std::vector<int32_t> t(nt); std::vector<float> d(nd);
  mbx_model_make_inputs(m, 1, 64, t.data(), &nt, d.data(), &nd);
  mbx_options o; mbx_options_default(&o);
  for (int i = 0; i < iters; ++i) {
    mbx_result* r; if (mbx_evaluate_batch(m, 64, t.data(), nt, d.data(), nd, &o, &r)) { printf("err %s\n", mbx_last_error(c)); return 1; }
    mbx_result_destroy(r);
  }
  printf("done\n");
}
