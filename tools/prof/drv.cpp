// gprof driver: repeated evaluate_batch of one model (host path; device < 0: dry context).
//   ./drv [iters] [model] [hidden] [batch] [device] [precision]
#include "mbx.h"
#include <cstdio>
#include <cstdlib>
#include <vector>
int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 500;
  const char* model = argc > 2 ? argv[2] : "treelstm";
  const int hidden = argc > 3 ? atoi(argv[3]) : 512, batch = argc > 4 ? atoi(argv[4]) : 64;
  const int device = argc > 5 ? atoi(argv[5]) : -1, prec = argc > 6 ? atoi(argv[6]) : 1;
  mbx_ctx* c;
  if (mbx_ctx_create(device, prec, &c)) { printf("ctx err\n"); return 1; }
  mbx_model* m;
  if (mbx_model_create(c, model, hidden, &m)) { printf("err %s\n", mbx_last_error(c)); return 1; }
  mbx_model_make_params(m, 1);
  int64_t nt = 0, nd = 0;
  mbx_model_make_inputs(m, 1, batch, nullptr, &nt, nullptr, &nd);
  std::vector<int32_t> t(nt);
  std::vector<float> d(nd);
  mbx_model_make_inputs(m, 1, batch, t.data(), &nt, d.data(), &nd);
  mbx_options o;
  mbx_options_default(&o);
  for (int i = 0; i < iters; ++i) {
    mbx_result* r;
    if (mbx_evaluate_batch(m, batch, t.data(), nt, d.data(), nd, &o, &r)) { printf("err %s\n", mbx_last_error(c)); return 1; }
    mbx_result_destroy(r);
  }
  printf("done\n");
}
