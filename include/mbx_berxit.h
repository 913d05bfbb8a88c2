/* mbx_berxit.h — C ABI of the Berxit early-exit encoder on B200 (BASELINE configs[4]).
 *
 * The reference has no Berxit model (proj/src/zoo.cpp:305-317) and no softmax / layernorm / GELU
 * op (proj/include/mbatch/backend.hpp:27-37); the model is the one the paper evaluates
 * (BERT-base hyper-parameters, all layers share one weight set, sequence
 * length 128, learned early exit).  This ABI is therefore modelled on the reference's whole-model
 * entry (runtime::evaluate_batch, proj/src/executor.cpp:782-787: params resident, a mini-batch
 * in, per-instance outputs and the batch schedule out) — parity unpinned (oracle/berxit_oracle.cpp).
 *
 * ACRoBat's batching for this model: after every layer each instance's learning-to-exit head
 * decides whether it stops; the next layer runs one batch over the instances still running, in
 * instance order.  Here the decision, the compaction of the running set and the next layer's
 * instance list stay on the device: a mini-batch is one enqueue of L layers (captured once as a
 * CUDA graph per batch size), every kernel reads the running-instance index array and count from
 * device memory, and nothing returns to the host until the results do.
 *
 * Model (per instance x[S][H]; one layer, repeated until exit; post-LN BERT):
 *   qkv = x Wqkv^T + bqkv;  ctx = per head softmax(q k^T / sqrt(H/heads)) v
 *   x1 = LN1(x + ctx Wo^T + bo);  x2 = LN2(x1 + GELU(x1 W1^T + b1) W2^T + b2)   (GELU: erf form)
 *   u = sigmoid(w_lte . x2[0] + b_lte); exit if u >= exit_threshold or last layer:
 *   logits = Wc x2[0] + bc, exit_layer = l.
 * Flat parameter order (mbx_berxit_param_count floats):
 *   Wqkv[3H][H] bqkv[3H] Wo[H][H] bo[H] ln1_g[H] ln1_b[H] W1[F][H] b1[F] W2[H][F] b2[H]
 *   ln2_g[H] ln2_b[H] w_lte[H] b_lte[1] Wc[C][H] bc[C]
 * Synthetic parameters / inputs (mbx_berxit_make_params / _make_input): mt19937(seed*7919+17) in
 * flat order, and mt19937(seed*104729+31*i+7) per instance (the zoo's seeding,
 * proj/src/zoo.cpp:332-341, :343-401); a draw is lo + (hi-lo)*((g()>>8)*2^-24).
 *
 * Device constraints: seq == 128 (one instance = one 128-row MMA tile), H / heads == 64,
 * H and F multiples of 256.
 * Arithmetic: MBX_PREC_BF16X3 (default; split-bf16 tcgen05 GEMMs, hi*hi + hi*lo + lo*hi, fp32
 * TMEM accumulation; softmax / LN / GELU / exit head in fp32) or MBX_PREC_BF16 (one bf16 pass).
 * All functions return 0 on success; mbx_berxit_last_error gives the message otherwise. */
#ifndef MBX_BERXIT_H
#define MBX_BERXIT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t hidden;       /* H, 768 for BERT-base */
  int32_t heads;        /* 12 */
  int32_t ffn;          /* F, 3072 */
  int32_t layers;       /* L, 12 */
  int32_t seq;          /* S, 128 */
  int32_t classes;      /* C, 8 */
  float exit_threshold; /* tau, 0.6 */
  float ln_eps;         /* 1e-12 */
} mbx_berxit_config;

typedef struct mbx_berxit mbx_berxit;

void mbx_berxit_config_default(mbx_berxit_config* c);
int64_t mbx_berxit_param_count(const mbx_berxit_config* c);
/* Host-side generators (the input spec shared with the oracle). */
int mbx_berxit_make_params(const mbx_berxit_config* c, unsigned seed, float* out);
int mbx_berxit_make_input(const mbx_berxit_config* c, unsigned seed, int instance, float* out /* [S][H] */);

/* Device state for mini-batches of up to max_batch instances on `device`. */
int mbx_berxit_create(int device, int precision, const mbx_berxit_config* c, int max_batch, mbx_berxit** out);
void mbx_berxit_destroy(mbx_berxit* m);
const char* mbx_berxit_last_error(const mbx_berxit* m);
/* Uploads the flat parameters (host) and builds the split-bf16 weight images once. */
int mbx_berxit_set_params(mbx_berxit* m, const float* params, int64_t n);
/* One mini-batch, end to end: x (host, [batch][S][H] floats) -> device, L layers with on-device
 * exits, results -> host.  logits [batch][C]; exit_layer [batch]; schedule (optional, may be NULL)
 * [L][batch] int32: row l lists the instances of layer l's batch in batch order, -1 padded.
 * Synchronous. */
int mbx_berxit_run(mbx_berxit* m, int batch, const float* x, float* logits, int32_t* exit_layer, int32_t* schedule);
/* Device-resident variant (benchmarking): x_dev is a device pointer ([batch][S][H] floats);
 * results stay on the device until mbx_berxit_read.  Asynchronous on mbx_berxit_stream. */
int mbx_berxit_run_device(mbx_berxit* m, int batch, const float* x_dev);
int mbx_berxit_read(mbx_berxit* m, int batch, float* logits, int32_t* exit_layer, int32_t* schedule);
void* mbx_berxit_stream(mbx_berxit* m);
/* Kernel launches one mini-batch enqueues (graph nodes). */
int mbx_berxit_launches_per_batch(const mbx_berxit* m, int batch);

#ifdef __cplusplus
}
#endif
#endif
