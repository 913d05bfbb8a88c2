/* oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of the CPU restatement of the reference hot path (oracle/oracle.cpp).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product (paper_2305_10611_b200/) never links or calls it.
 *
 * Values cross the ABI in the "hostval" encoding shared with the product's C ABI (include/mbx.h):
 * an int32 token stream plus a float32 data stream, depth-first:
 *   tensor: 0, rows, cols            (rows*cols floats consumed from the data stream)
 *   int:    1, value
 *   list:   2, n, items...
 *   tuple:  3, n, items...
 *   adt:    4, ctor (0 = Leaf, 1 = Node), n, fields...
 */
#ifndef MBATCH_ORACLE_H
#define MBATCH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_model orc_model;

/* Builds zoo model `name` at hidden size `hidden` with params from make_params(seed)
 * (proj/src/zoo.cpp:332-341).  Returns NULL on an unknown model. */
orc_model* orc_model_create(const char* name, int hidden, unsigned seed);
void orc_model_destroy(orc_model* m);

/* Generates make_inputs(seed, batch) (proj/src/zoo.cpp:343-401) into the model's input set. */
int orc_make_inputs(orc_model* m, unsigned seed, int batch);
/* Replaces the input set with `batch` encoded instances. */
int orc_set_inputs(orc_model* m, int batch, const int32_t* toks, int64_t ntok, const float* data,
                   int64_t ndata);
/* Size of / copy out the encoded input set (for feeding the same inputs to the B200 path). */
int64_t orc_inputs_ntok(const orc_model* m);
int64_t orc_inputs_ndata(const orc_model* m);
int orc_get_inputs(const orc_model* m, int32_t* toks, float* data);

/* FNV-1a digests in the layout of oracle/ref_harness.cpp (`digest`). */
uint64_t orc_params_digest(const orc_model* m);
uint64_t orc_inputs_digest(const orc_model* m);

/* Unbatched sequential evaluation of every instance (runtime::reference_evaluate,
 * proj/src/reference.cpp:338-345).  Outputs are encoded; sizes first, then copy. */
int orc_evaluate(orc_model* m);
int64_t orc_outputs_ntok(const orc_model* m);
int64_t orc_outputs_ndata(const orc_model* m);
int orc_get_outputs(const orc_model* m, int32_t* toks, float* data);
uint64_t orc_outputs_digest(const orc_model* m);
/* Number of tensor primitive ops the last orc_evaluate executed (work accounting). */
int64_t orc_last_prim_ops(const orc_model* m);

/* Parameter tensors in module order: count, then name / shape / data of parameter i. */
int orc_num_params(const orc_model* m);
const char* orc_param_name(const orc_model* m, int i);
int orc_param_shape(const orc_model* m, int i, int* rows, int* cols);
const float* orc_param_data(const orc_model* m, int i);

/* Primitive op restatement (proj/src/backend.cpp:105-181): op codes follow backend::OpCode
 * (0 dense, 1 add, 2 mul, 3 sigmoid, 4 tanh, 5 relu, 6 concat, 7 argmax, 8 fill). */
int orc_exec_primop(int op, int nin, const float* const* ins, const int* in_rows,
                    const int* in_cols, float* out, int out_rows, int out_cols, float fill);

/* schedule_depth restatement (proj/src/schedule.cpp:29-62) over a flat node table:
 * per node: id, phase, depth, sig, ghost, and its shared refs (node, out, offset) triples.
 * Writes batches as (phase, depth, sig, ghost, size) rows into `batches` (5 ints each) and the
 * node ids in batch order into `order`.  Returns the number of batches; *ops gets the
 * scheduler work counter. */
int orc_schedule_depth(int n, const int* id, const int* phase, const int* depth, const int* sig,
                       const int* ghost, const int* nshared, const int64_t* shared_refs,
                       int* batches, int* order, long* ops);

/* FNV-1a digest of `count` encoded values (same layout as the digests above). */
uint64_t orc_digest_encoded(const int32_t* toks, int64_t ntok, const float* data, int64_t ndata, int count);

/* Scalar restatements of the libm calls on the path, for unit tests: 0 expf, 1 tanhf,
 * 2 sigmoid 1/(1+expf(-x)). */
float orc_unary(int which, float x);

#ifdef __cplusplus
}
#endif
#endif
