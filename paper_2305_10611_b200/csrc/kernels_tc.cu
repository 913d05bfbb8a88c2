// kernels_tc.cu — host side of the generated per-plan kernels (device source: tc_gate.cuh).
//
// tc_prepare inspects each registered plan: if it has the shape
//     [concat(p0, p1)] -> dense / FusedDense(row, W_1..W_G shared) -> column-local tail
// (TreeLSTM internal cell add_mul_sigmoid_bias: concat(lh, rh) . [W_i|W_fl|W_fr|W_u], gates, c,
// tanh(c); bias_dense; the RNN cells ...) it generates the tensor-core kernel for it, and if it is
// purely elementwise (the hoisted TreeLSTM leaf cell, MV-RNN's matrix add) the pointwise kernel.
// The plan's tail is emitted as straight-line code over registers (no interpretation on the
// device) and compiled once with NVRTC (jit.cpp).  tc_launch picks the tiling of each launch
// from the batch size and packs the split-bf16 weights on first use.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <tuple>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "jit.h"
#include "tc.h"
#include "tc_abi.h"

namespace mbx {

extern std::atomic<int64_t> g_launches;

namespace {

constexpr int kTcThreads = 256;
constexpr int kM = 128;
constexpr int kRawStages = 3;  // MBX_RAW in tc_gate.cuh
constexpr int kMaxTail = 24;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kLevelsStaticSmem = 64 * int(sizeof(TcLevel)) + 64;  // mbx_tc_levels: its copy of the level table

// ---- tail IR: a plan's steps after the contraction as ops over per-element values --------------
enum : int8_t { kSrcNone = 0, kSrcSlot = 1, kSrcAcc = 2, kSrcBatched = 3, kSrcShared = 4, kSrcLoad = 5 };
constexpr int kOpCopy = 99;
struct EpiSrc {
  int8_t type = kSrcNone;
  int16_t idx = 0;  // slot / accumulator gate g / batched or shared input index / load index
  int32_t off = 0;  // column-slice offset into the input row
};
struct EpiOp {
  int op, dst;
  EpiSrc a, b;
};
struct EpiProg {
  int nslots = 0, nout = 0, nloads = 0;
  int out_slot[kMaxOut] = {};
  EpiSrc loads[MBX_MAX_LOADS];
  std::vector<EpiOp> ops;
};

// Split-bf16 parts of a weight / operand for a pass count: bf16 (1 MMA), bf16x3 (hi, lo; 3 MMAs),
// bf16x6 (hi, mid, lo; 6 MMAs: every product term down to 2^-24 relative).
__host__ __device__ inline int npass_parts(int npass) { return npass == 1 ? 1 : (npass == 3 ? 2 : 3); }
inline int npass_of(int precision) {
  return precision == MBX_PREC_BF16 ? 1 : (precision == MBX_PREC_BF16X6 ? 6 : 3);
}

// Packs G weights (each K x U fp32, row-major, in the arena) into per-unit-tile, per-chunk
// canonical K-major bf16 blocks: [tile][chunk][pass][M x KC].  Rows g*UC + j of tile t hold column
// t*UC + j of weight g; rows >= G*UC are zero.
__global__ void tc_pack_kernel(const float* arena, const int64_t* w_off, int G, int K, int U, int UC, int M, int KC,
                               int npass, uint8_t* out) {
  const int nchunks = K / KC;
  const int ntiles = U / UC;
  const int64_t total = int64_t(ntiles) * nchunks * M * KC;
  const int64_t chunk_bytes = int64_t(M) * KC * 2;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int kk = int(idx % KC);
    int64_t r1 = idx / KC;
    const int r = int(r1 % M);
    r1 /= M;
    const int c = int(r1 % nchunks);
    const int t = int(r1 / nchunks);
    float v = 0.0f;
    if (r < G * UC) {
      const int g = r / UC, col = t * UC + r % UC, k = c * KC + kk;
      v = arena[w_off[g] + int64_t(k) * U + col];
    }
    const int parts = npass_parts(npass);
    uint8_t* blk = out + ((int64_t(t) * nchunks + c) * parts) * chunk_bytes;
    const uint32_t off = uint32_t((r >> 3) * (KC * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
    for (int q = 0; q < parts; ++q) {  // successive residuals: hi, [mid,] lo
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(blk + q * chunk_bytes + off) = h;
      v = v - __bfloat162float(h);
    }
  }
}

struct TcState {
  int K = 0, KC = 0, nchunks = 0, U = 0, G = 0, UC = 0, dstep = 0;
  int npieces = 0;
  int piece_kind[2] = {0, 0}, piece_idx[2] = {0, 0}, piece_off[2] = {0, 0}, piece_k[2] = {0, 0};
  std::vector<int> w_shared;  // shared-input index of each weight
  EpiProg prog;
  std::string src;            // generated kernel source
  void* fn = nullptr;         // cudaKernel_t
  void* fn_fast = nullptr;    // pointwise plans: fast-activation variant (tensor-core precisions)
  void* fn4 = nullptr, *fn_fast4 = nullptr;  // pointwise plans, E % 4 == 0: 16-byte variants
  // Few output columns (U x G <= 64): the bit-exact CUDA-core small-dense kernel instead of the
  // tensor cores, in every precision (sfn != nullptr).
  void* sfn = nullptr;
  int s_npc = 0, s_uc = 0, s_kb = 0, s_st = 1, s_smem = 0;
  bool s_attr = false;
  // Narrow variant (8-unit slices of 8 nodes, compiled on first use) for batches too small to
  // give the wide one's grid a wave.  (4- and 2-unit slices were measured: the same kernel times,
  // but the flush slower in situ, 81-85 -> 96-106 us for TreeLSTM-256 b8.)
  struct SmallVar {
    void* fn = nullptr;
    int kb = 0, st = 1, smem = 0, threads = 0;
    bool attr = false;
  };
  SmallVar nv;
  bool narrow_ok = false;
  bool attr_set = false;
  // Persistent multi-level variant (mbx_tc_levels): K-split ranks, maximal node tile, smem layout.
  // mbx_tc_levels configurations: [0] deep — the largest K split, weight slice resident, for runs
  // of levels; [1] wide — a small K split, many node-tile groups, for one large batch.
  struct LevelsCfg {
    int S = 0, NT = 0, xch = 0;  // xch 0: K ranks form a cluster (DSMEM), 1: L2 exchange
    int parts = 2;               // split-bf16 parts the shared-memory layout holds (3: bf16x6)
    int w_off = 0, x_off = 0, recv_off = 0, bar_off = 0, smem = 0;
    std::string src;
    void* fn = nullptr;
    bool attr_set = false;
    // Per issue slot (mbx_ctx::issue_slot: the context's two streams, so two runs of one plan
    // can run at once):
    float* part[2] = {nullptr, nullptr};      // xch 1: partials buffer
    unsigned* flags[2] = {nullptr, nullptr};  // xch 1: arrival counters
    unsigned* ready[2] = {nullptr, nullptr};  // per unit tile readiness counters (monotonic)
    unsigned ready_count[2] = {0, 0};         // their value after every launch so far (stream order)
  } lv[3];
  // lv[2]: a deep configuration whose grid leaves room for a second one (two independent runs of
  // a flush at once, mbx_ctx::prefer_pair), built on first use; pair_tried: attempted.
  bool pair_tried = false;
  // packed-weight cache: (weight offsets, precision, upload epoch) -> device buffer
  struct Packed {
    std::vector<int64_t> offs;
    int npass = 0;
    uint64_t epoch = 0;
    uint8_t* buf = nullptr;
  };
  std::vector<Packed> packs;
};

// Compiles the plan's steps after the contraction into ops over per-element values.  A step s
// gets slot s - dstep - 1; the contraction's own columns are read from the accumulator (gate g).
bool compile_epilogue(const mbatch::backend::ExecutablePlan& p, TcState& st) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  EpiProg& pr = st.prog;
  pr = EpiProg{};
  const int dstep = st.dstep;
  bool ok = true;
  auto src = [&](const PlanRef& r) {
    EpiSrc s{};
    const int slice = r.cols >= 0 ? r.col_off : 0;
    if (r.kind == PlanRef::Kind::kTemp) {
      if (r.index == dstep) {
        s.type = kSrcAcc;
        s.idx = int16_t(slice / st.U);
      } else {
        s.type = kSrcSlot;
        s.idx = int16_t(r.index - dstep - 1);
      }
      return s;
    }
    // Input rows are read once per element: dedupe them into the load table.
    EpiSrc l{};
    l.type = r.kind == PlanRef::Kind::kBatched ? kSrcBatched : kSrcShared;
    l.idx = int16_t(r.index);
    l.off = slice;
    int j = 0;
    while (j < pr.nloads && !(pr.loads[j].type == l.type && pr.loads[j].idx == l.idx && pr.loads[j].off == l.off)) ++j;
    if (j == pr.nloads) {
      if (pr.nloads >= MBX_MAX_LOADS) {
        ok = false;
        return s;
      }
      pr.loads[pr.nloads++] = l;
    }
    s.type = kSrcLoad;
    s.idx = int16_t(j);
    return s;
  };
  const int nsteps = int(p.steps.size());
  pr.nslots = nsteps - dstep - 1;
  for (int s = dstep + 1; s < nsteps; ++s) {
    const PlanStep& ps = p.steps[s];
    const int dst = s - dstep - 1;
    if (ps.kind == PlanStep::Kind::kChain) {
      if (ps.chain.empty()) {
        pr.ops.push_back(EpiOp{kOpCopy, dst, src(ps.ins[0]), EpiSrc{}});
        continue;
      }
      for (size_t l = 0; l < ps.chain.size(); ++l) {
        EpiSrc a = l == 0 ? src(ps.ins[0]) : EpiSrc{kSrcSlot, int16_t(dst), 0};
        EpiSrc b = ps.chain[l].rhs ? src(*ps.chain[l].rhs) : EpiSrc{};
        pr.ops.push_back(EpiOp{int(ps.chain[l].op), dst, a, b});
      }
    } else {
      pr.ops.push_back(EpiOp{int(ps.op), dst, src(ps.ins[0]), ps.ins.size() > 1 ? src(ps.ins[1]) : EpiSrc{}});
    }
  }
  pr.nout = int(p.outputs.size());
  for (size_t k = 0; k < p.outputs.size(); ++k) {
    const PlanRef& o = p.outputs[k];
    if (o.kind != PlanRef::Kind::kTemp) return false;
    if (o.index == dstep) {  // the contraction itself is an output: copy it into a fresh slot
      const int dst = pr.nslots++;
      pr.ops.push_back(EpiOp{kOpCopy, dst, src(o), EpiSrc{}});
      pr.out_slot[k] = dst;
    } else {
      pr.out_slot[k] = o.index - dstep - 1;
    }
  }
  for (const EpiOp& o : pr.ops) {
    if (o.a.type == kSrcNone) return false;
    const bool binary = o.op == kAdd || o.op == kMul;
    if (binary && o.b.type == kSrcNone) return false;
    if (!(binary || o.op == kSigmoid || o.op == kTanh || o.op == kRelu || o.op == kOpCopy)) return false;
  }
  return ok && pr.nslots <= 64;
}

// The tail as a device function over registers: g = accumulator gates, l = loaded input rows.
// Gate tails (tolerance path) use the fast activations; pointwise tails the glibc-exact ones.
// fast_pw: the pointwise tail with the fast activations (tensor-core precisions only).
// exact_gate: a gate tail with the glibc-exact activations (mbx_tail_exact, the bit-exact
// small-dense kernel).
std::string gen_tail(const EpiProg& pr, bool pointwise, bool fast_pw = false, bool exact_gate = false) {
  std::ostringstream o;
  o << (pointwise ? (fast_pw ? "__device__ __forceinline__ void mbx_pw_tail_fast(const float* l, float* o) {\n"
                             : "__device__ __forceinline__ void mbx_pw_tail(const float* l, float* o) {\n")
                  : (exact_gate ? "__device__ __forceinline__ void mbx_tail_exact(const float* g, const float* l, float* o) {\n"
                                : "__device__ __forceinline__ void mbx_tail(const float* g, const float* l, float* o) {\n"));
  const bool exact = (pointwise && !fast_pw) || exact_gate;
  for (int s = 0; s < pr.nslots; ++s) o << "  float s" << s << " = 0.0f;\n";
  auto ref = [](const EpiSrc& s) -> std::string {
    switch (s.type) {
      case kSrcSlot: return "s" + std::to_string(s.idx);
      case kSrcAcc: return "g[" + std::to_string(s.idx) + "]";
      case kSrcLoad: return "l[" + std::to_string(s.idx) + "]";
      default: return "0.0f";
    }
  };
  for (const EpiOp& op : pr.ops) {
    o << "  s" << op.dst << " = ";
    const std::string a = ref(op.a), b = ref(op.b);
    switch (op.op) {
      case kAdd: o << "mbx_libm::fadd(" << a << ", " << b << ")"; break;
      case kMul: o << "mbx_libm::fmul(" << a << ", " << b << ")"; break;
      case kSigmoid: o << (exact ? "mbx_libm::sigmoidf_exact(" : "mbx_fsig(") << a << ")"; break;
      case kTanh: o << (exact ? "mbx_libm::tanhf_exact(" : "mbx_ftanh(") << a << ")"; break;
      case kRelu: o << "mbx_libm::reluf_exact(" << a << ")"; break;
      default: o << a; break;
    }
    o << ";\n";
  }
  for (int k = 0; k < pr.nout; ++k) o << "  o[" << k << "] = s" << pr.out_slot[k] << ";\n";
  o << "}\n";
  return o.str();
}

bool stamps_enabled() {
  static const bool on = std::getenv("MBX_TC_STAMPS") != nullptr;
  return on;
}

std::string gen_gate_source(const TcState& st) {
  std::ostringstream o;
  o << jit::prelude_source();
  o << "#define MBX_GATE_KERNEL 1\n"
    << "#define MBX_KC " << st.KC << "\n#define MBX_U " << st.U << "\n#define MBX_G " << st.G << "\n#define MBX_UC "
    << st.UC << "\n#define MBX_NCHUNKS " << st.nchunks << "\n#define MBX_NPIECES " << st.npieces
    << "\n#define MBX_PK0 " << st.piece_k[0] << "\n#define MBX_NLOADS " << st.prog.nloads << "\n#define MBX_NOUT "
    << st.prog.nout << "\n#define MBX_RAW " << kRawStages << "\n";
  o << gen_tail(st.prog, false);
  o << jit::kernel_source();
  return o.str();
}

// Source of one mbx_tc_levels configuration (same plan shape and tail as the gate kernel).
std::string gen_levels_source(const TcState& st, int k) {
  const TcState::LevelsCfg& L = st.lv[k];
  std::ostringstream o;
  if (stamps_enabled()) o << "#define MBX_STAMPS 1\n";
  o << jit::prelude_source();
  o << "#define MBX_LEVELS_KERNEL 1\n"
    << "#define MBX_KC " << st.KC << "\n#define MBX_U " << st.U << "\n#define MBX_G " << st.G << "\n#define MBX_UC "
    << st.UC << "\n#define MBX_NCHUNKS " << st.nchunks << "\n#define MBX_NPIECES " << st.npieces
    << "\n#define MBX_PK0 " << st.piece_k[0] << "\n#define MBX_NLOADS " << st.prog.nloads << "\n#define MBX_NOUT "
    << st.prog.nout << "\n#define MBX_LS " << L.S << "\n#define MBX_LNT " << L.NT << "\n#define MBX_LXCH " << L.xch
    << "\n#define MBX_LPARTS " << L.parts << "\n";
  if (L.parts == 3) {
    // bf16x6 (24-bit operands): the glibc-exact activations too, so the only difference from the
    // FP32 path left is the tensor core's summation order.
    o << gen_tail(st.prog, false, false, true) << "#define mbx_tail mbx_tail_exact\n";
  } else {
    o << gen_tail(st.prog, false);
  }
  o << jit::kernel_source();
  return o.str();
}

// Source of the bit-exact small-dense kernel (plans with few output columns, e.g. a classifier).
// Threads of a small-dense block: one per (gate, node, unit) when that fits 256 (the gates split
// over threads), else one per (node, unit); whole warps, at least 64.
int small_threads(const TcState& st, int npc, int uc) {
  const int t = npc * uc * st.G <= kTcThreads ? npc * uc * st.G : npc * uc;
  return std::clamp((t + 31) / 32 * 32, 64, kTcThreads);
}

std::string gen_small_source(const TcState& st, int npc, int uc, int kb, int stages) {
  std::ostringstream o;
  o << jit::prelude_source();
  o << "#define MBX_SMALL_KERNEL 1\n"
    << "#define MBX_KC 16\n#define MBX_K " << st.K << "\n#define MBX_U " << st.U << "\n#define MBX_G " << st.G
    << "\n#define MBX_NPIECES " << st.npieces << "\n#define MBX_PK0 " << st.piece_k[0] << "\n#define MBX_NLOADS "
    << st.prog.nloads << "\n#define MBX_NOUT " << st.prog.nout << "\n#define MBX_SNPC " << npc
    << "\n#define MBX_SUC " << uc << "\n#define MBX_SKB " << kb << "\n#define MBX_SST " << stages
    << "\n#define MBX_SGS " << (npc * uc * st.G <= kTcThreads ? st.G : 1) << "\n#define MBX_STHREADS "
    << small_threads(st, npc, uc) << "\n";
  o << gen_tail(st.prog, false, false, true);
  o << jit::kernel_source();
  return o.str();
}

std::string gen_pointwise_source(const TcState& st) {
  std::ostringstream o;
  o << jit::prelude_source();
  o << "#define MBX_POINTWISE_KERNEL 1\n#define MBX_KC 16\n#define MBX_PW_E " << st.U << "\n#define MBX_NLOADS "
    << st.prog.nloads << "\n#define MBX_NOUT " << st.prog.nout << "\n";
  o << gen_tail(st.prog, true);
  o << gen_tail(st.prog, true, true);
  o << jit::kernel_source();
  return o.str();
}

bool analyse(const mbatch::backend::ExecutablePlan& p, const DPlan& d, TcState& st) {
  using mbatch::backend::OpCode;
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  if (p.ghost || d.unit <= 0 || p.steps.empty()) return false;
  int dstep = -1;
  for (size_t s = 0; s < p.steps.size(); ++s) {
    const PlanStep& ps = p.steps[s];
    const bool dense = ps.kind == PlanStep::Kind::kFusedDense || (ps.kind == PlanStep::Kind::kOp && ps.op == OpCode::kDense);
    if (dense) {
      if (dstep >= 0) return false;  // one contraction per plan
      dstep = int(s);
    }
  }
  if (dstep < 0 || dstep > 1) return false;
  const PlanStep& D = p.steps[dstep];
  if (!d.steps[dstep].split || D.out_shape.rows != 1) return false;
  // A row: either a direct S/B ref or step 0 = concat of two S/B refs.
  const PlanRef& a = D.ins[0];
  auto width = [&](const PlanRef& r) {
    if (r.cols >= 0) return r.cols;
    return r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index].cols : p.batched_shapes[r.index].cols;
  };
  auto rows_of = [&](const PlanRef& r) {
    return r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index].rows : p.batched_shapes[r.index].rows;
  };
  std::vector<PlanRef> pieces;
  if (dstep == 1) {
    const PlanStep& c = p.steps[0];
    if (!(c.kind == PlanStep::Kind::kOp && c.op == OpCode::kConcat)) return false;
    if (!(a.kind == PlanRef::Kind::kTemp && a.index == 0 && a.cols < 0)) return false;
    pieces = {c.ins[0], c.ins[1]};
  } else {
    if (a.kind == PlanRef::Kind::kTemp) return false;
    pieces = {a};
  }
  bool any_batched = false;
  int k0 = 0;
  st.npieces = int(pieces.size());
  for (size_t i = 0; i < pieces.size(); ++i) {
    const PlanRef& r = pieces[i];
    if (r.kind == PlanRef::Kind::kTemp || rows_of(r) != 1) return false;
    any_batched = any_batched || r.kind == PlanRef::Kind::kBatched;
    const int w = width(r);
    if (w % 16 != 0) return false;
    st.piece_kind[i] = r.kind == PlanRef::Kind::kShared ? kRefShared : kRefBatched;
    st.piece_idx[i] = r.index;
    st.piece_off[i] = r.cols >= 0 ? r.col_off : 0;
    k0 += w;
    st.piece_k[i] = k0;
  }
  if (!any_batched) return false;  // all-shared contractions are hoisted, not batched
  st.K = k0;
  const int U = d.unit;
  st.U = U;
  st.w_shared.clear();
  for (size_t w = 1; w < D.ins.size(); ++w) {
    if (D.ins[w].kind != PlanRef::Kind::kShared || D.ins[w].cols >= 0) return false;
    const auto& sh = p.shared_shapes[D.ins[w].index];
    if (sh.rows != st.K || sh.cols != U) return false;
    st.w_shared.push_back(D.ins[w].index);
  }
  st.G = int(st.w_shared.size());
  if (st.G < 1 || st.G > 4) return false;
  // Units per tile: the largest multiple of 8 with G x UC <= 128 that tiles U exactly (the TMEM
  // epilogue reads 8 node columns at a time; G = 3 gives 32 units, 96 of the 128 MMA rows).
  st.UC = std::min(U, kM / st.G) / 8 * 8;
  while (st.UC >= 8 && U % st.UC != 0) st.UC -= 8;
  if (st.UC < 8) return false;
  // K chunks never straddle the two concatenated pieces.
  st.KC = (st.K % 32 == 0 && st.piece_k[0] % 32 == 0) ? 32 : 16;
  st.nchunks = st.K / st.KC;
  // Tail: every step after the contraction must be a split elementwise step that never reads
  // steps before the contraction.
  if (int(p.steps.size()) - dstep - 1 > kMaxTail) return false;
  for (size_t s = dstep + 1; s < p.steps.size(); ++s) {
    if (!d.steps[s].split) return false;
    const PlanStep& ps = p.steps[s];
    std::vector<PlanRef> refs = ps.ins;
    for (auto& l : ps.chain)
      if (l.rhs) refs.push_back(*l.rhs);
    for (auto& r : refs)
      if (r.kind == PlanRef::Kind::kTemp && r.index < dstep) return false;
  }
  for (int k = 0; k < d.nout; ++k)
    if (!d.out_split[k]) return false;
  st.dstep = dstep;
  return compile_epilogue(p, st);
}

// Pointwise plans: every step elementwise over one common shape.
bool analyse_pointwise(const mbatch::backend::ExecutablePlan& p, TcState& st) {
  using mbatch::backend::PlanRef;
  using mbatch::backend::PlanStep;
  using mbatch::backend::Shape;
  if (p.ghost || p.steps.empty() || p.outputs.empty()) return false;
  const Shape sh = p.steps[0].out_shape;
  for (const auto& ps : p.steps) {
    if (ps.out_shape != sh) return false;
    if (ps.kind == PlanStep::Kind::kFusedDense) return false;
    if (ps.kind == PlanStep::Kind::kOp && !mbatch::backend::is_elementwise(ps.op)) return false;
    std::vector<PlanRef> refs = ps.ins;
    for (auto& l : ps.chain)
      if (l.rhs) refs.push_back(*l.rhs);
    for (auto& r : refs) {
      if (r.kind == PlanRef::Kind::kTemp) {
        if (r.cols >= 0) return false;
        continue;
      }
      const Shape in = r.kind == PlanRef::Kind::kShared ? p.shared_shapes[r.index] : p.batched_shapes[r.index];
      if (r.cols >= 0 ? !(sh.rows == 1 && r.cols == sh.cols) : !(in == sh)) return false;
    }
  }
  for (auto& o : p.outputs)
    if (o.kind != PlanRef::Kind::kTemp || o.cols >= 0) return false;
  st.dstep = -1;
  st.U = sh.size();
  st.K = 0;
  return compile_epilogue(p, st);
}

// ---- launch geometry ------------------------------------------------------------------------

struct Layout {
  int stages = 0, ring_off = 0, raw_off = 0, recv_off = 0, src_off = 0, bar_off = 0, smem = 0;
};

// Shared-memory layout of one gate launch; stages = 0 if it does not fit.  The ring holds S
// stages of (W hi|lo, X landing zone = X hi|lo) and, once drained, the staged accumulator tile;
// split-K adds the receive buffer for the peers' partial slices.
Layout layout_for(const TcState& st, int NT, int S, int npass) {
  Layout L;
  const int wpass = npass > 1 ? 2 : 1;
  const int stage_bytes = kM * st.KC * 2 * wpass + NT * st.KC * 4;
  const int stg_bytes = NT * kM * 4;
  const int recv_bytes = S > 1 ? (S - 1) * (NT / S) * kM * 4 : 0;
  const int src_bytes = st.prog.nloads * (NT / S) * st.UC * 4;
  const int bar_bytes = (4 * 6 + 3) * 8 + 8 + NT * 2 * 8 + 16;
  auto al = [](int x) { return (x + 1023) / 1024 * 1024; };
  for (int stages = 4; stages == 4; --stages) {  // MBX_STAGES in tc_gate.cuh
    const int ring_region = al(std::max(stages * stage_bytes, stg_bytes));
    const int total = ring_region + al(recv_bytes) + al(src_bytes) + bar_bytes;
    if (total <= kSmemBudget) {
      L.stages = stages;
      L.ring_off = 0;
      L.recv_off = ring_region;
      L.raw_off = 0;
      L.src_off = L.recv_off + al(recv_bytes);
      L.bar_off = L.src_off + al(src_bytes);
      L.smem = L.bar_off + bar_bytes;
      return L;
    }
  }
  return L;
}

// Persistent multi-level layout (mbx_tc_levels): the CTA's resident weight slice
// [K/S x 128 rows, hi|lo], the node-row region (doubles as the accumulator staging of the DSMEM
// exchange), the peers' partials (DSMEM exchange only) and the barriers + row table.
// deep (k = 0): the largest K split S <= 16 whose grid (unit tiles x S) fits on the 148 SMs
// (smallest resident slice; more ranks per level is faster while the grid fits: NestedRNN's inner
// cell, K = U = 512, device 6.46 / 5.03 / 4.24 / 4.06 ms at S = 2 / 4 / 8 / 16; the 16-rank
// cluster is non-portable), then the largest node tile (up to 256: TreeLSTM-512's 205-node
// depth in one tile); the ranks exchange partials through L2 unless the grid forms at most 14
// clusters of S (co-resident on a 148-SM B200: GPCs of 16-20 SMs).
// wide (k = 1, one large batch): the smallest S that fits, then the largest node tile; partials
// through DSMEM inside clusters of S, so it needs no co-residency beyond its clusters.
// Returns false if the plan has no such layout (it then runs batch by batch).
__global__ void fill_u32(unsigned* p, size_t n, unsigned v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = v;
}

bool levels_layout(TcState& st, int k, int parts, int max_ctas) {
  auto al = [](int x) { return (x + 1023) / 1024 * 1024; };
  const int utiles = st.U / st.UC;
  TcState::LevelsCfg& C = st.lv[k];
  C = TcState::LevelsCfg{};
  auto try_cfg = [&](int S, int NT) {
    if (st.nchunks % S != 0 || utiles * S > max_ctas || utiles > 64) return false;
    const int cpr = st.nchunks / S;
    if (cpr > 16) return false;
    const int xch = (S > 1 && k == 0 && utiles * S > 14 * 8) ? 1 : 0;
    // tail elements per thread x operands held in registers (MBX_LEPT x MBX_NLOADS) <= 16
    const int lloc = xch ? ((NT / 8 + S - 1) / S) * 8 : NT / S;
    if (NT / S < 2 || lloc * st.UC * std::max(1, st.prog.nloads) > 16 * kTcThreads) return false;
    const int w = al(cpr * kM * st.KC * 2 * parts);
    const int x = al(std::max(cpr * parts * (NT * st.KC * 2 + 64), xch ? 0 : NT * kM * 4));  // xstride per chunk
    const int recv = al(S > 1 && xch == 0 ? (S - 1) * (NT / S) * kM * 4 : 0);
    const int bars = (2 * cpr + 6) * 8 + NT * 16;
    if (w + x + recv + bars > kSmemBudget - kLevelsStaticSmem) return false;
    C.S = S;
    C.NT = NT;
    C.xch = xch;
    C.parts = parts;
    C.w_off = 0;
    C.x_off = w;
    C.recv_off = w + x;
    C.bar_off = w + x + recv;
    C.smem = w + x + recv + bars;
    return true;
  };
  if (k == 0 || k == 2) {
    // (k = 2: the largest K split below deep's whose grid fits twice on the SMs.)
    for (int S : {16, 8, 4, 2, 1})
      for (int NT : {256, 128, 64, 32})
        if ((k == 0 || (S < st.lv[0].S && 2 * utiles * S <= 148)) && try_cfg(S, NT)) return true;
  } else {
    // The smallest K split first (its partial exchange through DSMEM costs (S-1)/S of the
    // accumulator tile per CTA and dominates the kernel), then the largest node tile: for the
    // TreeLSTM-512 leaf batch (639 nodes, K 512) S=2 / NT=64 runs in 16.1-16.9 us against
    // 17.8-18.8 us for S=4 / NT=128 (round-1 ncu).
    for (int S : {1, 2, 4, 8})
      for (int NT : {128, 64, 32})
        if (try_cfg(S, NT)) return true;
  }
  return false;
}

// Clusters of (1, cy, cz) CTAs (one CTA per SM at this shared-memory size) that can be resident
// at once.
int max_active_clusters(void* fn, int cy, int cz, int smem) {
  static std::map<std::tuple<void*, int, int, int>, int> cache;
  static std::mutex mu;  // contexts of a pool register and launch plans concurrently
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(fn, cy, cz, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 148 / (cy * cz);
  if (fn) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, unsigned(cy), unsigned(cz));
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = size_t(smem);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = unsigned(cy);
    at[0].val.clusterDim.z = unsigned(cz);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, fn, &cfg) == cudaSuccess && m > 0) n = m;
    else cudaGetLastError();
  }
  cache[key] = n;
  return n;
}
int max_active_clusters(void* fn, int S, int smem) { return max_active_clusters(fn, 1, S, smem); }

// Tiling of one launch: NT nodes per CTA (the MMA N) and S K-split ranks per tile (cluster).
// Cost model: each CTA ingests W_tile/S + its node rows through a per-SM pipe of ~110 GB/s
// (tools/bench_bulk.cu); node tiles multiply the L2 weight traffic; S > 1 adds the DSMEM push of
// the partial accumulators; the tail costs per element.  MBX_TC_NT / MBX_TC_KSPLIT force a choice.
struct Tiling {
  int NT = 16, S = 1;
  Layout L;
};

Tiling pick_tiling(const TcState& st, int b, int npass) {
  // (the per-SM ingest and L2 figures are measured; see tools/bench_bulk.cu)
  const int utiles = st.U / st.UC;
  const double wpass = npass > 1 ? 2 : 1;
  const double w_tile_bytes = double(kM) * st.K * 2 * wpass;
  Tiling best;
  double best_t = 1e30;
  for (int nt : {16, 32, 64, 128}) {
    if (nt > 16 && nt / 2 >= b) continue;  // do not over-pad small batches
    for (int s : {1, 2, 4, 8}) {
      if (st.nchunks % s != 0 || nt % s != 0) continue;
      const int tiles = (b + nt - 1) / nt;
      const int ctas = tiles * utiles * s;
      const Layout L = layout_for(st, nt, s, npass);
      if (!L.stages) continue;
      const int clusters = ctas / s;
      const double waves = std::ceil(double(clusters) / max_active_clusters(st.fn, s, L.smem));
      const double ingest_us = (w_tile_bytes / s + double(nt) * st.K / s * 4) / 110e3;
      const double mma_us = double(st.nchunks / s) * (st.KC / 16) * npass * std::max(16, nt / 2) / 1.9e3;
      const double l2_us = (tiles * w_tile_bytes * utiles + double(b) * st.K * 4 * utiles) / 16e6;
      const double red_us = s > 1 ? double(nt) * kM * 4 * (s - 1) / s / 35e3 + 0.5 : 0.0;  // DSMEM ~18 B/clk
      const double epi_us = std::ceil(double(nt / s) * st.UC / kTcThreads) * 0.1;
      const double t = 2.0 + waves * (std::max(std::max(ingest_us, mma_us), l2_us) + red_us + epi_us);
      if (t < best_t) {
        best_t = t;
        best.NT = nt;
        best.S = s;
        best.L = L;
      }
    }
  }
  if (!best.L.stages) best.L = layout_for(st, best.NT, best.S, npass);
  return best;
}

void* load_kernel(mbx_ctx* c, const std::string& src, const char* name) {
  static const bool jit_in_dry = std::getenv("MBX_JIT_IN_DRY") != nullptr;
  if (c->dry) {
    if (jit_in_dry) jit::compile(src);  // compile-only check on GPU-less hosts
    return nullptr;
  }
  return jit::get_kernel(src, name);
}

}  // namespace

void tc_prepare(mbx_ctx* c, PlanEntry& pe) {
  pe.tc_kind = -1;
  auto st = std::make_unique<TcState>();
  if (analyse(pe.exec_plan, pe.hplan, *st)) {
    // The bit-exact CUDA-core gate kernel: unit slices of <= 32 units, 256 / slice nodes per
    // CTA (at most 8: chains are latency-bound, CTAs spread the batch), K chunks of 64 (or K).
    st->s_uc = std::min(st->U, 32);
    st->s_npc = std::max(1, std::min(kTcThreads / st->s_uc, 8));
    st->s_kb = st->K % 64 == 0 ? 64 : (st->K % 32 == 0 ? 32 : (st->K % 8 == 0 ? 8 : 0));
    // Decision-feeding cells run a few nodes per launch, many times (NestedRNN's inner loops):
    // narrow unit slices spread the weights over more CTAs, and the whole slice is staged in one
    // go (one round trip) when it fits.
    if (pe.force_vm && st->U % 8 == 0 && st->K % 8 == 0) {
      st->s_uc = 8;
      if ((st->G * (st->K + 4) * 8 + st->s_npc * st->K) * 4 <= 160 * 1024) st->s_kb = st->K;
    }
    // As many chunks in flight as ~96 KB holds (all of K when it fits: the classifier's 64 x 512
    // x 8 stages 32 KB per CTA in one round trip instead of 8 dependent ones).
    // Otherwise the largest chunk (<= 64) that keeps >= 4 stages within the budget.
    auto staging = [&](int uc, int npc, int& kb, int& stages, int& smem) {
      auto chunk = [&](int k) { return (st->G * (k + 4) * uc + npc * k) * 4; };
      const int budget = 96 * 1024;
      if (st->K / kb > 1 && chunk(st->K) <= budget) {
        kb = st->K;
      } else if (st->K / kb > 1) {
        while (kb > 8 && budget / chunk(kb) < 4 && st->K % (kb / 2) == 0) kb /= 2;
      }
      const int nch = st->K / kb;
      stages = nch == 1 ? 1 : std::max(2, std::min(nch, budget / chunk(kb)));
      smem = stages * chunk(kb);
    };
    if (st->s_kb > 0 && st->U % st->s_uc == 0) {
      const int kb0 = st->s_kb;
      staging(st->s_uc, st->s_npc, st->s_kb, st->s_st, st->s_smem);
      const std::string ssrc = gen_small_source(*st, st->s_npc, st->s_uc, st->s_kb, st->s_st);
      st->sfn = load_kernel(c, ssrc, "mbx_small_dense");
      if (st->U % 8 == 0 && st->s_uc > 8) {
        st->narrow_ok = true;
        st->nv.kb = kb0;
        staging(8, 8, st->nv.kb, st->nv.st, st->nv.smem);
        st->nv.threads = small_threads(*st, 8, 8);
      }
      pe.tc_exact = true;
      // Few output columns: tensor-core tiles would be mostly padding; exact in every precision.
      pe.tc_small = st->U * st->G <= 64;
    }
    if (pe.force_vm) {  // decision-feeding: exact only
      pe.tc_small = pe.tc_exact;
      pe.tc_kind = pe.tc_exact ? 1 : -1;
      pe.tc_state = st.release();
      return;
    }
    st->src = gen_gate_source(*st);
    st->fn = load_kernel(c, st->src, "mbx_tc_gate");
    for (int k = 0; k < 2; ++k)
      if (levels_layout(*st, k, c->precision == MBX_PREC_BF16X6 ? 3 : 2, c->sm_budget)) {
        if (k == 1 && st->lv[1].S == st->lv[0].S && st->lv[1].NT == st->lv[0].NT) {
          st->lv[1].S = 0;  // same configuration as deep
          continue;
        }
        st->lv[k].src = gen_levels_source(*st, k);
        st->lv[k].fn = load_kernel(c, st->lv[k].src, "mbx_tc_levels");
      }
    pe.tc_kind = 1;
  } else {
    *st = TcState{};
    if (!analyse_pointwise(pe.exec_plan, *st)) return;
    st->src = gen_pointwise_source(*st);
    st->fn = load_kernel(c, st->src, "mbx_pointwise");
    st->fn_fast = load_kernel(c, st->src, "mbx_pointwise_fast");
    if (st->U % 4 == 0) {
      st->fn4 = load_kernel(c, st->src, "mbx_pointwise4");
      st->fn_fast4 = load_kernel(c, st->src, "mbx_pointwise_fast4");
    }
    pe.tc_kind = 2;
  }
  pe.tc_state = st.release();
}

void tc_release(PlanEntry& pe) {
  auto* st = static_cast<TcState*>(pe.tc_state);
  if (!st) return;
  for (auto& p : st->packs) cudaFree(p.buf);
  for (auto& L : st->lv)
    for (int k = 0; k < 2; ++k) {
      if (L.part[k]) cudaFree(L.part[k]);
      if (L.flags[k]) cudaFree(L.flags[k]);
      if (L.ready[k]) cudaFree(L.ready[k]);
    }
  delete st;
  pe.tc_state = nullptr;
}

namespace {

void fill_loads(const EpiProg& pr, TcLoad* out) {
  for (int j = 0; j < pr.nloads; ++j) {
    out[j].kind = pr.loads[j].type == kSrcBatched ? 1 : 0;
    out[j].idx = pr.loads[j].idx;
    out[j].off = pr.loads[j].off;
    out[j].pad = 0;
  }
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MBX_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// The split-bf16 weight pack of a gate plan for the weights at `shared_host` (host copy of a
// staged shared-offset table); packs on first use and after every parameter upload.
// 16-byte cp.async of the gathered rows needs every row segment 16-byte aligned.
static bool rows_vec16(mbx_ctx* c, const TcState* st, const PlanEntry& pe, const BatchLaunch& L) {
  bool ok = true;
  const int64_t* shared_host = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
  const int64_t* bat = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
  const int nb = int(pe.exec_plan.batched_shapes.size());
  for (int pc = 0; pc < st->npieces; ++pc) {
    ok = ok && st->piece_off[pc] % 4 == 0 && st->piece_k[pc] % 4 == 0;
    if (st->piece_kind[pc] == kRefShared) ok = ok && shared_host[st->piece_idx[pc]] % 4 == 0;
    else
      for (int i = 0; i < L.b && ok; ++i) ok = bat[int64_t(i) * nb + st->piece_idx[pc]] % 4 == 0;
  }
  return ok;
}

static cudaError_t ensure_pack(mbx_ctx* c, TcState* st, const int64_t* shared_host, int npass, TcState::Packed** out,
                        bool* fresh) {
  const int wpass = npass_parts(npass);
  std::vector<int64_t> offs;
  for (int w : st->w_shared) offs.push_back(shared_host[w]);
  TcState::Packed* pk = nullptr;
  for (auto& p : st->packs)
    if (p.offs == offs && p.npass == npass && p.epoch == c->upload_epoch) pk = &p;
  const int ntiles = st->U / st->UC;
  const size_t chunk_bytes = size_t(kM) * st->KC * 2;
  const size_t pack_bytes = size_t(ntiles) * st->nchunks * wpass * chunk_bytes;
  *fresh = false;
  if (!pk) {
    // (Re)pack: weights changed (new offsets or a host upload since the last pack).
    for (auto it = st->packs.begin(); it != st->packs.end(); ++it)
      if (it->offs == offs && it->npass == npass) {
        cudaFree(it->buf);
        st->packs.erase(it);
        break;
      }
    TcState::Packed p;
    p.offs = offs;
    p.npass = npass;
    p.epoch = c->upload_epoch;
    cudaError_t e = cudaMalloc(&p.buf, pack_bytes);
    if (e != cudaSuccess) return e;
    int64_t* d_off = nullptr;
    e = cudaMallocAsync(&d_off, offs.size() * 8, c->stream);
    if (e != cudaSuccess) return e;
    cudaMemcpyAsync(d_off, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, c->stream);
    const int64_t total = int64_t(ntiles) * st->nchunks * kM * st->KC;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
    tc_pack_kernel<<<blocks, 256, 0, c->stream>>>(arena_ptr(c), d_off, st->G, st->K, st->U, st->UC, kM, st->KC, npass,
                                                   p.buf);
    cudaFreeAsync(d_off, c->stream);
    ++c->launches;
    st->packs.push_back(p);
    pk = &st->packs.back();
    *fresh = true;
  }
  *out = pk;
  return cudaSuccess;
}

bool tc_small_kernel(const PlanEntry& pe) {
  const auto* st = static_cast<const TcState*>(pe.tc_state);
  return pe.tc_small && st && st->sfn;
}

cudaError_t tc_launch(mbx_ctx* c, const PlanEntry& pe, const BatchLaunch& L) {
  auto* st = static_cast<TcState*>(pe.tc_state);
  if ((pe.tc_small || (pe.tc_exact && (c->precision == MBX_PREC_FP32 || c->precision == MBX_PREC_BF16X6))) && st->sfn) {
    SmallArgs a{};
    a.arena = arena_ptr(c);
    a.shared_off = meta_dev<long long>(c, L.shared_meta);
    a.batched_off = meta_dev<long long>(c, L.batched_meta);
    a.out_base = meta_dev<long long>(c, L.out_meta);
    a.out_node = L.out_node ? meta_dev<long long>(c, L.out_node_meta) : nullptr;
    a.b = L.b;
    a.nb = int(pe.exec_plan.batched_shapes.size());
    for (int i = 0; i < 2; ++i) {
      a.piece_kind[i] = st->piece_kind[i];
      a.piece_idx[i] = st->piece_idx[i];
      a.piece_off[i] = st->piece_off[i];
    }
    for (int g = 0; g < st->G; ++g) a.w_idx[g] = st->w_shared[size_t(g)];
    a.nloads = st->prog.nloads;
    fill_loads(st->prog, a.loads);
    // The wide variant unless its grid would leave most SMs idle (a few nodes over few unit
    // slices, e.g. TreeLSTM-256 b8's internal depths): then 8-unit slices, 4x the CTAs.
    // The wide variant unless its grid would leave most SMs idle (a few nodes over few unit
    // slices, e.g. TreeLSTM-256 b8's internal depths): then 8-unit slices, 4x the CTAs.
    TcState::SmallVar* nv =
        st->narrow_ok && ((L.b + st->s_npc - 1) / st->s_npc) * (st->U / st->s_uc) < 74 ? &st->nv : nullptr;
    if (nv && !nv->fn) nv->fn = load_kernel(c, gen_small_source(*st, 8, 8, nv->kb, nv->st), "mbx_small_dense");
    void* fn = nv ? nv->fn : st->sfn;
    const int npc = nv ? 8 : st->s_npc, uc = nv ? 8 : st->s_uc, smem = nv ? nv->smem : st->s_smem;
    const int threads = nv ? nv->threads : small_threads(*st, st->s_npc, st->s_uc);
    bool& attr = nv ? nv->attr : st->s_attr;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((L.b + npc - 1) / npc), unsigned(st->U / uc));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    if (pdl_enabled()) {
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    static const bool sstamps = std::getenv("MBX_SMALL_STAMPS") != nullptr;  // profiling aid
    static unsigned long long* sbuf = nullptr;
    const int nctas = int(cfg.gridDim.x * cfg.gridDim.y);
    if (sstamps) {
      if (!sbuf) cudaMalloc(&sbuf, size_t(4096) * 8 * 8);
      cudaMemsetAsync(sbuf, 0, size_t(nctas) * 8 * 8, c->stream);
      a.stamps = sbuf;
    }
    void* args[] = {&a};
    cudaError_t le = cudaLaunchKernelExC(&cfg, fn, args);
    if (sstamps && le == cudaSuccess) {
      std::vector<unsigned long long> h(size_t(nctas) * 8);
      cudaStreamSynchronize(c->stream);
      cudaMemcpy(h.data(), sbuf, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull;
      for (int i = 0; i < nctas; ++i) t0 = std::min(t0, h[size_t(i) * 8]);
      std::fprintf(stderr, "small b=%d grid=%dx%d threads=%d uc=%d:", L.b, cfg.gridDim.x, cfg.gridDim.y, threads, uc);
      for (int k = 0; k < 6; ++k) {
        double mx = 0, sum = 0;
        int cnt = 0;
        for (int i = 0; i < nctas; ++i)
          if (h[size_t(i) * 8 + k]) {
            const double v = double(h[size_t(i) * 8 + k] - t0) / 1000.0;
            mx = std::max(mx, v), sum += v, ++cnt;
          }
        std::fprintf(stderr, " s%d %.2f/%.2f", k, cnt ? sum / cnt : 0.0, mx);
      }
      std::fprintf(stderr, "\n");
    }
    return le;
  }
  if (pe.tc_kind == 2) {
    PwArgs a{};
    a.arena = arena_ptr(c);
    a.shared_off = meta_dev<long long>(c, L.shared_meta);
    a.batched_off = meta_dev<long long>(c, L.batched_meta);
    a.out_base = meta_dev<long long>(c, L.out_meta);
    a.b = L.b;
    a.E = st->U;
    a.nb = int(pe.exec_plan.batched_shapes.size());
    a.nloads = st->prog.nloads;
    fill_loads(st->prog, a.loads);
    // 16-byte variant when every row it touches is 16-byte aligned (checked on the host copies
    // of this batch's offset tables).
    // FP32 contexts: glibc-exact activations (bit-identical to the reference); the tensor-core
    // precisions use the fast ones, as their gate tails do.
    const bool exact = c->precision == MBX_PREC_FP32 || c->precision == MBX_PREC_BF16X6;
    // The exact activations are long dependent chains (double-precision expf, fdlibm expm1f,
    // divisions): one element per thread and enough CTAs to cover the SMs beats 16-byte
    // vectors on few SMs (TreeLSTM-256 b8 leaf cells, 73 x 256 elements: 19 CTAs of 4 elements
    // per thread), unless a later tensor-core level needs this launch's shadows or images.
    bool v4 = st->fn4 != nullptr && !(exact && !L.shadow_out && L.img_slot < 0);
    if (v4) {
      const int64_t* sh = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
      const int64_t* bt = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
      const int64_t* ob = reinterpret_cast<const int64_t*>(c->meta.host + L.out_meta);
      for (int k = 0; k < st->prog.nout && v4; ++k) v4 = ob[k] % 4 == 0;
      for (int j = 0; j < a.nloads && v4; ++j) {
        const TcLoad& d = a.loads[j];
        v4 = d.off % 4 == 0;
        if (d.kind == 0) v4 = v4 && sh[d.idx] % 4 == 0;
        else
          for (int i = 0; i < L.b && v4; ++i) v4 = bt[int64_t(i) * a.nb + d.idx] % 4 == 0;
      }
    }
    // Split-bf16 shadows of the outputs a later tensor-core level gathers (plan_shadows); only the
    // 16-byte variant writes them, and plan_shadows requires it.
    a.shadow = reinterpret_cast<unsigned char*>(c->shadow_base);
    a.shadow_out = v4 ? L.shadow_out : 0u;
    a.img = c->img_buf;
    a.img_slot = v4 ? L.img_slot : -1;
    a.img_dst = L.img_slot >= 0 ? meta_dev<int4>(c, L.img_dst_meta) : nullptr;
    if ((L.shadow_out || L.img_slot >= 0) && !v4) return cudaErrorInvalidValue;
    const int64_t total = int64_t(L.b) * a.E / (v4 ? 4 : 1);
    // Block size: 256, or smaller (>= 64) so that a small batch still spreads over all SMs.
    const int threads = int(std::clamp<int64_t>(((total + 147) / 148 + 31) / 32 * 32, 64, 256));
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((total + threads - 1) / threads, 148 * 8)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    if (pdl_enabled()) {
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    void* args[] = {&a};
    void* fn = exact ? (v4 ? st->fn4 : st->fn) : (v4 ? st->fn_fast4 : st->fn_fast);
    return cudaLaunchKernelExC(&cfg, fn, args);
  }
  const int npass = npass_of(c->precision);
  const int64_t* shared_host = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
  const int ntiles = st->U / st->UC;
  TcState::Packed* pk = nullptr;
  bool fresh_pack = false;
  if (cudaError_t e = ensure_pack(c, st, shared_host, npass, &pk, &fresh_pack); e != cudaSuccess) return e;
  const Tiling tl = pick_tiling(*st, L.b, npass);
  if (!tl.L.stages) return cudaErrorInvalidConfiguration;
  TcGateArgs a{};
  a.arena = arena_ptr(c);
  a.shared_off = meta_dev<long long>(c, L.shared_meta);
  a.batched_off = meta_dev<long long>(c, L.batched_meta);
  a.out_base = meta_dev<long long>(c, L.out_meta);
  a.wpack = pk->buf;
  a.b = L.b;
  a.NT = tl.NT;
  a.ksplit = tl.S;
  a.stages = tl.L.stages;
  a.nb = int(pe.exec_plan.batched_shapes.size());
  a.npass = npass;
  a.sep_recv = 0;
  for (int i = 0; i < 2; ++i) {
    a.piece_kind[i] = st->piece_kind[i];
    a.piece_idx[i] = st->piece_idx[i];
    a.piece_off[i] = st->piece_off[i];
  }
  a.nloads = st->prog.nloads;
  fill_loads(st->prog, a.loads);
  a.ring_off = tl.L.ring_off;
  a.raw_off = tl.L.raw_off;
  a.recv_off = tl.L.recv_off;
  a.src_off = tl.L.src_off;
  a.bar_off = tl.L.bar_off;
  a.tmem_cols = a.NT < 32 ? 32 : a.NT;
  // 16-byte cp.async for the gathered rows needs every row segment 16-byte aligned.
  a.vec16 = rows_vec16(c, st, pe, L) ? 1 : 0;
  if (!st->attr_set) {
    cudaError_t e = cudaFuncSetAttribute(st->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(st->fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    st->attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((L.b + a.NT - 1) / a.NT, ntiles, a.ksplit);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = size_t(tl.L.smem);
  cfg.stream = c->stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (a.ksplit > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = unsigned(a.ksplit);
    ++na;
  }
  // Programmatic dependent launch: the weight stream may start while the previous kernel drains
  // (it only reads the packed weights, which are complete unless packed just now).
  if (!fresh_pack && pdl_enabled()) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = unsigned(na);
  void* args[] = {&a};
  return cudaLaunchKernelExC(&cfg, st->fn, args);
}

// ---- persistent multi-level launches (mbx_tc_levels) ------------------------------------------

static bool levels_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MBX_LEVELS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}


// Node tiles of each level for configuration C (the smallest power of two >= b, >= 16, at most
// C.NT), and the node-tile groups (grid x) a launch uses.
static int level_tiles(const TcState::LevelsCfg& C, int utiles, const std::vector<BatchLaunch>& Ls, size_t i, int n,
                       std::vector<int>& nts, int sm_budget) {
  int max_tiles = 1;
  nts.assign(static_cast<size_t>(n), 16);
  for (int k = 0; k < n; ++k) {
    const int b = Ls[i + size_t(k)].b;
    int nt = 16;
    while (nt < b && nt < C.NT) nt *= 2;
    nt = std::max(nt, std::min(C.NT, 2 * C.S));
    nts[size_t(k)] = nt;
    max_tiles = std::max(max_tiles, (b + nt - 1) / nt);
  }
  return std::clamp(max_tiles, 1, std::max(1, sm_budget / (utiles * C.S)));
}

int plan_levels(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i, size_t* table, int* groups, int* cfg) {
  const BatchLaunch& L0 = Ls[i];
  const PlanEntry& pe = c->plans[L0.plan_id];
  if (!levels_enabled() || pe.tc_kind != 1 || pe.tc_small || c->precision == MBX_PREC_FP32 || pe.prefix_plan >= 0)
    return 0;
  auto* st = static_cast<TcState*>(pe.tc_state);
  if (!st || st->lv[0].S == 0 || (!st->lv[0].fn && !c->dry)) return 0;
  // The kernel's split parts are 1 (bf16) or its layout's MBX_LPARTS: a plan registered under
  // another multi-part precision runs batch by batch.
  const int need_parts = npass_parts(npass_of(c->precision));
  if (need_parts != 1 && need_parts != st->lv[0].parts) return 0;
  const size_t ns = pe.exec_plan.shared_shapes.size();
  const int64_t* sh0 = reinterpret_cast<const int64_t*>(c->meta.host + L0.shared_meta);
  size_t j = i;
  for (; j < Ls.size(); ++j) {
    const BatchLaunch& L = Ls[j];
    if (L.plan_id != L0.plan_id || !L.gathers.empty()) break;
    // Same weights and shared inputs: one resident weight slice serves every level.
    if (std::memcmp(c->meta.host + L.shared_meta, sh0, ns * 8) != 0) break;
  }
  const int n = int(j - i);
  if (n < 1) return 0;
  const int utiles = st->U / st->UC;
  std::vector<int> nts;
  int k = 0;
  int ng = level_tiles(st->lv[0], utiles, Ls, i, n, nts, c->sm_budget);
  // A flush with two independent runs (runtime.cpp: BiRNN's directions, issued on two streams):
  // runs take the paired configuration so that both grids are resident at once.
  if (n > 1 && c->prefer_pair && c->sm_budget > 74) {
    if (!st->pair_tried) {
      st->pair_tried = true;
      if (levels_layout(*st, 2, st->lv[0].parts, 148) && !c->dry) {
        st->lv[2].src = gen_levels_source(*st, 2);
        st->lv[2].fn = load_kernel(c, st->lv[2].src, "mbx_tc_levels");
      }
    }
    if (st->lv[2].S > 0 && (st->lv[2].fn || c->dry)) {
      k = 2;
      ng = level_tiles(st->lv[2], utiles, Ls, i, n, nts, 74);
    }
  }
  if (n == 1 && st->lv[1].S > 0 && (st->lv[1].fn || c->dry)) {
    // One batch with more node tiles than the deep configuration has groups for, or a large one
    // (>= 128 nodes: the same MMA work per CTA, but a K split of 2 exchanges an eighth of the
    // partials of deep's 8; BiRNN's 510-node input transform 33 -> ~18 us): go wide.
    // (A single-level launch with in-cluster exchange needs no co-residency and no lane: it may
    // use the whole device even in a half-device context.)
    std::vector<int> nts1;
    const int ng1 = level_tiles(st->lv[1], utiles, Ls, i, n, nts1, st->lv[1].xch == 0 ? 148 : c->sm_budget);
    if ((L0.b + nts[0] - 1) / nts[0] > ng || L0.b >= 128) {
      k = 1;
      ng = ng1;
      nts = nts1;
    }
  }
  TcState::LevelsCfg& C = st->lv[k];
  if (!c->dry) {
    if (!C.attr_set) {
      if (cudaFuncSetAttribute(C.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C.smem) != cudaSuccess ||
          cudaFuncSetAttribute(C.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      C.attr_set = true;
    }
    // Every CTA must be resident at once (readiness counters between levels, peers' partials):
    // resident clusters (DSMEM exchange) or SMs vs what one node-tile group needs.
    int resident, per_group;
    // (Half-device contexts: two such launches must fit at once.)
    const int budget = k == 2 ? 74 : (k == 1 && n == 1 && C.xch == 0) ? 148 : c->sm_budget;
    if (C.S > 1 && C.xch == 0) {
      resident = max_active_clusters(C.fn, C.S, C.smem) * budget / 148;
      per_group = utiles;
    } else {
      resident = budget;
      per_group = utiles * C.S;
    }
    if (resident < per_group) return 0;
    ng = std::min(ng, resident / per_group);
  }
  *groups = ng;
  *cfg = k;
  std::vector<TcLevel> tbl(static_cast<size_t>(n));
  for (int q = 0; q < n; ++q) {
    const BatchLaunch& L = Ls[i + size_t(q)];
    tbl[q].shared_off = meta_dev<long long>(c, L.shared_meta);
    tbl[q].batched_off = meta_dev<long long>(c, L.batched_meta);
    tbl[q].out_base = meta_dev<long long>(c, L.out_meta);
    tbl[q].b = L.b;
    tbl[q].nt = nts[size_t(q)];
    tbl[q].vec16 = rows_vec16(c, st, pe, L) ? 1 : 0;
    tbl[q].shadow = 0;      // plan_shadows decides, once every run of the flush is known
    tbl[q].shadow_out = 0;
    tbl[q].img_slot = -1;
    tbl[q].img = -1;
    tbl[q].img_dst = nullptr;
  }
  *table = meta_stage(c, tbl.data(), tbl.size() * sizeof(TcLevel));
  return n;
}

// The 16-byte pointwise variant runs (and can write shadows) when every row it touches is
// 16-byte aligned.
static bool pointwise_v4(mbx_ctx* c, const TcState* st, const PlanEntry& pe, const BatchLaunch& L) {
  if (!st->fn4 && !c->dry) return false;
  if (st->U % 4 != 0) return false;
  const int nb = int(pe.exec_plan.batched_shapes.size());
  const int64_t* sh = reinterpret_cast<const int64_t*>(c->meta.host + L.shared_meta);
  const int64_t* bt = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
  const int64_t* ob = reinterpret_cast<const int64_t*>(c->meta.host + L.out_meta);
  for (int k = 0; k < st->prog.nout; ++k)
    if (ob[k] % 4 != 0) return false;
  for (int j = 0; j < st->prog.nloads; ++j) {
    const EpiSrc& d = st->prog.loads[j];
    if (d.off % 4 != 0) return false;
    if (d.type == kSrcShared) {
      if (sh[d.idx] % 4 != 0) return false;
    } else {
      for (int i = 0; i < L.b; ++i)
        if (bt[int64_t(i) * nb + d.idx] % 4 != 0) return false;
    }
  }
  return true;
}

static int ilog2(int x) {
  int l = 0;
  while ((1 << (l + 1)) <= x) ++l;
  return l;
}

void plan_shadows(mbx_ctx* c, std::vector<BatchLaunch>& Ls, const std::vector<LevelsRun>& runs) {
  // MBX_OPERANDS=convert|shadow: restrict the operand paths (A/B measurements and tests).
  static const int allow = [] {
    const char* e = std::getenv("MBX_OPERANDS");
    return !e ? 2 : std::strcmp(e, "convert") == 0 ? 0 : std::strcmp(e, "shadow") == 0 ? 1 : 2;
  }();
  if (c->precision == MBX_PREC_FP32 || Ls.empty() || allow == 0) return;
  const int parts = npass_parts(npass_of(c->precision));
  // Output regions whose producer can write split-bf16 shadows: the pointwise kernel (16-byte
  // variant) and every level of a persistent run.  Regions never overlap (bump allocation).
  struct Region {
    int64_t lo, hi;
    int launch, slot;
  };
  std::vector<Region> regions;
  std::vector<int> run_of(Ls.size(), -1);  // launch -> index of the run covering it
  for (size_t r = 0; r < runs.size(); ++r)
    for (int q = 0; q < runs[r].n; ++q) run_of[size_t(runs[r].start) + size_t(q)] = int(r);
  for (size_t j = 0; j < Ls.size(); ++j) {
    const BatchLaunch& L = Ls[j];
    const PlanEntry& pe = c->plans[L.plan_id];
    if (pe.plan.ghost || !L.gathers.empty() || !L.sub.empty()) continue;
    bool capable = run_of[j] >= 0;
    if (!capable && pe.tc_kind == 2 && pe.tc_state)
      capable = pointwise_v4(c, static_cast<const TcState*>(pe.tc_state), pe, L);
    if (!capable) continue;
    const int64_t* ob = reinterpret_cast<const int64_t*>(c->meta.host + L.out_meta);
    for (size_t k = 0; k < pe.out_shapes.size() && k < 32; ++k)
      regions.push_back({ob[k], ob[k] + int64_t(L.b) * pe.out_shapes[k].size(), int(j), int(k)});
  }
  if (regions.empty()) return;
  std::sort(regions.begin(), regions.end(), [](const Region& a, const Region& b) { return a.lo < b.lo; });
  // (Consecutive rows of a level mostly come from one producer region: the last hit is tried
  // first, then the binary search.)
  const Region* last = nullptr;
  auto find = [&](int64_t lo, int64_t hi) -> const Region* {
    if (last && lo >= last->lo && hi <= last->hi) return last;
    auto it = std::upper_bound(regions.begin(), regions.end(), lo, [](int64_t v, const Region& r) { return v < r.lo; });
    if (it == regions.begin()) return nullptr;
    --it;
    if (lo >= it->lo && hi <= it->hi) return last = &*it;
    return nullptr;
  };
  // Per consumer level, in flush order: an operand image when every gathered row is a whole
  // output row of an earlier capable launch that no other level consumes (trees: each child row
  // feeds one parent); else MMA-ready shadow gathers when every row has a shadow; else fp32
  // gathers with the in-kernel conversion.
  // Per producer launch: its image slot (-1: none yet), per-row destinations and claim marks.
  std::vector<int> img_slot_of(Ls.size(), -1);
  std::vector<std::vector<int4>> dst(Ls.size());
  std::vector<std::vector<uint8_t>> claimed(Ls.size());
  size_t img_used = 0;
  std::vector<std::pair<int, int>> marks;
  struct Cand {
    int launch, slot, row;
    int4 d;
  };
  std::vector<Cand> cands;
  for (const LevelsRun& run : runs) {
    const BatchLaunch& L0 = Ls[size_t(run.start)];
    const PlanEntry& pe = c->plans[L0.plan_id];
    const auto* st = static_cast<const TcState*>(pe.tc_state);
    const int nb = int(pe.exec_plan.batched_shapes.size());
    const TcState::LevelsCfg& C = st->lv[run.cfg];
    const int kslice = (st->nchunks / C.S) * st->KC;
    TcLevel* tbl = reinterpret_cast<TcLevel*>(c->meta.host + run.table);
    for (int q = 0; q < run.n; ++q) {
      const size_t j = size_t(run.start) + size_t(q);
      const BatchLaunch& L = Ls[j];
      const int64_t* bt = reinterpret_cast<const int64_t*>(c->meta.host + L.batched_meta);
      const int nt = tbl[q].nt;
      // Rows that no capable launch of this flush produced (earlier flushes, inputs, other
      // kernels): neither an image nor shadow gathers can serve the level — one scan decides.
      bool produced = true;
      for (int pc = 0; pc < st->npieces && produced; ++pc) {
        if (st->piece_kind[pc] != kRefBatched) continue;
        const int width = st->piece_k[pc] - (pc ? st->piece_k[0] : 0);
        for (int i = 0; i < L.b && produced; ++i) {
          const int64_t row = bt[int64_t(i) * nb + st->piece_idx[pc]] + st->piece_off[pc];
          produced = find(row, row + width) != nullptr;
        }
      }
      if (!produced) continue;
      // -- operand image --
      bool img_ok = allow >= 2 && st->K < 4096 && kslice < 4096 && (kslice & (kslice - 1)) == 0 && nt < 65536 &&
                    (st->KC == 16 || st->KC == 32);
      cands.clear();
      const int64_t tile_bytes = int64_t(nt) * st->K * 2 * parts;
      for (int pc = 0; pc < st->npieces && img_ok; ++pc) {
        const int k0 = pc ? st->piece_k[0] : 0, width = st->piece_k[pc] - k0;
        if (st->piece_kind[pc] != kRefBatched || st->piece_off[pc] != 0 || k0 % 8 != 0) img_ok = false;
        for (int i = 0; i < L.b && img_ok; ++i) {
          const int64_t row = bt[int64_t(i) * nb + st->piece_idx[pc]];
          const Region* r = find(row, row + width);
          if (!r || size_t(r->launch) >= j) {
            img_ok = false;
            break;
          }
          const int64_t rows = (r->hi - r->lo) / std::max<int64_t>(1, Ls[size_t(r->launch)].b);
          const int pj = r->launch;
          const int ri = int((row - r->lo) / std::max<int64_t>(1, rows));
          if (rows != width || (row - r->lo) % rows != 0 || (img_slot_of[size_t(pj)] >= 0 && img_slot_of[size_t(pj)] != r->slot)) {
            img_ok = false;
            break;
          }
          auto& cl = claimed[size_t(pj)];
          if (cl.empty()) cl.assign(size_t(Ls[size_t(pj)].b), 0);
          if (cl[size_t(ri)]) {  // consumed twice (by another level, or twice by this one)
            img_ok = false;
            break;
          }
          cl[size_t(ri)] = 1;
          Cand cd;
          cd.launch = pj;
          cd.slot = r->slot;
          cd.row = ri;
          const int64_t base = int64_t(img_used) + int64_t(i / nt) * tile_bytes;
          cd.d.x = int(uint32_t(uint64_t(base) & 0xffffffffu));
          cd.d.y = int(uint32_t(uint64_t(base) >> 32));
          cd.d.z = (i % nt) | (nt << 16);
          cd.d.w = k0 | (ilog2(st->KC) << 12) | (ilog2(kslice) << 16) | (parts << 20);
          cands.push_back(cd);
        }
      }
      if (!img_ok)
        for (const Cand& cd : cands) claimed[size_t(cd.launch)][size_t(cd.row)] = 0;  // undo this level's claims
      if (img_ok) {
        for (const Cand& cd : cands) {
          img_slot_of[size_t(cd.launch)] = cd.slot;
          auto& v = dst[size_t(cd.launch)];
          if (v.empty()) v.assign(size_t(Ls[size_t(cd.launch)].b), make_int4(0, -1, 0, 0));
          v[size_t(cd.row)] = cd.d;
        }
        tbl[q].img = int64_t(img_used);
        img_used += size_t((L.b + nt - 1) / nt) * size_t(tile_bytes);
        img_used = (img_used + 1023) & ~size_t(1023);
        continue;
      }
      // -- shadow gathers (the shadow holds two parts: not for bf16x6) --
      bool ready = parts == 2;
      marks.clear();
      for (int pc = 0; pc < st->npieces && ready; ++pc) {
        const int width = st->piece_k[pc] - (pc ? st->piece_k[0] : 0);
        // Parameters (shared rows) carry no shadow; the 16-byte quads of a row must be whole
        // 8-float groups of the shadow.
        if (st->piece_kind[pc] != kRefBatched || width % 8 != 0 || st->piece_off[pc] % 8 != 0) ready = false;
        for (int i = 0; i < L.b && ready; ++i) {
          const int64_t row = bt[int64_t(i) * nb + st->piece_idx[pc]] + st->piece_off[pc];
          const Region* r = row % 8 == 0 ? find(row, row + width) : nullptr;
          if (!r || size_t(r->launch) >= j) {
            ready = false;
          } else if (marks.empty() || marks.back() != std::make_pair(r->launch, r->slot)) {
            marks.emplace_back(r->launch, r->slot);
          }
        }
      }
      if (!ready) continue;
      tbl[q].shadow = 1;
      for (auto [pj, k] : marks) {
        const int pr = run_of[size_t(pj)];
        if (pr >= 0)
          reinterpret_cast<TcLevel*>(c->meta.host + runs[size_t(pr)].table)[pj - runs[size_t(pr)].start].shadow_out |=
              1u << k;
        else
          Ls[size_t(pj)].shadow_out |= 1u << k;
      }
    }
  }
  // Stage the producers' destination tables and point them at their image slot.
  for (size_t pj = 0; pj < Ls.size(); ++pj) {
    const auto& v = dst[pj];
    const int k = img_slot_of[pj];
    if (v.empty() || k < 0) continue;
    if (c->meta.cursor % 16) {  // int4 loads: 16-byte aligned tables
      const int64_t pad = 0;
      meta_stage(c, &pad, 8);
    }
    const size_t off = meta_stage(c, v.data(), v.size() * sizeof(int4));
    const int pr = run_of[pj];
    if (pr >= 0) {
      TcLevel& t = reinterpret_cast<TcLevel*>(c->meta.host + runs[size_t(pr)].table)[int(pj) - runs[size_t(pr)].start];
      t.img_slot = k;
      t.img_dst = meta_dev<int4>(c, off);
    } else {
      Ls[pj].img_slot = k;
      Ls[pj].img_dst_meta = off;
    }
  }
  if (img_used > c->img_cap && !c->dry) {
    // Grows rarely (first mini-batches): nothing in flight may still read the old buffer.
    cuda_check(cudaStreamSynchronize(c->stream), "operand image grow");
    if (c->img_buf) cudaFree(c->img_buf);
    c->img_buf = nullptr;
    const size_t cap = std::max(img_used, c->img_cap * 2);
    cuda_check(cudaMalloc(&c->img_buf, cap), "operand images");
    // Columns past a level's last node are never written: keep them finite (zero).
    cuda_check(cudaMemsetAsync(c->img_buf, 0, cap, c->stream), "operand images");
    c->img_cap = cap;
  }
}

// Profiling aid (MBX_TC_STAMPS=1 builds only, never on a measured path): waits for the launch and
// prints, per level, the median / max over CTAs of each in-kernel clock64 phase stamp.
static void report_level_stamps(mbx_ctx* c, const unsigned long long* dev, int nctas, int n, const TcLevel* tbl,
                                const TcState::LevelsCfg& C, int cfg, int groups) {
  std::vector<unsigned long long> h(size_t(nctas) * 64 * 16);
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(h.data(), dev, h.size() * 8, cudaMemcpyDeviceToHost);
  std::fprintf(stderr, "levels: %d levels, %d CTAs (cfg %d, %d groups, S=%d, NT<=%d, exchange %s)\n", n, nctas, cfg,
               groups, C.S, C.NT, C.xch ? "L2" : "DSMEM");
  const char* names[] = {"start", "mma_wait", "mma_done", "pushed", "reduced", "tile_end", "ready", "converted",
                         "g_sync", "g_issued", "stored", "mma_issued", "tmem_stg", "tails", "entry", "summed"};
  for (int lv = 0; lv < std::min(n, 63); ++lv) {
    std::fprintf(stderr, "  lv %2d b=%3d nt=%3d sh=%d:", lv, tbl[lv].b, tbl[lv].nt, tbl[lv].shadow);
    for (int k = 0; k < 16; ++k) {
      std::vector<double> v;
      for (int i2 = 0; i2 < nctas; ++i2) {
        const unsigned long long x = h[(size_t(i2) * 64 + lv) * 16 + k];
        const unsigned long long t0 = h[size_t(i2) * 64 * 16];
        if (x && t0) v.push_back((double(x) - double(t0)) / 1965.0);
      }
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      std::fprintf(stderr, " %s %.2f/%.2f", names[k], v[v.size() / 2], v.back());
    }
    std::fprintf(stderr, "\n");
  }
}

void issue_levels(mbx_ctx* c, const std::vector<BatchLaunch>& Ls, size_t i, int n, size_t table, int groups,
                  int cfg) {
  if (c->dry) return;
  const BatchLaunch& L0 = Ls[i];
  const PlanEntry& pe = c->plans[L0.plan_id];
  auto* st = static_cast<TcState*>(pe.tc_state);
  TcState::LevelsCfg& C = st->lv[cfg];
  const int npass = npass_of(c->precision);
  const int64_t* shared_host = reinterpret_cast<const int64_t*>(c->meta.host + L0.shared_meta);
  TcState::Packed* pk = nullptr;
  bool fresh_pack = false;
  cuda_check(ensure_pack(c, st, shared_host, npass, &pk, &fresh_pack), "weight pack");
  const int utiles = st->U / st->UC;
  const int slot = c->issue_slot;
  if (!C.ready[slot]) {
    cuda_check(cudaMalloc(&C.ready[slot], size_t(64) * 32 * 4), "levels readiness counters");
    cuda_check(cudaMemsetAsync(C.ready[slot], 0, size_t(64) * 32 * 4, c->stream), "levels readiness counters");
    C.ready_count[slot] = 0;
  }
  TcLevelsArgs a{};
  a.arena = arena_ptr(c);
  a.shadow = reinterpret_cast<unsigned char*>(c->shadow_base);
  a.wpack = pk->buf;
  a.levels = meta_dev<TcLevel>(c, table);
  a.nlevels = n;
  a.nb = int(pe.exec_plan.batched_shapes.size());
  a.npass = npass;
  for (int k = 0; k < 2; ++k) {
    a.piece_kind[k] = st->piece_kind[k];
    a.piece_idx[k] = st->piece_idx[k];
    a.piece_off[k] = st->piece_off[k];
  }
  a.w_off = C.w_off;
  a.x_off = C.x_off;
  a.recv_off = C.recv_off;
  a.bar_off = C.bar_off;
  a.tmem_cols = std::max(32, C.NT);
  a.ready = C.ready[slot];
  a.ready_base = C.ready_count[slot];
  a.img = c->img_buf;
  // Unit tiles whose output columns each K rank's slice of the gathered rows covers (rows this
  // plan produced at an earlier level of the run; rows from earlier launches are complete by
  // stream order).  A piece that is not a column range of this plan's U-wide outputs depends on
  // every unit tile; parameter rows on none.
  const int cpr = st->nchunks / C.S;
  for (int r = 0; r < C.S; ++r) {
    unsigned long long m = 0;
    for (int pc = 0; pc < st->npieces; ++pc) {
      const int p0 = pc ? st->piece_k[0] : 0, p1 = st->piece_k[pc];
      const int k0 = std::max(p0, r * cpr * st->KC), k1 = std::min(p1, (r + 1) * cpr * st->KC);
      if (k0 >= k1 || st->piece_kind[pc] != kRefBatched) continue;
      const int c0 = k0 - p0 + st->piece_off[pc], c1 = k1 - p0 + st->piece_off[pc];
      if (st->piece_off[pc] + (p1 - p0) <= st->U) {
        for (int t = c0 / st->UC; t <= (c1 - 1) / st->UC; ++t) m |= 1ull << t;
      } else {
        m = ~0ull;
      }
    }
    a.dep_mask[r] = m;
  }
  if (C.xch == 1) {
    if (!C.part[slot]) {
      const size_t ngmax = size_t(std::max(1, 148 / (utiles * C.S)));
      const size_t lloc = size_t((C.NT / 8 + C.S - 1) / C.S) * 8;  // MBX_LLOC
      const size_t part_bytes = size_t(2) * ngmax * utiles * C.S * C.S * lloc * kM * 4;
      cuda_check(cudaMalloc(&C.part[slot], part_bytes), "levels partials");
      cuda_check(cudaMalloc(&C.flags[slot], ngmax * utiles * C.S * 4), "levels flags");
      cuda_check(cudaMemsetAsync(C.flags[slot], 0, ngmax * utiles * C.S * 4, c->stream), "levels flags");
    }
    a.part = C.part[slot];
    a.xflags = C.flags[slot];
  }
  fill_loads(st->prog, a.loads);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(groups), unsigned(utiles), unsigned(C.S));
  lc.blockDim = dim3(kTcThreads);
  lc.dynamicSmemBytes = size_t(C.smem);
  lc.stream = c->stream;
  cudaLaunchAttribute attrs[3];
  int na = 0;
  if (C.S > 1 && C.xch == 0) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = unsigned(C.S);
    ++na;
  }
  if (!fresh_pack && pdl_enabled()) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  // Readiness counters / cross-cluster exchange counters need every CTA resident at once.
  // Launched cooperatively, the grid is placed whole (never left spinning partly resident while
  // other contexts' kernels take the SMs it waits for), and such launches go through the
  // device's persistent lane, so two of them never run concurrently.  Not under Nsight Compute
  // (it fails cooperative launches and serialises kernels anyway).
  static const bool under_ncu = std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
                                std::getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr ||
                                std::getenv("CUDA_INJECTION64_PATH") != nullptr;
  const bool needs_all = n > 1 || (C.xch == 1 && C.S > 1);
  if (!under_ncu && needs_all) {
    attrs[na].id = cudaLaunchAttributeCooperative;
    attrs[na].val.cooperative = 1;
    ++na;
  }
  lc.attrs = attrs;
  lc.numAttrs = unsigned(na);
  const int nctas = groups * utiles * C.S;
  static unsigned long long* lstamps = nullptr;
  if (stamps_enabled()) {
    if (!lstamps) cudaMalloc(&lstamps, size_t(148) * 64 * 16 * 8);
    cudaMemsetAsync(lstamps, 0, size_t(nctas) * 64 * 16 * 8, c->stream);
    a.stamps = lstamps;
  }
  void* args[] = {&a};
  // Half-lane eligible when two such grids always fit together: at most half the SMs, and (DSMEM
  // clusters) twice its clusters co-resident.  Pool contexts planned for half the device already.
  bool half = 2 * nctas <= 148;
  if (half && c->sm_budget > 74 && C.S > 1 && C.xch == 0)
    half = 2 * groups * utiles <= max_active_clusters(C.fn, C.S, C.smem);
  if (needs_all) lc.stream = persistent_lane_begin(c, half);
  // A failed cooperative launch (e.g. too large to be co-resident) is an error, never retried as
  // a plain launch: a partly resident grid would spin at its first readiness wait.
  const cudaError_t le = cudaLaunchKernelExC(&lc, C.fn, args);
  if (needs_all) persistent_lane_end(c);
  cuda_check(le, "multi-level tensor-core kernel");
  if (stamps_enabled())
    report_level_stamps(c, lstamps, nctas, n, reinterpret_cast<const TcLevel*>(c->meta.host + table), C, cfg, groups);
  C.ready_count[slot] += unsigned(groups * C.S) * unsigned(n - 1);
  ++c->launches;
  ++g_launches;
}

}  // namespace mbx
