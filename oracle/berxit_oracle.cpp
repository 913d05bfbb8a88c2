// berxit_oracle.cpp — TEST INFRASTRUCTURE ONLY: CPU restatement of the Berxit early-exit encoder
// (BASELINE configs[4]).  Loaded by tests/ and bench.py's cpu_baseline leg through
// ctypes; the product never links or calls it.
//
// PARITY UNPINNED.  The reference has no Berxit model (proj/src/zoo.cpp:305-317 lists rnn, birnn,
// treelstm, mvrnn, nestedrnn, drnn, stackrnn, fig5) and no softmax / layernorm / GELU op in its IR
// (proj/include/mbatch/backend.hpp:27-37), so there is no reference output to pin this file to.
// It restates the model the paper evaluates ("Early exit for BERT inference. All
// layers share weights", sequence length 128; BERT-base hyper-parameters) from
// the published algorithms:
//   * BERT encoder layer, post-LN (Devlin et al. 2019): qkv = x Wqkv^T + b; per head
//     softmax(q k^T / sqrt(dh)) v; x1 = LN(x + ctx Wo^T + bo); x2 = LN(x1 + GELU(x1 W1^T + b1) W2^T + b2);
//     GELU(x) = 0.5 x (1 + erf(x / sqrt 2)); LN over the hidden dimension, biased variance.
//   * BERxiT's learning-to-exit module (Xin et al. 2021): after every layer, certainty
//     u = sigmoid(w_lte . h_cls + b_lte) on the first token; the instance exits when u >= tau
//     (or after the last layer) with logits = Wc h_cls + bc.  One weight set for all layers.
// The batch schedule ACRoBat forms for it (one batch per layer over the instances still running,
// in instance order) follows from the exit layers: batch l = { i : exit_layer[i] >= l }.
//
// Generators (the input spec shared with the product, include/mbx_berxit.h): parameters from
// mt19937(seed*7919+17) in flat order, inputs per instance from mt19937(seed*104729+31*i+7), as the
// zoo seeds its generators (proj/src/zoo.cpp:332-341, :343-401); a uniform draw is
// lo + (hi - lo) * ((g() >> 8) * 2^-24) in float.
//
// Arithmetic: float, contractions in a fixed order (8 interleaved partial sums over k, then summed
// pairwise) so the compiler can vectorise without reassociating; expf / erff / sqrtf from libm.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

struct Cfg {
  int H, heads, F, L, S, C;
  float tau, eps;
};

struct Params {
  const float *wqkv, *bqkv, *wo, *bo, *g1, *be1, *w1, *b1, *w2, *b2, *g2, *be2, *wl, *bl, *wc, *bc;
};

int64_t param_count(const Cfg& c) {
  const int64_t H = c.H, F = c.F;
  return 3 * H * H + 3 * H + H * H + H + 2 * H + F * H + F + H * F + H + 2 * H + H + 1 + c.C * H + c.C;
}

Params bind(const Cfg& c, const float* p) {
  const int64_t H = c.H, F = c.F;
  Params r;
  r.wqkv = p; p += 3 * H * H;
  r.bqkv = p; p += 3 * H;
  r.wo = p; p += H * H;
  r.bo = p; p += H;
  r.g1 = p; p += H;
  r.be1 = p; p += H;
  r.w1 = p; p += F * H;
  r.b1 = p; p += F;
  r.w2 = p; p += H * F;
  r.b2 = p; p += H;
  r.g2 = p; p += H;
  r.be2 = p; p += H;
  r.wl = p; p += H;
  r.bl = p; p += 1;
  r.wc = p; p += c.C * H;
  r.bc = p;
  return r;
}

inline float uni(std::mt19937& g, float lo, float hi) {
  return lo + (hi - lo) * (float(g() >> 8) * (1.0f / 16777216.0f));
}

// Fixed-order dot product: 8 interleaved partial sums, then ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)).
inline float dot(const float* a, const float* b, int n) {
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int k = 0;
  for (; k + 8 <= n; k += 8)
    for (int j = 0; j < 8; ++j) s[j] += a[k + j] * b[k + j];
  for (; k < n; ++k) s[k & 7] += a[k] * b[k];
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// out[t][n] = bias[n] + x[t] . W[n]  (W row-major [N][K])
void linear(const float* x, int T, int K, const float* W, const float* bias, int N, float* out) {
  for (int t = 0; t < T; ++t)
    for (int n = 0; n < N; ++n) out[(int64_t)t * N + n] = dot(x + (int64_t)t * K, W + (int64_t)n * K, K) + bias[n];
}

void layernorm(float* x, int T, int H, const float* g, const float* b, float eps) {
  for (int t = 0; t < T; ++t) {
    float* r = x + (int64_t)t * H;
    float mean = 0;
    for (int k = 0; k < H; ++k) mean += r[k];
    mean /= float(H);
    float var = 0;
    for (int k = 0; k < H; ++k) { const float d = r[k] - mean; var += d * d; }
    var /= float(H);
    const float inv = 1.0f / std::sqrt(var + eps);
    for (int k = 0; k < H; ++k) r[k] = (r[k] - mean) * inv * g[k] + b[k];
  }
}

// One instance, layers until exit.  x: [S][H] (overwritten).  Returns the exit layer.
int run_instance(const Cfg& c, const Params& P, float* x, float* logits) {
  const int S = c.S, H = c.H, F = c.F, dh = H / c.heads;
  std::vector<float> qkv((size_t)S * 3 * H), ctx((size_t)S * H), tmp((size_t)S * H), ff((size_t)S * F),
      sc(S), kt((size_t)S * dh);
  const float scale = 1.0f / std::sqrt(float(dh));
  for (int l = 0; l < c.L; ++l) {
    linear(x, S, H, P.wqkv, P.bqkv, 3 * H, qkv.data());
    for (int h = 0; h < c.heads; ++h) {
      for (int i = 0; i < S; ++i) {
        const float* q = &qkv[(size_t)i * 3 * H + h * dh];
        float m = -INFINITY;
        for (int j = 0; j < S; ++j) {
          sc[j] = dot(q, &qkv[(size_t)j * 3 * H + H + h * dh], dh) * scale;
          m = std::max(m, sc[j]);
        }
        float sum = 0;
        for (int j = 0; j < S; ++j) { sc[j] = std::exp(sc[j] - m); sum += sc[j]; }
        const float inv = 1.0f / sum;
        float* o = &ctx[(size_t)i * H + h * dh];
        for (int d = 0; d < dh; ++d) o[d] = 0;
        for (int j = 0; j < S; ++j) {
          const float p = sc[j] * inv;
          const float* v = &qkv[(size_t)j * 3 * H + 2 * H + h * dh];
          for (int d = 0; d < dh; ++d) o[d] += p * v[d];
        }
      }
    }
    linear(ctx.data(), S, H, P.wo, P.bo, H, tmp.data());
    for (size_t k = 0; k < tmp.size(); ++k) x[k] += tmp[k];
    layernorm(x, S, H, P.g1, P.be1, c.eps);
    linear(x, S, H, P.w1, P.b1, F, ff.data());
    for (auto& v : ff) v = 0.5f * v * (1.0f + std::erf(v * 0.70710678118654752f));
    linear(ff.data(), S, F, P.w2, P.b2, H, tmp.data());
    for (size_t k = 0; k < tmp.size(); ++k) x[k] += tmp[k];
    layernorm(x, S, H, P.g2, P.be2, c.eps);
    const float z = dot(P.wl, x, H) + P.bl[0];
    const float u = 1.0f / (1.0f + std::exp(-z));
    if (u >= c.tau || l == c.L - 1) {
      for (int k = 0; k < c.C; ++k) logits[k] = dot(P.wc + (int64_t)k * H, x, H) + P.bc[k];
      return l;
    }
  }
  return c.L - 1;
}

}  // namespace

extern "C" {

int64_t orc_berxit_param_count(int H, int heads, int F, int L, int S, int C) {
  Cfg c{H, heads, F, L, S, C, 0, 0};
  return param_count(c);
}

// Flat parameters in the documented order; ranges: weights U[-0.05, 0.05), biases U[-0.02, 0.02),
// LN gains U[0.9, 1.1), LN shifts U[-0.1, 0.1), w_lte U[-0.1, 0.1), b_lte U[-0.1, 0.1).
void orc_berxit_make_params(int H, int heads, int F, int L, int S, int C, unsigned seed, float* out) {
  Cfg c{H, heads, F, L, S, C, 0, 0};
  std::mt19937 g(seed * 7919u + 17u);
  const int64_t h = H, f = F;
  auto fill = [&](int64_t n, float lo, float hi) { for (int64_t k = 0; k < n; ++k) *out++ = uni(g, lo, hi); };
  const float a = 0.05f, bb = 0.02f;
  fill(3 * h * h, -a, a); fill(3 * h, -bb, bb);
  fill(h * h, -a, a); fill(h, -bb, bb);
  fill(h, 0.9f, 1.1f); fill(h, -0.1f, 0.1f);
  fill(f * h, -a, a); fill(f, -bb, bb);
  fill(h * f, -a, a); fill(h, -bb, bb);
  fill(h, 0.9f, 1.1f); fill(h, -0.1f, 0.1f);
  fill(h, -0.1f, 0.1f); fill(1, -0.1f, 0.1f);
  fill(C * h, -a, a); fill(C, -bb, bb);
  (void)c;
}

// Instance i's input [S][H], U[-1, 1).
void orc_berxit_make_input(int H, int S, unsigned seed, int i, float* out) {
  std::mt19937 g(seed * 104729u + 31u * unsigned(i) + 7u);
  for (int64_t k = 0; k < (int64_t)S * H; ++k) out[k] = uni(g, -1.0f, 1.0f);
}

// Evaluates the n instances whose inputs are x[n][S][H] (independently, on `threads` threads):
// logits[n][C], exit_layer[n].
int orc_berxit_run(int H, int heads, int F, int L, int S, int C, float tau, float eps, const float* params, int n,
                   const float* x, float* logits, int32_t* exit_layer, int threads) {
  Cfg c{H, heads, F, L, S, C, tau, eps};
  if (H % heads) return 1;
  const Params P = bind(c, params);
  auto work = [&](int t) {
    std::vector<float> xi((size_t)S * H);
    for (int i = t; i < n; i += threads) {
      std::memcpy(xi.data(), x + (size_t)i * S * H, sizeof(float) * S * H);
      exit_layer[i] = run_instance(c, P, xi.data(), logits + (size_t)i * C);
    }
  };
  if (threads <= 1) {
    threads = 1;
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
    for (auto& t : th) t.join();
  }
  return 0;
}

}  // extern "C"
