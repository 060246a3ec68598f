/*
 * oracle/oracle.c — THE ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of what the hot path
 * computes: the per-layer MoE block at single-request decode of arXiv 2512.16473
 * (router gating, the N-index x M-way LRU expert cache, SwiGLU expert FFNs and
 * the gate-weighted combine). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. It shares no code with the
 * CUDA path (paper_2512_16473_b200/): no headers, helpers or tables.
 *
 * Precision: bf16 inputs converted exactly to fp32, fp32 accumulation in plain
 * sequential index order (north_star: "a plain, slow fp32 CPU implementation";
 * DESIGN.md reading R5). Logits are additionally returned in fp64 for the
 * margin check. Row-parallel OpenMP only (each output element is one sequential
 * loop), so results are bit-identical for any thread count.
 *
 * Citations: P:<line> = PAPER.md, S:<line> = SPEC.md, R<k> = DESIGN.md readings.
 * Pins: tests/test_oracle_*.py. Parity of the
 * full-size output values is pinned only transitively (dense brute force and
 * float64 NumPy on small shapes, same code at scale) — "parity unpinned" beyond.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static float bf(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* ---------------------------------------------------------------- router (a1, a2)
 * P:44 "the router network determines which experts to activate"; Mixtral gating
 * (P:228 builds on the MistralAI code): logits z = Wg x, top-K, softmax over the K
 * (reading R1). Tie-break: larger z first, then lower expert index (R2).          */

/* z[e] = sum_i Wg[e][i] * x[i]   (fp32, i ascending); z64 the same in fp64. */
void oracle_gate_logits(const uint16_t* Wg, const uint16_t* x, int n, int d, float* z, double* z64) {
  for (int e = 0; e < n; ++e) {
    float acc = 0.0f;
    double acc64 = 0.0;
    for (int i = 0; i < d; ++i) {
      acc += bf(Wg[(int64_t)e * d + i]) * bf(x[i]);
      acc64 += (double)bf(Wg[(int64_t)e * d + i]) * (double)bf(x[i]);
    }
    z[e] = acc;
    if (z64) z64[e] = acc64;
  }
}

/* S[0..K-1]: the K experts with the largest z (ties: lower index first), in rank
 * order; w[r] = exp(z[S_r] - z[S_0]) / sum_q exp(z[S_q] - z[S_0]) (fp32, rank order). */
void oracle_topk_softmax(const float* z, int n, int K, int32_t* S, float* w) {
  char* taken = (char*)calloc((size_t)n, 1);
  for (int r = 0; r < K; ++r) {
    int best = -1;
    for (int e = 0; e < n; ++e) {
      if (taken[e]) continue;
      if (best < 0 || z[e] > z[best]) best = e; /* strict '>' keeps the lower index on ties */
    }
    S[r] = best;
    taken[best] = 1;
  }
  free(taken);
  const float m = z[S[0]];
  float sum = 0.0f;
  for (int r = 0; r < K; ++r) {
    w[r] = expf(z[S[r]] - m);
    sum += w[r];
  }
  for (int r = 0; r < K; ++r) w[r] = w[r] / sum;
}

/* ---------------------------------------------------------------- expert FFN (a6, a7)
 * P:44 "FFNs ... decomposed into multiple smaller expert models"; Mixtral/Phi expert
 * = SwiGLU without biases (reading R4):  o = W2 ( silu(W1 x) * (W3 x) ),
 * silu(a) = a / (1 + exp(-a)).
 *   W1, W3 : [ff][d] row-major (row j = d contiguous)
 *   W2     : [d][ff] row-major (row c = ff contiguous)
 * h (scratch, ff floats) receives the SwiGLU activations.                         */
void oracle_expert_ffn(const uint16_t* W1, const uint16_t* W3, const uint16_t* W2,
                       const uint16_t* x, int d, int ff, float* h, float* o) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < ff; ++j) {
    float g = 0.0f, u = 0.0f;
    for (int i = 0; i < d; ++i) {
      g += bf(W1[(int64_t)j * d + i]) * bf(x[i]);
      u += bf(W3[(int64_t)j * d + i]) * bf(x[i]);
    }
    h[j] = g / (1.0f + expf(-g)) * u;
  }
#pragma omp parallel for schedule(static)
  for (int c = 0; c < d; ++c) {
    float acc = 0.0f;
    for (int j = 0; j < ff; ++j) acc += bf(W2[(int64_t)c * ff + j]) * h[j];
    o[c] = acc;
  }
}

/* Gate-weighted combine (Fig.1): y[c] = sum_r w[r] * o_r[c], rank order. */
void oracle_combine(const float* o /* [K][d] */, const float* w, int K, int d, float* y) {
  for (int c = 0; c < d; ++c) {
    float acc = 0.0f;
    for (int r = 0; r < K; ++r) acc += w[r] * o[(int64_t)r * d + c];
    y[c] = acc;
  }
}

/* ---------------------------------------------------------------- expert cache (a3, a4)
 * P:196 "N-index, M-way set-associative structure spanning layers 0 through N-1";
 * P:197-198 step 1 cache check on each layer access; P:200 step 3 missed experts are
 * copied in "to update the cache for future access"; P:201 layers beyond coverage
 * never cache; P:217 LRU eviction (FIFO P:218 as the compared policy).
 * Readings: set l <-> layer l (R7); logical insertion at miss time (R11); partition
 * against the pre-access state, touch hits then insert misses in rank order, never
 * evict a way holding an expert of the current access (R10); insertion counts as a
 * use; one global recency clock (R21); warm start = experts 0..M-1 in ways
 * 0..M-1 with stamps 1..M (R9).                                                    */

enum { ORACLE_LRU = 0, ORACLE_FIFO = 1, ORACLE_STATIC = 2 };

/* P:360 random static policy: M distinct experts per covered layer, drawn once with a
 * counter-based generator (partial Fisher-Yates, splitmix64 of seed ^ layer<<32 ^ i), way i
 * holding the i-th draw; never mutated by accesses. */
static uint64_t oracle_splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t accesses, at_least_one_hit, all_k_hit, expert_hits, expert_misses, coverage_misses,
      evictions;
} oracle_stats;

typedef struct {
  int L, N, M, K, policy;
  int32_t* tag;    /* [N][M], -1 = invalid */
  uint64_t* stamp; /* [N][M] */
  uint64_t clock;
  oracle_stats* stats; /* [L] */
} oracle_cache;

oracle_cache* oracle_cache_new_seeded(int L, int N, int M, int K, int policy, int warm_start, int n,
                                     uint64_t seed);

oracle_cache* oracle_cache_new(int L, int N, int M, int K, int policy, int warm_start) {
  return oracle_cache_new_seeded(L, N, M, K, policy, warm_start, 0, 0);
}

oracle_cache* oracle_cache_new_seeded(int L, int N, int M, int K, int policy, int warm_start, int n,
                                     uint64_t seed) {
  oracle_cache* c = (oracle_cache*)calloc(1, sizeof(oracle_cache));
  c->L = L; c->N = N < L ? N : L; c->M = M; c->K = K; c->policy = policy;
  c->tag = (int32_t*)malloc(sizeof(int32_t) * (size_t)(c->N > 0 ? c->N : 1) * (size_t)(M > 0 ? M : 1));
  c->stamp = (uint64_t*)calloc((size_t)(c->N > 0 ? c->N : 1) * (size_t)(M > 0 ? M : 1), sizeof(uint64_t));
  c->stats = (oracle_stats*)calloc((size_t)L, sizeof(oracle_stats));
  for (int s = 0; s < c->N; ++s)
    for (int w = 0; w < M; ++w) {
      c->tag[s * M + w] = warm_start ? w : -1;
      c->stamp[s * M + w] = warm_start ? (uint64_t)(w + 1) : 0;
    }
  c->clock = warm_start ? (uint64_t)M : 0;
  if (policy == ORACLE_STATIC) {
    int* perm = (int*)malloc(sizeof(int) * (size_t)n);
    for (int s = 0; s < c->N; ++s) {
      for (int e = 0; e < n; ++e) perm[e] = e;
      for (int i = 0; i < M; ++i) {
        uint64_t z = oracle_splitmix(seed ^ ((uint64_t)(uint32_t)s << 32) ^ (uint64_t)(uint32_t)i);
        int j = i + (int)(z % (uint64_t)(n - i));
        int tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
      }
      for (int w = 0; w < M; ++w) {
        c->tag[s * M + w] = perm[w];
        c->stamp[s * M + w] = 0;
      }
    }
    free(perm);
    c->clock = 0;
  }
  return c;
}

void oracle_cache_free(oracle_cache* c) {
  if (!c) return;
  free(c->tag); free(c->stamp); free(c->stats); free(c);
}

/* One access of layer `layer` by the rank-ordered experts S[0..K-1].
 * Outputs per rank r: hit[r] (1/0), way[r] (-1 if uncovered), evicted[r] (-1 if none),
 * coverage[r] (1 if the layer is beyond coverage). */
void oracle_cache_access(oracle_cache* c, int layer, const int32_t* S,
                         int8_t* hit, int8_t* way, int16_t* evicted, int8_t* coverage) {
  const int K = c->K, M = c->M;
  oracle_stats* st = &c->stats[layer];
  st->accesses++;
  if (layer >= c->N) { /* P:201 / S:218: beyond coverage -> every expert a miss, no insertion */
    for (int r = 0; r < K; ++r) { hit[r] = 0; way[r] = -1; evicted[r] = -1; coverage[r] = 1; }
    st->expert_misses += (uint64_t)K;
    st->coverage_misses += (uint64_t)K;
    return;
  }
  int32_t* tag = c->tag + (int64_t)layer * M;
  uint64_t* stamp = c->stamp + (int64_t)layer * M;
  /* step 1: partition against the pre-access state */
  for (int r = 0; r < K; ++r) {
    hit[r] = 0; way[r] = -1; evicted[r] = -1; coverage[r] = 0;
    for (int w = 0; w < M; ++w)
      if (tag[w] == S[r]) { hit[r] = 1; way[r] = (int8_t)w; }
  }
  /* step 2: touch hits in rank order (LRU only; FIFO keeps insertion order) */
  for (int r = 0; r < K; ++r)
    if (hit[r] && c->policy == ORACLE_LRU) stamp[way[r]] = ++c->clock;
  if (c->policy == ORACLE_STATIC) { /* static residents: misses are never inserted */
    int nh = 0;
    for (int r = 0; r < K; ++r) nh += hit[r];
    st->expert_hits += (uint64_t)nh;
    st->expert_misses += (uint64_t)(K - nh);
    if (nh > 0) st->at_least_one_hit++;
    if (nh == K) st->all_k_hit++;
    return;
  }
  /* step 3: insert misses in rank order into the lowest invalid way, else the
   * least-recent way that holds no expert of this access */
  for (int r = 0; r < K; ++r) {
    if (hit[r]) continue;
    int v = -1;
    for (int w = 0; w < M && v < 0; ++w)
      if (tag[w] == -1) v = w;
    if (v < 0) {
      for (int w = 0; w < M; ++w) {
        int pinned = 0;
        for (int q = 0; q < K; ++q)
          if (tag[w] == S[q]) pinned = 1;
        if (pinned) continue;
        if (v < 0 || stamp[w] < stamp[v]) v = w;
      }
    }
    evicted[r] = (int16_t)tag[v];
    if (tag[v] != -1) st->evictions++;
    tag[v] = S[r];
    stamp[v] = ++c->clock;
    way[r] = (int8_t)v;
  }
  int nh = 0;
  for (int r = 0; r < K; ++r) nh += hit[r];
  st->expert_hits += (uint64_t)nh;
  st->expert_misses += (uint64_t)(K - nh);
  if (nh > 0) st->at_least_one_hit++;
  if (nh == K) st->all_k_hit++;
}

/* stats of one layer, or the sum over layers if layer < 0; out[7] in oracle_stats order */
void oracle_cache_stats(const oracle_cache* c, int layer, uint64_t* out) {
  memset(out, 0, 7 * sizeof(uint64_t));
  for (int l = 0; l < c->L; ++l) {
    if (layer >= 0 && l != layer) continue;
    const uint64_t* s = (const uint64_t*)&c->stats[l];
    for (int k = 0; k < 7; ++k) out[k] += s[k];
  }
}

/* current contents of set `layer` (tags [M], stamps [M]) for invariant checks */
void oracle_cache_set(const oracle_cache* c, int layer, int32_t* tags, uint64_t* stamps) {
  for (int w = 0; w < c->M; ++w) {
    tags[w] = c->tag[(int64_t)layer * c->M + w];
    stamps[w] = c->stamp[(int64_t)layer * c->M + w];
  }
}

/* Thread count of the row-parallel loops (bench.py's cpu_baseline times the oracle at one
 * thread and at all host threads, as Table III sweeps CPU threads). Results are
 * identical for any count: every output row is one sequential sum. */
#include <omp.h>
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_max_threads(void) { return omp_get_max_threads(); }
