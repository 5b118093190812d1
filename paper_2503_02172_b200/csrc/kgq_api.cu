// libkgq.so: C ABI (include/kgq.h) + host planner.
//
// The planner replaces the paper's Graph Capturer / Pattern Recognizer / Operator Fuser
// (Eq. 2, Eq. 4, Alg. 1) by static per-structure plans decided
// at compile time: for each query structure it launches a fixed chain of fused kernels
// (horizontal fusion of projection chains, vertical fusion of branches, union fused into the
// scorer), then the entity scorer and the top-k selection, all on the caller's stream.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kgq_internal.cuh"
#include "nccl_dl.h"

using namespace kgq;

namespace kgq {

// ---- static plans --------------------------------------------------------
#define BR(a, n, o0, o1, o2) {a, n, {o0, o1, o2, 0}}
static const Plan kPlans[KGQ_NUM_STRUCTURES] = {
    /* 1p  */ {kSingle, 1, {BR(0, 1, 0, 0, 0)}, 0, {0, 0}, 1, 1, 1, false},
    /* 2p  */ {kSingle, 1, {BR(0, 2, 0, 1, 0)}, 0, {0, 0}, 1, 2, 1, false},
    /* 3p  */ {kSingle, 1, {BR(0, 3, 0, 1, 2)}, 0, {0, 0}, 1, 3, 1, false},
    /* 2i  */ {kInter, 2, {BR(0, 1, 0, 0, 0), BR(1, 1, 1, 0, 0)}, 0, {0, 0}, 2, 2, 1, false},
    /* 3i  */ {kInter, 3, {BR(0, 1, 0, 0, 0), BR(1, 1, 1, 0, 0), BR(2, 1, 2, 0, 0)}, 0, {0, 0}, 3, 3, 1, false},
    /* pi  */ {kInter, 2, {BR(0, 2, 0, 1, 0), BR(1, 1, 2, 0, 0)}, 0, {0, 0}, 2, 3, 1, false},
    /* ip  */ {kInter, 2, {BR(0, 1, 0, 0, 0), BR(1, 1, 1, 0, 0)}, 1, {2, 0}, 2, 3, 1, false},
    /* 2u  */ {kUnion, 2, {BR(0, 1, 0, 0, 0), BR(1, 1, 1, 0, 0)}, 0, {0, 0}, 2, 2, 2, false},
    /* up  */ {kUnion, 2, {BR(0, 2, 0, 2, 0), BR(1, 2, 1, 2, 0)}, 0, {0, 0}, 2, 3, 2, false},
    /* 2in */ {kInter, 2, {BR(0, 1, 0, 0, 0), BR(1, 2, 1, kOpNeg, 0)}, 0, {0, 0}, 2, 2, 1, true},
    /* 3in */ {kInter, 3, {BR(0, 1, 0, 0, 0), BR(1, 1, 1, 0, 0), BR(2, 2, 2, kOpNeg, 0)}, 0, {0, 0}, 3, 3, 1, true},
    /* inp */ {kInter, 2, {BR(0, 1, 0, 0, 0), BR(1, 2, 1, kOpNeg, 0)}, 1, {2, 0}, 2, 3, 1, true},
    /* pin */ {kInter, 2, {BR(0, 2, 0, 1, 0), BR(1, 2, 2, kOpNeg, 0)}, 0, {0, 0}, 2, 3, 1, true},
    /* pni */ {kInter, 2, {BR(0, 3, 0, 1, kOpNeg), BR(1, 1, 2, 0, 0)}, 0, {0, 0}, 2, 3, 1, true},
    /* 2u-DM */ {kInter, 2, {BR(0, 2, 0, kOpNeg, 0), BR(1, 2, 1, kOpNeg, 0)}, 0, {0, 0}, 2, 2, 1, true, true},
    /* up-DM */ {kInter, 2, {BR(0, 2, 0, kOpNeg, 0), BR(1, 2, 1, kOpNeg, 0)}, 1, {2, 0}, 2, 3, 1, true, true},
};
#undef BR
static const char* kNames[KGQ_NUM_STRUCTURES] = {"1p", "2p", "3p", "2i", "3i", "pi", "ip",
                                                 "2u", "up", "2in", "3in", "inp", "pin", "pni",
                                                 "2u-DM", "up-DM"};
const Plan* plan_of(int s) {
  return (s >= 0 && s < KGQ_NUM_STRUCTURES) ? &kPlans[s] : nullptr;
}

}  // namespace kgq

namespace {

thread_local std::string g_create_err;

kgq_status fail(kgq_ctx* c, kgq_status s, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
kgq_status fail(kgq_ctx* c, kgq_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_create_err = buf;
  return s;
}

kgq_status cuda_fail(kgq_ctx* c, cudaError_t e, const char* what) {
  return fail(c, e == cudaErrorMemoryAllocation ? KGQ_ENOMEM : KGQ_ECUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define CK(call, what)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
  } while (0)

template <typename T>
kgq_status dalloc(kgq_ctx* ctx, T** p, size_t n, const char* what) {
  *p = nullptr;
  if (n == 0) return KGQ_OK;
  CK(cudaMalloc((void**)p, n * sizeof(T)), what);
  return KGQ_OK;
}

// Three bf16 planes of [rows, ld] in one allocation (freed through b0); ld = w rounded up to 8
// elements so every row starts 16-byte aligned (TMA operand maps).
kgq_status alloc_split(kgq_ctx* ctx, Split* s, int64_t rows, int64_t w, const char* what) {
  s->ld = (w + 7) / 8 * 8;
  const size_t plane = (size_t)(rows * s->ld);
  kgq_status st = dalloc(ctx, &s->b0, 3 * plane, what);
  if (st) return st;
  s->b1 = s->b0 + plane;
  s->b2 = s->b1 + plane;
  return KGQ_OK;
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---- profiling (CUDA events on the launching stream) ------------------------------------
struct StageTimer {
  kgq_ctx* ctx;
  cudaStream_t st;
  int stage;
  cudaEvent_t a = nullptr;
  double work;
  StageTimer(kgq_ctx* c, cudaStream_t s, int stg, double w = 0.0) : ctx(c), st(s), stage(stg), work(w) {
    if (!ctx->profile) return;
    cudaEventCreate(&a);
    record(a);
  }
  // inside stream capture the record must be an external event-record node to be replayed
  void record(cudaEvent_t e) {
    if (ctx->capture_entry)
      cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else
      cudaEventRecord(e, st);
  }
  ~StageTimer() {
    if (!ctx->profile) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    record(b);
    if (ctx->capture_entry)
      ctx->capture_entry->evs.push_back({stage, a, b, work});
    else
      ctx->prof_recs.push_back({stage, a, b, work});
  }
};

// Fold completed stage events into the context's accumulators.
void harvest(kgq_ctx* ctx, std::vector<ProfRec>& recs, bool destroy) {
  for (auto& r : recs) {
    float t = 0;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();  // do not leave a sticky error for the next checked call
      t = 0;
    }
    ctx->prof_acc_ms[r.stage] += t;
    ctx->prof_acc_n[r.stage] += 1;
    ctx->prof_acc_work[r.stage] += r.work;
    if (destroy) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
  if (destroy) recs.clear();
}

void destroy_graph_entry(kgq_ctx::GraphEntry& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& r : g.evs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g.evs.clear();
}

void clear_mix_graphs(kgq_ctx* ctx) {
  for (auto& m : ctx->mgraphs) {
    if (m.exec) cudaGraphExecDestroy(m.exec);
    if (m.map_host) cudaFreeHost(m.map_host);
  }
  ctx->mgraphs.clear();
}


ChainArgs chain_args(kgq_ctx* ctx, const Plan* P, int B, const int32_t* anchors,
                     const int32_t* rels) {
  ChainArgs a{};
  a.model = ctx->cfg.model;
  a.d = ctx->cfg.dim;
  a.nb = P->nbranch;
  for (int i = 0; i < P->nbranch; ++i) a.br[i] = P->br[i];
  a.anchors = anchors;
  a.n_a = P->n_anchor;
  a.rels = rels;
  a.n_r = P->n_rel;
  a.n_entity = ctx->cfg.n_entity;
  a.n_relation = ctx->cfg.n_relation;
  a.err = ctx->d_err;
  a.invalid = ctx->d_invalid;
  (void)B;
  return a;
}

// Every dense layer of the chain goes through here: timed as stage kStDense when profiling,
// with 2 M N K algorithmic FLOPs.
// KGQ_DEBUG_LAUNCH=1: report the first failing launch (by site) on stderr.
bool debug_launch() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KGQ_DEBUG_LAUNCH");
    v = (e && e[0] && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}
bool relterm_disabled() {  // KGQ_NO_RELTERM=1: first projection layer on the assembled [x; R[r]] input
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KGQ_NO_RELTERM");
    v = (e && e[0] && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}
// fp16x2 range flags of every converting translation unit (process-wide per device: any context's
// conversion since the last check)
static bool range_flags_taken() {
  const unsigned int a = range_flag_chain(), b = range_flag_linear(), c = range_flag_score_tc();
  return (a | b | c) != 0;
}

// Hop-0 first layer from a per-entity precompute (chain.cu k_mix_h0_pre) when the [N, H] fp32
// table fits this budget; KGQ_NO_HPRE=1 disables it (A/B)
constexpr double kHpreBytesMax = 2.0 * (1ull << 30);
static bool hpre_enabled() {
  static const bool v = [] {
    const char* e = getenv("KGQ_NO_HPRE");
    return !(e && e[0] && e[0] != '0');
  }();
  return v;
}

// KGQ_NO_FUSED_TOPK=1: new contexts default to KGQ_FUSED_OFF (A/B runs)
bool fused_topk_disabled() {
  static const bool v = [] {
    const char* e = getenv("KGQ_NO_FUSED_TOPK");
    return e && e[0] && e[0] != '0';
  }();
  return v;
}
// Fused top-k for a tensor-core scorer launch of `rows` GEMM rows?  AUTO: only launches of
// >= 8,192 rows -- each list's warm-up (the first ~10 chunks insert on almost every position,
// and a warp pays for every lane's insert) costs about one tile, so stripes must be long and the
// rows many for the saved top-k pass to win; measured on C2.
// AUTO keeps every stripe >= 16 tiles long; ON (tests) lets the planner cut as many stripes as
// balance the machine best (up to 64)
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && e[0] ? atoi(e) : dflt;
}
static int topk_min_tiles(const kgq_ctx* ctx) {
  static const int auto_min = env_int("KGQ_TOPK_MIN_TILES", 16);  // tuning experiments only
  return ctx->fused_topk == KGQ_FUSED_ON ? 1 : auto_min;
}
// AUTO: fuse launches of >= 8,192 rows, or any launch whose 256 x 256 tiles per cluster (74 per
// B200) reach 64 -- long stripes amortise the lists' warm-up: the 2M-entity table (C5b) at 1,024
// rows has ~420 tiles per cluster and gains 13% from the fused top-k (no 8 GB distance block per
// chunk), while C2's 4,096 union rows (~12 tiles per cluster) lose with it
static bool use_fused_topk(const kgq_ctx* ctx, int64_t rows, int k) {
  static const int auto_rows = env_int("KGQ_TOPK_AUTO_ROWS", 8192);  // tuning experiments only
  static const int auto_tiles = env_int("KGQ_TOPK_AUTO_TILES", 64);  // tuning experiments only
  if (k > kFusedTopkMax || ctx->fused_topk == KGQ_FUSED_OFF) return false;
  const double tiles_per_cluster = (double)((rows + 255) / 256) * (double)((ctx->np + 255) / 256) / 74.0;
  return ctx->fused_topk == KGQ_FUSED_ON || rows >= auto_rows || tiles_per_cluster >= auto_tiles;
}
bool topk_cmin_disabled() {  // KGQ_NO_TOPK_CMIN=1: full-row top-k (A/B and debugging)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KGQ_NO_TOPK_CMIN");
    v = (e && e[0] && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}
void check_site(const char* site) {
  if (!debug_launch()) return;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) fprintf(stderr, "libkgq: launch error after %s: %s\n", site, cudaGetErrorString(e));
}

// dense layer into a split (bf16x3) state, or into an fp32 buffer [M, ld]
int dense(kgq_ctx* ctx, const Split& A, int M, int K, const Linear& L, int epi, const Split& out, int neg0,
          int neg1, cudaStream_t st, const GemmWs* ws = nullptr) {
  StageTimer t(ctx, st, kStDense, 2.0 * M * (double)L.out_f * K);
  const int r = launch_linear(A, M, K, L, epi, out, nullptr, 0, neg0, neg1, ws ? ws : &ctx->gws, st);
  check_site("dense layer");
  return r;
}
int dense(kgq_ctx* ctx, const Split& A, int M, int K, const Linear& L, int epi, float* out, int64_t ld,
          cudaStream_t st, const GemmWs* ws = nullptr) {
  StageTimer t(ctx, st, kStDense, 2.0 * M * (double)L.out_f * K);
  const int r = launch_linear(A, M, K, L, epi, Split{}, out, ld, 0, 0, ws ? ws : &ctx->gws, st);
  check_site("dense layer");
  return r;
}

// BetaE: one projection hop (Eq. 4 MLP) for the contiguous branch run [br0, br0+n) of rows
// B each.  Input from anchors (hop 0) or state S; output written back into S rows; rows of
// branches whose next op is a negation get 1/x in the same epilogue.
int betae_hop(kgq_ctx* ctx, const ChainArgs& ca, int B, int hop, int br0, int n,
              const int (*proj)[kMaxOps], const bool (*neg_after)[kMaxOps], Split src_state,
              int64_t src_row0, cudaStream_t st) {
  const int d = ctx->cfg.dim;
  MlpGroup g{};
  g.n = n;
  for (int gi = 0; gi < n; ++gi) {
    const int br = br0 + gi;
    g.rel_slot[gi] = proj[br][hop];
    g.anchor_slot[gi] = hop == 0 && src_row0 < 0 ? ca.br[br].anchor : -1;
    g.src_row[gi] = src_row0 < 0 ? (int64_t)br * B : src_row0 + (int64_t)gi * B;
  }
  int L = 0;
  const int M = n * B;
  Split A = ctx->Z;
  int K = 3 * d;
  int l0 = 0;
  if (ctx->RW) {
    // first layer with the relation input factored out (RelTerm): K = 2d straight from the state
    // rows (contiguous run) or from the gathered anchor rows; accumulators start at RW[r]
    if (src_row0 < 0 && ctx->Hpre) {
      // hop 0 from the per-entity precompute: H0 = ReLU(Hpre[anchor] + RW[r]) (b1 is in Hpre), no GEMM
      MixSegs sg;
      for (int gi = 0; gi < n; ++gi) {
        MixSeg& m = sg.s[sg.n++];
        m.dst0 = gi * B; m.B = B; m.q0 = 0; m.kind = 0; m.src0 = 0;
        m.anchors = ca.anchors; m.n_a = ca.n_a; m.aslot = g.anchor_slot[gi];
        m.rels = ca.rels; m.n_r = ca.n_r; m.rslot = g.rel_slot[gi];
      }
      L += launch_mix_h0_pre(sg, M, ctx->Hpre, ctx->RW, ctx->lin1x.out_f, ctx->H[0], ctx->cfg.n_entity,
                             ctx->cfg.n_relation, ca.err, ca.invalid, st);
    } else {
      if (src_row0 < 0) {
        L += launch_betae_mlp_input(ca, ctx->ent, ctx->rel[0], B, g, src_state, ctx->Z, st, false);
        A = ctx->Z;
      } else {
        A = src_state.at(src_row0);
      }
      RelTerm rt;
      rt.RW = ctx->RW;
      rt.ldrw = ctx->cfg.hidden;
      rt.M = M;
      rt.B = B;
      rt.rels = ca.rels;
      rt.n_r = ca.n_r;
      rt.n_relation = ca.n_relation;
      for (int gi = 0; gi < n; ++gi) rt.rel_slot[gi] = g.rel_slot[gi];
      rt.err = ca.err;
      rt.invalid = ca.invalid;
      {
        StageTimer t(ctx, st, kStDense, 2.0 * M * (double)ctx->lin1x.out_f * 2 * d);
        L += launch_linear_rel(A, M, 2 * d, ctx->lin1x, rt, ctx->H[0], &ctx->gws, st);
        check_site("dense layer (relation term)");
      }
    }  // first layer done (precompute gather or GEMM)
    A = ctx->H[0];
    K = ctx->lin1x.out_f;
    l0 = 1;
  } else {
    L += launch_betae_mlp_input(ca, ctx->ent, ctx->rel[0], B, g, src_state, ctx->Z, st);
  }
  for (int l = l0; l < ctx->cfg.n_hidden_layers; ++l) {
    const Linear& lin = ctx->lin[KGQ_LAYER_PROJ_HIDDEN + l];
    L += dense(ctx, A, M, K, lin, kEpiRelu, ctx->H[l & 1], 0, 0, st);
    A = ctx->H[l & 1];
    K = lin.out_f;
  }
  int neg0 = M, neg1 = M;  // rows of this group to negate (a single interval suffices for the
  std::vector<std::pair<int, int>> extra;  // 14 plans; other patterns get extra launches)
  for (int gi = 0; gi < n; ++gi) {
    if (!neg_after[br0 + gi][hop]) continue;
    const int r0 = gi * B, r1 = r0 + B;
    if (neg0 == M) {
      neg0 = r0;
      neg1 = r1;
    } else if (r0 == neg1) {
      neg1 = r1;
    } else {
      extra.emplace_back(r0, r1);
    }
  }
  Split out = ctx->S.at((int64_t)br0 * B);
  const Linear& lo = ctx->lin[KGQ_LAYER_PROJ_OUT];
  if (ctx->cfg.terminal == KGQ_TERM_SOFTMAX) {
    L += dense(ctx, A, M, K, lo, kEpiNone, ctx->T, 2 * d, st);
    L += launch_softmax_terminal(ctx->T, 2 * d, M, 2 * d, out, 0, neg0, neg1, st);
  } else {
    L += dense(ctx, A, M, K, lo, kEpiBetaReg, out, neg0, neg1, st);
  }
  for (auto& e : extra) L += launch_negate(out, e.first, e.second, 2 * d, st);
  return L;
}

// Operator chain for one batch: writes ctx->Q [B, n_out, qw].
int run_chain(kgq_ctx* ctx, int s, int B, const int32_t* anchors, const int32_t* rels,
              cudaStream_t st, bool want_q = true) {
  const Plan* P = plan_of(s);
  const int model = ctx->cfg.model;
  const int d = ctx->cfg.dim;
  ChainArgs ca = chain_args(ctx, P, B, anchors, rels);
  int L = 0;
  const int nb = P->nbranch;
  const int64_t M = (int64_t)nb * B;

  if (model != KGQ_BETAE) {
    if (P->kind != kInter) {
      return launch_translate_chain(ca, ctx->ent, ctx->rel[0], ctx->rel[1], B, Split{}, ctx->Q, st);
    }
    L += launch_translate_chain(ca, ctx->ent, ctx->rel[0], ctx->rel[1], B, ctx->S, nullptr, st);
    // attention logits over centres (Q6): W2 ReLU(W1 x + b1) + b2, rows br*B + b
    const Split centres = ctx->S;
    L += dense(ctx, centres, (int)M, d, ctx->lin[KGQ_LAYER_INTER_1], kEpiRelu, ctx->I, 0, 0, st);
    L += dense(ctx, ctx->I, (int)M, d, ctx->lin[KGQ_LAYER_INTER_2], kEpiNone, ctx->T, ctx->tw, st);
    const float* gate = nullptr;
    if (model == KGQ_Q2B) {  // offset gate: sigmoid(V2 mean_i ReLU(V1 o_i + c1) + c2)
      const Split offs = ctx->S.at(0, q2b_off(d));  // offsets start 16-byte aligned (common.cuh)
      L += dense(ctx, offs, (int)M, d, ctx->lin[KGQ_LAYER_OFFSET_1], kEpiRelu, ctx->T2, ctx->tw, st);
      L += launch_branch_mean(ctx->T2, ctx->tw, nb, B, d, ctx->M, st);
      L += dense(ctx, ctx->M, B, d, ctx->lin[KGQ_LAYER_OFFSET_2], kEpiNone, ctx->T2, ctx->tw, st);
      gate = ctx->T2;
    }
    CombineArgs c{};
    c.model = model; c.nb = nb; c.B = B; c.d = d; c.ldl = ctx->tw; c.ldg = ctx->tw;
    c.rel = ctx->rel[0]; c.rel_off = ctx->rel[1]; c.rels = rels; c.n_r = P->n_rel;
    c.n_relation = ctx->cfg.n_relation; c.post_slot = P->npost ? P->post[0] : -1;
    c.err = ctx->d_err; c.invalid = ctx->d_invalid;
    L += launch_attention_combine(c, ctx->S, ctx->T, gate, Split{}, ctx->Q, st);
    return L;
  }

  // ---- BetaE ------------------------------------------------------------------------------
  int proj[kMaxBranches][kMaxOps];
  bool neg_after[kMaxBranches][kMaxOps];
  int nproj[kMaxBranches];
  int maxh = 0;
  for (int br = 0; br < nb; ++br) {
    nproj[br] = 0;
    for (int o = 0; o < P->br[br].nops; ++o) {
      const int op = P->br[br].ops[o];
      if (op == kOpNeg) {
        neg_after[br][nproj[br] - 1] = true;  // plans never negate a bare anchor
      } else {
        proj[br][nproj[br]] = op;
        neg_after[br][nproj[br]] = false;
        nproj[br]++;
      }
    }
    maxh = std::max(maxh, nproj[br]);
  }
  for (int h = 0; h < maxh; ++h) {
    int br = 0;
    while (br < nb) {  // contiguous runs of branches that still project at hop h
      if (nproj[br] <= h) { ++br; continue; }
      int e = br;
      while (e < nb && nproj[e] > h) ++e;
      L += betae_hop(ctx, ca, B, h, br, e - br, proj, neg_after, ctx->S, h == 0 ? -1 : (int64_t)br * B,
                     st);
      br = e;
    }
  }
  if (P->kind != kInter) return want_q ? L + launch_state_to_q(ctx->S, P->n_out, B, 2 * d, ctx->Q, st) : L;
  // intersection (Q6): attention over [alpha_i; beta_i] (2d -> 2d -> d), shared weights a_i
  L += dense(ctx, ctx->S, (int)M, 2 * d, ctx->lin[KGQ_LAYER_INTER_1], kEpiRelu, ctx->I, 0, 0, st);
  L += dense(ctx, ctx->I, (int)M, 2 * d, ctx->lin[KGQ_LAYER_INTER_2], kEpiNone, ctx->T, ctx->tw, st);
  CombineArgs c{};
  c.model = model; c.nb = nb; c.B = B; c.d = d; c.ldl = ctx->tw; c.ldg = 0;
  c.rels = rels; c.n_r = P->n_rel; c.n_relation = ctx->cfg.n_relation; c.post_slot = -1;
  c.negate_out = P->neg_inter ? 1 : 0;
  c.err = ctx->d_err; c.invalid = ctx->d_invalid;
  if (P->npost == 0)
    return L + launch_attention_combine(c, ctx->S, ctx->T, nullptr, Split{}, ctx->Q, st);
  L += launch_attention_combine(c, ctx->S, ctx->T, nullptr, ctx->M, nullptr, st);
  // post projections (ip, inp): MLP hops on the combined state, result in S rows [0, B)
  int pproj[kMaxBranches][kMaxOps] = {};
  bool pneg[kMaxBranches][kMaxOps] = {};
  Split src = ctx->M;
  for (int p = 0; p < P->npost; ++p) {
    pproj[0][p] = P->post[p];
    ChainArgs cb = ca;
    L += betae_hop(ctx, cb, B, p, 0, 1, pproj, pneg, src, 0, st);
    src = ctx->S;
  }
  return want_q ? L + launch_state_to_q(ctx->S, 1, B, 2 * d, ctx->Q, st) : L;
}

// True when every chunk of a BetaE batch of B queries is scored on the tensor cores and the
// chain's final state stays in the split state rows S (no intersection as the last operator):
// the scorer's prep then reads S directly and the chain skips the fp32 Q copy.
static bool q_in_state(const kgq_ctx* ctx, const Plan* P, int B) {
  if (ctx->cfg.model != KGQ_BETAE || (P->kind == kInter && P->npost == 0)) return false;
  for (int64_t b0 = 0; b0 < B; b0 += ctx->bchunk)
    if (score_uses_stream(KGQ_BETAE, P->n_out, (int)std::min<int64_t>(ctx->bchunk, B - b0))) return false;
  return true;
}

kgq_status check_submit(kgq_ctx* ctx, int32_t s, int32_t batch, int32_t k, bool need_k) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (!ctx->finalized) return fail(ctx, KGQ_ESTATE, "kgq_finalize() has not been called");
  const Plan* P = plan_of(s);
  if (!P)
    return fail(ctx, KGQ_EINVAL,
                "unknown structure %d; valid: 0..13 = 1p 2p 3p 2i 3i pi ip 2u up 2in 3in inp pin pni", s);
  if (P->negation && ctx->cfg.model != KGQ_BETAE)
    return fail(ctx, KGQ_EUNSUPPORTED, "structure %s uses negation; GQE/Q2B do not support the n operator",
                kNames[s]);
  if (batch < 0 || batch > ctx->cfg.max_batch)
    return fail(ctx, KGQ_EINVAL, "batch %d outside [0, max_batch=%d]", batch, ctx->cfg.max_batch);
  if (need_k && (k < 1 || k > ctx->cfg.max_k || k > ctx->ns))
    return fail(ctx, KGQ_EINVAL, "k %d outside [1, min(max_k=%d, shard size=%lld)]", k, ctx->cfg.max_k,
                (long long)ctx->ns);
  return KGQ_OK;
}

}  // namespace

// =========================================================================================
extern "C" {

const char* kgq_status_string(kgq_status s) {
  switch (s) {
    case KGQ_OK: return "KGQ_OK";
    case KGQ_EINVAL: return "KGQ_EINVAL";
    case KGQ_ERANGE: return "KGQ_ERANGE";
    case KGQ_EUNSUPPORTED: return "KGQ_EUNSUPPORTED";
    case KGQ_ESTATE: return "KGQ_ESTATE";
    case KGQ_ENOMEM: return "KGQ_ENOMEM";
    case KGQ_ECUDA: return "KGQ_ECUDA";
    case KGQ_ENCCL: return "KGQ_ENCCL";
  }
  return "KGQ_UNKNOWN";
}

int32_t kgq_num_anchors(int32_t s) { return plan_of(s) ? plan_of(s)->n_anchor : -1; }
int32_t kgq_num_relations(int32_t s) { return plan_of(s) ? plan_of(s)->n_rel : -1; }
int32_t kgq_num_branches(int32_t s) { return plan_of(s) ? plan_of(s)->n_out : -1; }
int32_t kgq_uses_negation(int32_t s) { return plan_of(s) ? (plan_of(s)->negation ? 1 : 0) : -1; }
const char* kgq_structure_name(int32_t s) { return plan_of(s) ? kNames[s] : nullptr; }
int32_t kgq_structure_from_name(const char* n) {
  if (!n) return -1;
  for (int i = 0; i < KGQ_NUM_STRUCTURES; ++i)
    if (strcmp(n, kNames[i]) == 0) return i;
  return -1;
}
int32_t kgq_embedding_width(int32_t model, int32_t dim) {
  if (model == KGQ_GQE) return dim;
  if (model == KGQ_Q2B || model == KGQ_BETAE) return 2 * dim;
  return -1;
}

kgq_status kgq_shard_range(int64_t n, int32_t w, int32_t r, int64_t* b, int64_t* e) {
  if (n < 1 || w < 1 || r < 0 || r >= w || !b || !e) return KGQ_EINVAL;
  const int64_t per = (n + w - 1) / w;
  *b = std::min<int64_t>(n, (int64_t)r * per);
  *e = std::min<int64_t>(n, (int64_t)(r + 1) * per);
  return KGQ_OK;
}
int64_t kgq_shard_begin(const kgq_ctx* c) { return c ? c->e0 : -1; }
int64_t kgq_shard_end(const kgq_ctx* c) { return c ? c->e1 : -1; }

const char* kgq_last_error(const kgq_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

kgq_status kgq_create(const kgq_config* cfg, kgq_ctx** out) {
  if (!out) return fail(nullptr, KGQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, KGQ_EINVAL, "cfg is NULL");
  if (cfg->abi_version != KGQ_ABI_VERSION)
    return fail(nullptr, KGQ_EINVAL, "abi_version %u != %u", cfg->abi_version, KGQ_ABI_VERSION);
  if (cfg->model < KGQ_GQE || cfg->model > KGQ_BETAE) return fail(nullptr, KGQ_EINVAL, "bad model %d", cfg->model);
  if (cfg->n_entity < 1 || cfg->n_entity > INT32_MAX) return fail(nullptr, KGQ_EINVAL, "n_entity %lld", (long long)cfg->n_entity);
  if (cfg->n_relation < 1) return fail(nullptr, KGQ_EINVAL, "n_relation %d", cfg->n_relation);
  if (cfg->dim < 4 || cfg->dim % 4) return fail(nullptr, KGQ_EINVAL, "dim %d must be a positive multiple of 4", cfg->dim);
  if (cfg->model == KGQ_BETAE && (cfg->hidden < 1 || cfg->n_hidden_layers < 1 || cfg->n_hidden_layers > 8))
    return fail(nullptr, KGQ_EINVAL, "BetaE needs hidden >= 1 and 1 <= n_hidden_layers <= 8");
  if (cfg->terminal != KGQ_TERM_REGULARIZER && cfg->terminal != KGQ_TERM_SOFTMAX)
    return fail(nullptr, KGQ_EINVAL, "bad terminal %d", cfg->terminal);
  if (cfg->max_batch < 1) return fail(nullptr, KGQ_EINVAL, "max_batch %d", cfg->max_batch);
  if (cfg->max_k < 1 || cfg->max_k > kMaxK) return fail(nullptr, KGQ_EINVAL, "max_k %d outside [1, %d]", cfg->max_k, kMaxK);
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    return fail(nullptr, KGQ_EINVAL, "rank %d / world_size %d", cfg->rank, cfg->world_size);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
    return fail(nullptr, KGQ_ECUDA, "CUDA device %d not available (%d devices)", cfg->device, ndev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, cfg->device);
  if (prop.major != 10)
    return fail(nullptr, KGQ_EUNSUPPORTED, "libkgq is built for sm_100a (B200); device is sm_%d%d", prop.major, prop.minor);
  kgq_ctx* ctx = new kgq_ctx();
  ctx->cfg = *cfg;
  const char* ng = getenv("KGQ_NO_GRAPHS");
  ctx->use_graphs = !(ng && ng[0] && ng[0] != '0');
  ctx->fused_topk = fused_topk_disabled() ? KGQ_FUSED_OFF : KGQ_FUSED_AUTO;
  DeviceGuard g(cfg->device);
  kgq_shard_range(cfg->n_entity, cfg->world_size, cfg->rank, &ctx->e0, &ctx->e1);
  ctx->ns = ctx->e1 - ctx->e0;
  ctx->np = std::max<int64_t>(kEntityPad, round_up(ctx->ns, kEntityPad));
  ctx->ew = cfg->model == KGQ_BETAE ? 2 * cfg->dim : cfg->dim;
  ctx->qw = kgq_embedding_width(cfg->model, cfg->dim);
  ctx->ent_loaded.assign((size_t)cfg->n_entity, 0);
  kgq_status st = dalloc(ctx, &ctx->ent, (size_t)(cfg->n_entity * ctx->ew), "entity table");
  if (!st) st = dalloc(ctx, &ctx->d_err, 4, "error word");
  if (!st) st = dalloc(ctx, &ctx->d_invalid, (size_t)cfg->max_batch, "invalid flags");
  if (st) {
    g_create_err = ctx->err;
    kgq_destroy(ctx);
    return st;
  }
  cudaMemset(ctx->d_err, 0, 4 * sizeof(int32_t));
  cudaMemset(ctx->d_invalid, 0, cfg->max_batch * sizeof(int32_t));
  *out = ctx;
  return KGQ_OK;
}

void kgq_destroy(kgq_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->cfg.device);
  cudaDeviceSynchronize();
  auto F = [](void* p) { if (p) cudaFree(p); };
  F(ctx->ent); F(ctx->rel[0]); F(ctx->rel[1]); F(ctx->score_tab);
  for (auto& l : ctx->lin) { F(l.W); F(l.Wsp.b0); F(l.b); }
  for (Split* s : {&ctx->S, &ctx->Z, &ctx->H[0], &ctx->H[1], &ctx->I, &ctx->M}) F(s->b0);
  F(ctx->T); F(ctx->T2); F(ctx->Q); F(ctx->Qt); F(ctx->dist); F(ctx->cmin); F(ctx->cand); F(ctx->Hpre); F(ctx->d_err); F(ctx->d_invalid);
  F(ctx->topk_tmp_d); F(ctx->topk_tmp_i); F(ctx->uv.b0); F(ctx->Esum); F(ctx->uvT); F(ctx->lin1x.Wsp.b0); F(ctx->RW);
  F(ctx->mix_rid); F(ctx->mix_map);
  if (ctx->mix_map_host) cudaFreeHost(ctx->mix_map_host);
  if (ctx->mix_map_ev) cudaEventDestroy(ctx->mix_map_ev);
  for (auto& e : ctx->side_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->side_st) cudaStreamDestroy(ctx->side_st);
  F(ctx->uvsums); F(ctx->Atc.b0); F(ctx->Ptc); F(ctx->gws.ws); F(ctx->gws.cnt); F(ctx->gws2.ws); F(ctx->gws2.cnt);
  F(ctx->d_anchor_stage); F(ctx->d_rel_stage); F(ctx->d_topd_stage); F(ctx->d_topi_stage); F(ctx->d_epoch);
  if (ctx->comm) nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
  F(ctx->cm_d); F(ctx->cm_i); F(ctx->cg_d); F(ctx->cg_i); F(ctx->kt_buf);
  for (auto& gr : ctx->graphs) destroy_graph_entry(gr);
  clear_mix_graphs(ctx);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (auto& r : ctx->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  delete ctx;
}

kgq_status kgq_load_entities(kgq_ctx* ctx, const float* rows, int64_t first, int64_t n) {
  if (!ctx || !rows) return fail(ctx, KGQ_EINVAL, "NULL argument");
  if (ctx->finalized) return fail(ctx, KGQ_ESTATE, "tables are frozen after kgq_finalize()");
  if (first < 0 || n < 0 || first + n > ctx->cfg.n_entity)
    return fail(ctx, KGQ_EINVAL, "rows [%lld, %lld) outside [0, %lld)", (long long)first,
                (long long)(first + n), (long long)ctx->cfg.n_entity);
  DeviceGuard g(ctx->cfg.device);
  CK(cudaMemcpy(ctx->ent + first * ctx->ew, rows, (size_t)(n * ctx->ew) * sizeof(float),
                cudaMemcpyHostToDevice), "entity upload");
  for (int64_t i = first; i < first + n; ++i) {
    if (!ctx->ent_loaded[(size_t)i]) ctx->ent_rows_loaded++;
    ctx->ent_loaded[(size_t)i] = 1;
  }
  return KGQ_OK;
}

kgq_status kgq_load_relations(kgq_ctx* ctx, int32_t which, const float* rows, int32_t n) {
  if (!ctx || !rows) return fail(ctx, KGQ_EINVAL, "NULL argument");
  if (ctx->finalized) return fail(ctx, KGQ_ESTATE, "tables are frozen after kgq_finalize()");
  if (which != KGQ_REL_MAIN && which != KGQ_REL_OFFSET) return fail(ctx, KGQ_EINVAL, "bad relation table %d", which);
  if (which == KGQ_REL_OFFSET && ctx->cfg.model != KGQ_Q2B)
    return fail(ctx, KGQ_EINVAL, "relation offsets exist only for Q2B");
  if (n != ctx->cfg.n_relation) return fail(ctx, KGQ_EINVAL, "n %d != n_relation %d", n, ctx->cfg.n_relation);
  DeviceGuard g(ctx->cfg.device);
  const size_t bytes = (size_t)n * ctx->cfg.dim * sizeof(float);
  if (!ctx->rel[which]) {
    kgq_status st = dalloc(ctx, &ctx->rel[which], bytes / sizeof(float), "relation table");
    if (st) return st;
  }
  CK(cudaMemcpy(ctx->rel[which], rows, bytes, cudaMemcpyHostToDevice), "relation upload");
  return KGQ_OK;
}

kgq_status kgq_load_linear(kgq_ctx* ctx, int32_t id, const float* W, const float* b, int32_t out_f,
                           int32_t in_f) {
  if (!ctx || !W || !b) return fail(ctx, KGQ_EINVAL, "NULL argument");
  if (ctx->finalized) return fail(ctx, KGQ_ESTATE, "tables are frozen after kgq_finalize()");
  const int d = ctx->cfg.dim, H = ctx->cfg.hidden, m = ctx->cfg.model;
  int eo = -1, ei = -1;
  if (m == KGQ_BETAE && id == KGQ_LAYER_PROJ_OUT) { eo = 2 * d; ei = H; }
  else if (m == KGQ_BETAE && id >= KGQ_LAYER_PROJ_HIDDEN && id < KGQ_LAYER_PROJ_HIDDEN + ctx->cfg.n_hidden_layers) {
    eo = H; ei = id == KGQ_LAYER_PROJ_HIDDEN ? 3 * d : H;
  } else if (id == KGQ_LAYER_INTER_1) { eo = ei = (m == KGQ_BETAE ? 2 * d : d); }
  else if (id == KGQ_LAYER_INTER_2) { eo = d; ei = (m == KGQ_BETAE ? 2 * d : d); }
  else if (m == KGQ_Q2B && (id == KGQ_LAYER_OFFSET_1 || id == KGQ_LAYER_OFFSET_2)) { eo = ei = d; }
  if (eo < 0) return fail(ctx, KGQ_EINVAL, "layer id %d does not exist for this model", id);
  if (out_f != eo || in_f != ei)
    return fail(ctx, KGQ_EINVAL, "layer %d: shape [%d, %d], expected [%d, %d]", id, out_f, in_f, eo, ei);
  DeviceGuard g(ctx->cfg.device);
  Linear& L = ctx->lin[id];
  const size_t n = (size_t)out_f * in_f;
  kgq_status st = KGQ_OK;
  if (!L.W) {
    if (!st) st = dalloc(ctx, &L.W, n, "linear W");
    if (!st) st = alloc_split(ctx, &L.Wsp, out_f, in_f, "linear W (bf16x3)");
    if (!st) st = dalloc(ctx, &L.b, (size_t)out_f, "linear b");
    if (st) return st;
  }
  L.out_f = out_f;
  L.in_f = in_f;
  CK(cudaMemcpy(L.W, W, n * sizeof(float), cudaMemcpyHostToDevice), "linear W upload");
  CK(cudaMemcpy(L.b, b, (size_t)out_f * sizeof(float), cudaMemcpyHostToDevice), "linear b upload");
  launch_split_copy_rows(L.W, out_f, in_f, L.Wsp, 0);
  CK(cudaDeviceSynchronize(), "linear split");
  return KGQ_OK;
}

kgq_status kgq_finalize(kgq_ctx* ctx) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (ctx->finalized) return fail(ctx, KGQ_ESTATE, "already finalized");
  const kgq_config& c = ctx->cfg;
  const int d = c.dim;
  if (ctx->ent_rows_loaded != c.n_entity)
    return fail(ctx, KGQ_ESTATE, "entity table incomplete: %lld of %lld rows loaded",
                (long long)ctx->ent_rows_loaded, (long long)c.n_entity);
  if (!ctx->rel[0]) return fail(ctx, KGQ_ESTATE, "relation table not loaded");
  if (c.model == KGQ_Q2B && !ctx->rel[1]) return fail(ctx, KGQ_ESTATE, "Q2B relation offsets not loaded");
  std::vector<int> need = {KGQ_LAYER_INTER_1, KGQ_LAYER_INTER_2};
  if (c.model == KGQ_Q2B) { need.push_back(KGQ_LAYER_OFFSET_1); need.push_back(KGQ_LAYER_OFFSET_2); }
  if (c.model == KGQ_BETAE) {
    need.push_back(KGQ_LAYER_PROJ_OUT);
    for (int l = 0; l < c.n_hidden_layers; ++l) need.push_back(KGQ_LAYER_PROJ_HIDDEN + l);
  }
  for (int id : need)
    if (!ctx->lin[id].W) return fail(ctx, KGQ_ESTATE, "linear layer %d not loaded", id);
  DeviceGuard g(c.device);
  const int64_t Bm = c.max_batch;
  ctx->rows_max = (int64_t)kMaxBranches * Bm;
  ctx->tw = 2 * d;
  ctx->rpad = round_up(2 * Bm, kRowPad);
  const int nplanes = c.model == KGQ_GQE ? 1 : (c.model == KGQ_Q2B ? 2 : 3);
  // bytes for the distance scratch [bchunk, np] fp32: queries are scored in chunks of bchunk.
  // Every chunk re-reads the whole scoring table, so on large tables the chunk must hold enough
  // rows for the tensor-core scorer to stay compute-bound: at 2M entities a 4 GB scratch gave
  // 512-query chunks (2 M blocks per table tile: ~4.4 TB/s of table reads plus the 1.9 TB/s of
  // distance writes -- HBM-bound at 0.6 of the tensor peak).  Up to 16 GB, at most a quarter of
  // the free memory, at least 256 MB (KGQ_DIST_BUDGET_MB overrides: tests of the chunked path).
  int64_t budget = (int64_t)16 << 30;
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min<int64_t>(budget, (int64_t)(fr / 4));
    else cudaGetLastError();
    budget = std::max<int64_t>(budget, (int64_t)256 << 20);
    const char* e = getenv("KGQ_DIST_BUDGET_MB");
    if (e && atoll(e) > 0) budget = atoll(e) << 20;
  }
  ctx->bchunk = std::max<int64_t>(1, std::min<int64_t>(Bm, budget / (ctx->np * 4)));
  kgq_status st = KGQ_OK;
  const int iw = c.model == KGQ_BETAE ? 2 * d : d;
  // Q2B states hold [centre | offset] with the offset half at a 16-byte aligned column
  const int64_t sw = c.model == KGQ_Q2B ? q2b_off(d) + d : ctx->qw;
  if (!st) st = alloc_split(ctx, &ctx->S, ctx->rows_max, sw, "state S");
  if (!st) st = alloc_split(ctx, &ctx->I, ctx->rows_max, iw, "intersection hidden");
  if (!st) st = alloc_split(ctx, &ctx->M, Bm, ctx->qw, "combined state");
  if (!st && c.model == KGQ_BETAE) {
    st = alloc_split(ctx, &ctx->Z, ctx->rows_max, 3 * d, "MLP input");
    if (!st) st = alloc_split(ctx, &ctx->H[0], ctx->rows_max, c.hidden, "MLP hidden 0");
    if (!st) st = alloc_split(ctx, &ctx->H[1], ctx->rows_max, c.hidden, "MLP hidden 1");
  }
  if (!st) st = dalloc(ctx, &ctx->T, (size_t)(ctx->rows_max * ctx->tw), "T");
  if (!st) st = dalloc(ctx, &ctx->T2, (size_t)(ctx->rows_max * ctx->tw), "T2");
  if (!st) st = dalloc(ctx, &ctx->Q, (size_t)(Bm * 2 * ctx->qw), "Q");
  if (!st) st = dalloc(ctx, &ctx->Qt, (size_t)(nplanes * d * ctx->rpad), "Qt");
  if (!st) st = dalloc(ctx, &ctx->dist, (size_t)(ctx->bchunk * ctx->np), "dist");
  if (!st && c.model == KGQ_BETAE) st = dalloc(ctx, &ctx->cmin, (size_t)(ctx->bchunk * (ctx->np / 32)), "block minima");
  if (!st && c.model == KGQ_BETAE)
    st = dalloc(ctx, &ctx->cand, (size_t)ctx->bchunk * kFusedTopkLists * kFusedTopkMax, "fused top-k lists");
  if (!st) st = dalloc(ctx, &ctx->topk_tmp_d, (size_t)(ctx->bchunk * 4096), "top-k candidates");
  if (!st) st = dalloc(ctx, &ctx->topk_tmp_i, (size_t)(ctx->bchunk * 4096), "top-k candidates");
  if (!st && c.model == KGQ_BETAE) {
    st = alloc_split(ctx, &ctx->uv, ctx->np, 2 * d, "uv table");
    if (!st) st = dalloc(ctx, &ctx->Esum, (size_t)ctx->np, "entity sums");
    if (!st && !ctx->uvT) st = dalloc(ctx, &ctx->uvT, (size_t)2 * d * ctx->np, "uv table (dim-major)");
    if (!st) st = dalloc(ctx, &ctx->uvsums, (size_t)(2 * d + 2 * kLogTab), "uv sums + log table");
    if (!st) {  // ln c_i and 1 / c_i, c_i = 1 + i / kLogTab, after the sums (common.cuh log_tab)
      double tab[2 * kLogTab];
      for (int i = 0; i < kLogTab; ++i) {
        const double ci = 1.0 + (double)i / kLogTab;
        tab[i] = std::log(ci);
        tab[kLogTab + i] = 1.0 / ci;
      }
      CK(cudaMemcpy(ctx->uvsums + 2 * d, tab, sizeof tab, cudaMemcpyHostToDevice), "log table");
    }
    if (!st) st = alloc_split(ctx, &ctx->Atc, 2 * ctx->bchunk, 2 * d, "tc query rows");
    if (!st) st = dalloc(ctx, &ctx->Ptc, (size_t)(2 * ctx->bchunk), "tc query sums");
  }
  if (!st) st = dalloc(ctx, &ctx->gws.ws, kGemmWsFloats, "gemm split workspace");
  if (!st) st = dalloc(ctx, &ctx->gws.cnt, (size_t)kGemmCntInts, "gemm split counters");
  if (!st) CK(cudaMemset(ctx->gws.cnt, 0, kGemmCntInts * sizeof(int)), "gemm split counters");
  // the side stream's own split-K workspace (mixed path: two row halves' GEMMs run concurrently)
  if (!st) st = dalloc(ctx, &ctx->gws2.ws, kGemmWsFloats, "gemm split workspace (side)");
  if (!st) st = dalloc(ctx, &ctx->gws2.cnt, (size_t)kGemmCntInts, "gemm split counters (side)");
  if (!st) CK(cudaMemset(ctx->gws2.cnt, 0, kGemmCntInts * sizeof(int)), "gemm split counters (side)");
  if (!st) st = dalloc(ctx, &ctx->score_tab, (size_t)((c.model == KGQ_BETAE ? 3 : 1) * d * ctx->np), "score table");
  if (!st) st = dalloc(ctx, &ctx->d_anchor_stage, (size_t)(Bm * kMaxBranches), "staging");
  if (!st) st = dalloc(ctx, &ctx->d_rel_stage, (size_t)(Bm * kMaxBranches), "staging");
  if (!st) st = dalloc(ctx, &ctx->d_topd_stage, (size_t)(Bm * c.max_k), "staging");
  if (!st) st = dalloc(ctx, &ctx->d_topi_stage, (size_t)(Bm * c.max_k), "staging");
  if (st) return st;
  if (c.model == KGQ_BETAE && !relterm_disabled()) {
    // first projection layer with the relation input factored out (RelTerm, kgq_internal.cuh);
    // recomputed at every finalize (tables or weights may have been reloaded)
    const Linear& l1 = ctx->lin[KGQ_LAYER_PROJ_HIDDEN];
    if (!ctx->RW) {
      st = alloc_split(ctx, &ctx->lin1x.Wsp, l1.out_f, 2 * d, "layer-1 state weights");
      if (!st) st = dalloc(ctx, &ctx->RW, (size_t)c.n_relation * l1.out_f, "relation term");
      if (st) return st;
    }
    ctx->lin1x.b = l1.b;
    ctx->lin1x.out_f = l1.out_f;
    ctx->lin1x.in_f = 2 * d;
    launch_split_copy_rows(l1.W, l1.out_f, 2 * d, ctx->lin1x.Wsp, 0, l1.in_f);
    launch_relation_term(ctx->rel[0], c.n_relation, d, l1.W, l1.in_f, 2 * d, l1.out_f, ctx->RW, 0);
  }
  if (c.model == KGQ_BETAE) {
    launch_beta_regularize(ctx->ent, c.n_entity * ctx->ew, 0);
    launch_betae_entity_terms(ctx->ent, ctx->e0, ctx->ns, d, ctx->score_tab, ctx->np, 0);
    launch_betae_uv_table(ctx->ent, c.n_entity, ctx->e0, ctx->ns, ctx->np, d, ctx->uvsums, ctx->uv,
                          ctx->Esum, ctx->uvT, 0);
    // weights / entity terms converted so far must be in the operand format's range
    CK(cudaDeviceSynchronize(), "finalize");
    if (range_flags_taken())
      return fail(ctx, KGQ_ERANGE, "a weight (|w| >= 32) or BetaE entity term is outside the fp16x2 operand range; "
                  "use the bf16x3 build (libkgq_bf16x3.so, KGQ_OPERANDS=bf16x3)");
    if (ctx->RW && hpre_enabled() && (double)c.n_entity * ctx->lin1x.out_f * sizeof(float) <= kHpreBytesMax) {
      // hop-0 first layer per entity: Hpre = X W1[:, :2d]^T + b1 over the regularised table (the
      // same tensor-core GEMM as the layer itself, its bias folded in so the per-query gather adds
      // only RW[r]), through a temporary split copy of X.  An
      // entity row outside the fp16x2 range only disables the precompute (hop 0 then gathers and
      // multiplies per query, and flags such an anchor when a query uses it).
      const int H = ctx->lin1x.out_f;
      if (!ctx->Hpre) {
        kgq_status st2 = dalloc(ctx, &ctx->Hpre, (size_t)c.n_entity * H, "hop-0 layer-1 precompute");
        if (st2) return st2;
      }
      Split X;
      kgq_status st2 = alloc_split(ctx, &X, c.n_entity, 2 * d, "entity split (finalize)");
      if (st2) return st2;
      launch_split_copy_rows(ctx->ent, c.n_entity, 2 * d, X, 0, 2 * d, true);
      launch_linear(X, (int)c.n_entity, 2 * d, ctx->lin1x, kEpiNone, Split{}, ctx->Hpre, H, 0, 0, &ctx->gws, 0);
      CK(cudaDeviceSynchronize(), "hop-0 precompute");
      cudaFree(X.b0);
      if (range_flag_chain()) {  // the X split (the only conversion of this interval) overflowed
        cudaFree(ctx->Hpre);
        ctx->Hpre = nullptr;
      }
    }
  } else {
    launch_transpose_shard(ctx->ent, ctx->e0, ctx->ns, d, ctx->ew, ctx->score_tab, ctx->np, 0);
  }
  CK(cudaGetLastError(), "finalize launch");
  CK(cudaDeviceSynchronize(), "finalize");
  if (range_flags_taken())
    return fail(ctx, KGQ_ERANGE, "a weight (|w| >= 32) or BetaE entity term is outside the fp16x2 operand range; "
                "use the bf16x3 build (libkgq_bf16x3.so, KGQ_OPERANDS=bf16x3)");
  ctx->finalized = true;
  return KGQ_OK;
}

// Distances of query rows [b0, b0 + nb) (chain already run) to every entity of the shard,
// into ctx->dist rows [0, nb).  Returns the number of kernels launched.
// KGQ_BETAE_STREAM=cuv: the round-1 small-batch BetaE scorer on the C, U, V planes (A/B only)
static bool betae_stream_cuv() {
  static const bool v = [] {
    const char* e = getenv("KGQ_BETAE_STREAM");
    return e && e[0] == 'c';
  }();
  return v;
}

// fused_k > 0 (BetaE tensor-core path only): the scorer keeps per-stripe top-k lists in its
// epilogue (ctx->cand, *nlists per row) instead of writing ctx->dist.
static int score_rows(kgq_ctx* ctx, const Plan* P, int64_t b0, int nb, cudaStream_t st, int B = 0,
                      bool from_state = false, int fused_k = 0, int* nlists = nullptr) {
  const kgq_config& c = ctx->cfg;
  int L = 0;
  const float* qb = ctx->Q + b0 * P->n_out * ctx->qw;
  if (fused_k > 0) {
    StageTimer t(ctx, st, kStScore, 2.0 * nb * P->n_out * (double)ctx->ns * 2 * c.dim);
    if (from_state)
      L += launch_mix_score_prep(nullptr, ctx->S, nb * P->n_out, c.dim, ctx->uvsums, c.n_entity, ctx->Atc, ctx->Ptc,
                                 st, B, b0, P->n_out);
    else
      L += launch_score_prep_tc(qb, nb * P->n_out, c.dim, ctx->uvsums, c.n_entity, ctx->Atc, ctx->Ptc, st);
    L += launch_score_tc_topk(nb * P->n_out, P->n_out, c.dim, ctx->Atc, ctx->Ptc, ctx->uv, ctx->Esum, ctx->np, ctx->ns,
                              fused_k, ctx->cand, (int64_t)kFusedTopkLists * fused_k, &ctx->gws, st, nlists, topk_min_tiles(ctx));
    check_site("tensor-core scorer (fused top-k)");
  } else if (from_state) {  // BetaE, query state still in S (q_in_state): prep straight from the split rows
    StageTimer t(ctx, st, kStScore, 2.0 * nb * P->n_out * (double)ctx->ns * 2 * c.dim);
    L += launch_mix_score_prep(nullptr, ctx->S, nb * P->n_out, c.dim, ctx->uvsums, c.n_entity, ctx->Atc, ctx->Ptc,
                               st, B, b0, P->n_out);
    L += launch_score_tc_gemm(nb * P->n_out, P->n_out, c.dim, ctx->Atc, ctx->Ptc, ctx->uv, ctx->Esum, ctx->np,
                              ctx->dist, ctx->np, ctx->cmin, ctx->np / 32, ctx->ns, &ctx->gws, st);
    check_site("tensor-core scorer");
  } else if (c.model == KGQ_BETAE && !score_uses_stream(c.model, P->n_out, nb)) {
    // past the HBM ridge BetaE scoring is a dense contraction: tensor cores (score_tc.cu)
    StageTimer t(ctx, st, kStScore, 2.0 * nb * P->n_out * (double)ctx->ns * 2 * c.dim);
    L += launch_score_betae_tc(qb, nb * P->n_out, P->n_out, c.dim, ctx->uvsums, c.n_entity, ctx->Atc,
                               ctx->Ptc, ctx->uv, ctx->Esum, ctx->np, ctx->dist, ctx->np, ctx->cmin,
                               ctx->np / 32, ctx->ns, &ctx->gws, st);
    check_site("tensor-core scorer");
  } else if (c.model == KGQ_BETAE && !betae_stream_cuv()) {
    // HBM regime: stream the centred (u, v) table, 8 bytes per (entity, dim)
    {
      StageTimer t(ctx, st, kStPrep);
      L += launch_score_prep_tc(qb, nb * P->n_out, c.dim, ctx->uvsums, c.n_entity, ctx->Atc, ctx->Ptc, st);
    }
    StageTimer t(ctx, st, kStScore, 2.0 * nb * P->n_out * (double)ctx->ns * c.dim);
    L += launch_score_betae_stream(ctx->Atc, ctx->Ptc, ctx->uvT, ctx->Esum, ctx->np, c.dim, ctx->dist, ctx->np, nb,
                                   P->n_out, st);
  } else {
    {
      StageTimer t(ctx, st, kStPrep);
      L += launch_score_prep(c.model, qb, nb, P->n_out, c.dim, ctx->Qt, ctx->rpad, st);
    }
    StageTimer t(ctx, st, kStScore, (c.model == KGQ_GQE ? 2.0 : 4.0) * nb * P->n_out * (double)ctx->ns * c.dim);
    L += launch_score(c.model, P->n_out, nb, c.dim, c.cen, ctx->Qt, ctx->rpad, ctx->score_tab, ctx->np,
                      ctx->ns, ctx->dist, ctx->np, st);
  }
  return L;
}

static kgq_status submit_impl(kgq_ctx* ctx, int32_t s, int32_t B, const int32_t* anchors,
                              const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                              float* shard_dist, cudaStream_t st) {
  const Plan* P = plan_of(s);
  int L = 0;
  const bool push = ctx->peers.on() && ctx->push_row0 >= 0;  // N2: fused all-gather of the top-k
  CK(cudaMemsetAsync(ctx->d_invalid, 0, (size_t)B * sizeof(int32_t), st), "reset flags");
  const bool from_state = q_in_state(ctx, P, B);
  {
    StageTimer t(ctx, st, kStChain);
    L += run_chain(ctx, s, B, anchors, rels, st, !from_state);
  }
  check_site("operator chain");
  for (int64_t b0 = 0; b0 < B; b0 += ctx->bchunk) {
    const int nb = (int)std::min<int64_t>(ctx->bchunk, B - b0);
    const bool tc = ctx->cfg.model == KGQ_BETAE && !score_uses_stream(ctx->cfg.model, P->n_out, nb);
    // fused top-k in the tensor-core scorer's epilogue unless the distance rows are wanted
    const bool fused = tc && !shard_dist && use_fused_topk(ctx, (int64_t)nb * P->n_out, k);
    int nl = 0;
    L += score_rows(ctx, P, b0, nb, st, B, from_state, fused ? k : 0, &nl);
    {
      StageTimer t(ctx, st, kStTopk);
      // the tensor-core scorer's epilogue wrote 32-entity block minima: pruned top-k
      const bool blockmin = tc && k <= 32 && !topk_cmin_disabled();
      PeerPush pp{};
      if (push) {
        pp = ctx->peers;
        pp.row0 = ctx->push_row0 + (int)b0;
      }
      if (fused) {
        L += launch_topk_lists(ctx->cand, (int64_t)kFusedTopkLists * k, k, nb, nb, nl, nl, ctx->e0,
                               ctx->d_invalid + b0, nullptr, topk_dist + b0 * k, topk_id + b0 * k, st, pp);
      } else if (blockmin) {
        L += launch_topk_cmin(ctx->dist, ctx->np, ctx->cmin, ctx->np / 32, nb, ctx->ns, k, ctx->e0,
                              ctx->d_invalid + b0, topk_dist + b0 * k, topk_id + b0 * k, st, pp);
      } else {
        L += launch_topk(ctx->dist, ctx->np, nb, ctx->ns, k, ctx->e0, ctx->d_invalid + b0,
                         topk_dist + b0 * k, topk_id + b0 * k, ctx->topk_tmp_d, ctx->topk_tmp_i, st);
        if (push) L += launch_peer_push(pp, nb, k, topk_dist + b0 * k, topk_id + b0 * k, st);
      }
      check_site("top-k");
    }
    if (shard_dist)
      CK(cudaMemcpy2DAsync(shard_dist + b0 * ctx->ns, ctx->ns * sizeof(float), ctx->dist,
                           ctx->np * sizeof(float), ctx->ns * sizeof(float), nb, cudaMemcpyDeviceToDevice, st),
         "shard_dist copy");
  }
  {  // perf probe only: KGQ_DBG_EMPTY_NODES=n appends n empty dependent kernels (per-node cost)
    static const int n_empty = [] { const char* e = getenv("KGQ_DBG_EMPTY_NODES"); return e ? atoi(e) : 0; }();
    for (int i = 0; i < n_empty; ++i) L += launch_empty(st);
  }
  ctx->launches = L;
  CK(cudaGetLastError(), "submit launch");
  return KGQ_OK;
}

// Replays a captured CUDA graph of the whole submit (one cudaGraphLaunch instead of ~10-15
// kernel launches) when the same (structure, batch, k, buffers) was submitted before; the
// first call runs eagerly, the second captures.  With profiling on, the graph contains the
// stage events; each replay's times are harvested before the next replay or at profile_read.
static kgq_status submit_graphed(kgq_ctx* ctx, int32_t s, int32_t B, const int32_t* anchors,
                                 const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                                 cudaStream_t st) {
  const void* key[4] = {anchors, rels, topk_dist, topk_id};
  kgq_ctx::GraphEntry* e = nullptr;
  for (auto& g : ctx->graphs)
    if (g.s == s && g.B == B && g.k == k && g.prof == ctx->profile && std::equal(key, key + 4, g.ptr)) e = &g;
  ctx->graph_clock++;
  if (e && e->exec) {
    e->last = ctx->graph_clock;
    if (e->pending) harvest(ctx, e->evs, false);  // previous replay's stage times
    CK(cudaGraphLaunch(e->exec, st), "graph launch");
    e->pending = !e->evs.empty();
    ctx->launches = e->launches;
    return KGQ_OK;
  }
  if (!e) {
    if (ctx->graphs.size() >= 64) {  // evict the least recently used entry
      auto lru = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                  [](const kgq_ctx::GraphEntry& a, const kgq_ctx::GraphEntry& b) { return a.last < b.last; });
      if (lru->pending) harvest(ctx, lru->evs, false);
      destroy_graph_entry(*lru);
      ctx->graphs.erase(lru);
    }
    kgq_ctx::GraphEntry ne{s, B, k, ctx->profile, {key[0], key[1], key[2], key[3]}, nullptr, 0, 1,
                           ctx->graph_clock, {}, false};
    ctx->graphs.push_back(ne);
    return submit_impl(ctx, s, B, anchors, rels, k, topk_dist, topk_id, nullptr, st);
  }
  e->last = ctx->graph_clock;
  if (++e->seen < 2 || e->seen > 2) return submit_impl(ctx, s, B, anchors, rels, k, topk_dist, topk_id, nullptr, st);
  // capture on the context's private stream, then launch on the caller's
  if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking), "capture stream");
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  ctx->capture_entry = e;
  kgq_status r = submit_impl(ctx, s, B, anchors, rels, k, topk_dist, topk_id, nullptr, ctx->cap_stream);
  ctx->capture_entry = nullptr;
  cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
  if (r != KGQ_OK || ce != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    destroy_graph_entry(*e);
    e->seen = 3;  // never retry this key; run eagerly
    return submit_impl(ctx, s, B, anchors, rels, k, topk_dist, topk_id, nullptr, st);
  }
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) {
    cudaGetLastError();
    destroy_graph_entry(*e);
    e->seen = 3;
    return submit_impl(ctx, s, B, anchors, rels, k, topk_dist, topk_id, nullptr, st);
  }
  e->exec = exec;
  e->launches = ctx->launches;
  CK(cudaGraphLaunch(exec, st), "graph launch");
  e->pending = !e->evs.empty();
  return KGQ_OK;
}

// ---- N2 host-side pairing of pushes and merges (peer.cuh) ----
constexpr int64_t kPeerHdrBytes = 256;
static int64_t peer_flag_bytes(const kgq_ctx* ctx, int world) {  // header + flags, 256-byte aligned
  return kPeerHdrBytes + ((int64_t)2 * world * ctx->cfg.max_batch * (int64_t)sizeof(uint32_t) + 255) / 256 * 256;
}
// A pushing submit and its merge come in pairs (peer.cuh): reject a second push before the merge.
static kgq_status peer_push_check(kgq_ctx* ctx) {
  if (ctx->peers.on() && ctx->push_outstanding)
    return fail(ctx, KGQ_ESTATE, "peered context: the previous submit's top-k push has not been merged "
                                 "(call kgq_merge_peers after every submit)");
  return KGQ_OK;
}
static kgq_status peer_push_done(kgq_ctx* ctx, kgq_status st) {
  if (st == KGQ_OK && ctx->peers.on()) ctx->push_outstanding = true;
  return st;
}

// ---- multi-GPU data plane (kgq_comm_init): the context's NCCL communicator ------------------
static void query_range(int32_t B, int32_t W, int32_t r, int32_t* lo, int32_t* hi) {
  const int32_t c = (B + W - 1) / W;
  *lo = std::min<int64_t>(B, (int64_t)r * c);
  *hi = std::min<int64_t>(B, (int64_t)*lo + c);
}
static kgq_status nccl_fail(kgq_ctx* ctx, ncclResult_t r, const char* what) {
  return fail(ctx, KGQ_ENCCL, "%s: %s", what, nccl_api().GetErrorString(r));
}
// All-gather n floats + n ints per rank (this rank's cm_d / cm_i) into cg_d / cg_i [W * n], one
// NCCL group (one kernel) on the caller's stream.
static kgq_status comm_gather(kgq_ctx* ctx, size_t n, cudaStream_t cs) {
  const NcclApi& api = nccl_api();
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->comm);
  ncclResult_t r = api.GroupStart();
  if (r == ncclSuccess) r = api.AllGather(ctx->cm_d, ctx->cg_d, n, ncclFloat32, comm, cs);
  if (r == ncclSuccess) r = api.AllGather(ctx->cm_i, ctx->cg_i, n, ncclInt32, comm, cs);
  const ncclResult_t r2 = api.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllGather");
  if (r2 != ncclSuccess) return nccl_fail(ctx, r2, "ncclGroupEnd");
  return KGQ_OK;
}
// The local (one-shard, one-device) path: a captured graph when possible, else eager launches.
static kgq_status submit_local(kgq_ctx* ctx, int32_t s, int32_t B, const int32_t* anchors, const int32_t* rels,
                               int32_t k, float* td, int32_t* ti, float* sd, cudaStream_t cs) {
  if (ctx->use_graphs && !sd && B <= ctx->bchunk) return submit_graphed(ctx, s, B, anchors, rels, k, td, ti, cs);
  return submit_impl(ctx, s, B, anchors, rels, k, td, ti, sd, cs);
}
// A submit of the replicated batch through the communicator's data plane (kgq.h kgq_comm_init).
static kgq_status submit_comm(kgq_ctx* ctx, int32_t s, int32_t B, const int32_t* anchors, const int32_t* rels,
                              int32_t k, float* td, int32_t* ti, float* sd, cudaStream_t cs) {
  const int W = ctx->comm_world;
  if (ctx->comm_split == KGQ_SPLIT_ENTITIES) {  // local top-k -> all-gather -> merge (a9)
    kgq_status st = submit_local(ctx, s, B, anchors, rels, k, ctx->cm_d, ctx->cm_i, sd, cs);
    if (st) return st;
    int L = ctx->launches;
    if ((st = comm_gather(ctx, (size_t)B * k, cs))) return st;
    L += launch_merge(W, B, k, ctx->cg_d, ctx->cg_i, td, ti, cs);
    ctx->launches = L;
    CK(cudaGetLastError(), "merge launch");
    return KGQ_OK;
  }
  if (sd) return fail(ctx, KGQ_EINVAL, "shard_dist is not available in query-split mode");
  const Plan* P = plan_of(s);
  int32_t lo, hi;
  query_range(B, W, ctx->comm_rank, &lo, &hi);
  const int32_t c = (B + W - 1) / W;
  ctx->launches = 0;
  if (hi > lo) {
    kgq_status st = submit_local(ctx, s, hi - lo, anchors + (int64_t)lo * P->n_anchor,
                                 rels + (int64_t)lo * P->n_rel, k, ctx->cm_d, ctx->cm_i, nullptr, cs);
    if (st) return st;
  }
  kgq_status st = comm_gather(ctx, (size_t)c * k, cs);  // rank r's rows land at [r c, r c + c)
  if (st) return st;
  CK(cudaMemcpyAsync(td, ctx->cg_d, (size_t)B * k * sizeof(float), cudaMemcpyDeviceToDevice, cs), "gather copy");
  CK(cudaMemcpyAsync(ti, ctx->cg_i, (size_t)B * k * sizeof(int32_t), cudaMemcpyDeviceToDevice, cs), "gather copy");
  return KGQ_OK;
}
static kgq_status submit_dev(kgq_ctx* ctx, int32_t s, int32_t B, const int32_t* anchors, const int32_t* rels,
                             int32_t k, float* td, int32_t* ti, float* sd, cudaStream_t cs) {
  return ctx->comm ? submit_comm(ctx, s, B, anchors, rels, k, td, ti, sd, cs)
                   : submit_local(ctx, s, B, anchors, rels, k, td, ti, sd, cs);
}

kgq_status kgq_submit(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors, const int32_t* rels,
                      int32_t k, float* topk_dist, int32_t* topk_id, float* shard_dist, kgq_stream stream) {
  kgq_status st = check_submit(ctx, s, batch, k, true);
  if (st) return st;
  if (batch == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !topk_dist || !topk_id) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  if ((st = peer_push_check(ctx))) return st;
  DeviceGuard g(ctx->cfg.device);
  ctx->push_row0 = ctx->peers.on() ? 0 : -1;
  return peer_push_done(ctx, submit_dev(ctx, s, batch, anchors, rels, k, topk_dist, topk_id, shard_dist,
                                        (cudaStream_t)stream));
}

// ---- mixed-structure batches ---------------------------------------------
// Several (structure, batch) groups in one call.  BetaE runs level-synchronously: every
// projection hop of every group's branches (and then every post-intersection hop) is ONE MLP
// over all their rows, the intersections of all groups are one pair of attention GEMMs, and the
// scorer and the top-k run once over all queries -- the dense layers see M = sum of the groups'
// branch rows instead of one structure's.  GQE / Q2B (cheap translation chains) submit group by
// group.  Rows of S: intersection groups' branch blocks first (contiguous attention input),
// then the others; hop batches are gathered into Z, run through the MLP into I and scattered
// back; final query embeddings stay in S (branch 0 block, union: blocks 0 and 1).
namespace {
struct MixGroup {
  int s, B, q0;
  const Plan* P;
  const int32_t* anchors;
  const int32_t* rels;
  int nb, maxh;
  int nproj[kMaxBranches];
  int proj[kMaxBranches][kMaxOps];
  bool neg_after[kMaxBranches][kMaxOps];
  int64_t srow[kMaxBranches];
};
}  // namespace

// The projection MLP (Eq. 4) over rows [r0, r0 + M) of a hop batch already gathered into Z
// (relation ids in mix_rid); rows >= neg0 (batch-relative) are negated.  On `st` with split-K
// workspace / span group `ws`.
// rm (optional, regulariser terminal): the last layer writes its rows straight into S through
// this remap (batch row -> S row) instead of into I (then no scatter is needed).
static int mlp_rows(kgq_ctx* ctx, int r0, int M, int neg0, cudaStream_t st, const GemmWs* ws, bool l1_done,
                    const RowMap* rm = nullptr) {
  const int d = ctx->cfg.dim;
  int L = 0;
  RelTerm rt;
  rt.RW = ctx->RW;
  rt.ldrw = ctx->cfg.hidden;
  rt.M = M;
  rt.rid = ctx->mix_rid + r0;
  if (!l1_done) {  // else H0 rows came from the per-entity precompute (hop 0)
    StageTimer t(ctx, st, kStDense, 2.0 * M * (double)ctx->lin1x.out_f * 2 * d);
    L += launch_linear_rel(ctx->Z.at(r0), M, 2 * d, ctx->lin1x, rt, ctx->H[0].at(r0), ws, st);
  }
  Split A = ctx->H[0].at(r0);
  int K = ctx->lin1x.out_f;
  for (int l = 1; l < ctx->cfg.n_hidden_layers; ++l) {
    const Linear& lin = ctx->lin[KGQ_LAYER_PROJ_HIDDEN + l];
    L += dense(ctx, A, M, K, lin, kEpiRelu, ctx->H[l & 1].at(r0), 0, 0, st, ws);
    A = ctx->H[l & 1].at(r0);
    K = lin.out_f;
  }
  const Linear& lo = ctx->lin[KGQ_LAYER_PROJ_OUT];
  const int ng = std::max(0, std::min(neg0 - r0, M));  // negated rows of this range: [ng, M)
  if (ctx->cfg.terminal == KGQ_TERM_SOFTMAX) {
    float* T = ctx->T + (int64_t)r0 * 2 * d;
    L += dense(ctx, A, M, K, lo, kEpiNone, T, 2 * d, st);
    L += launch_softmax_terminal(T, 2 * d, M, 2 * d, ctx->I.at(r0), 0, ng, M, st);
  } else if (rm) {
    RowMap h = *rm;  // this range's rows are batch rows r0 + i: shift the segment starts by r0
    for (int i = 0; i < h.n; ++i) h.dst0[i] -= r0;
    StageTimer t(ctx, st, kStDense, 2.0 * M * (double)lo.out_f * K);
    L += launch_linear_map(A, M, K, lo, kEpiBetaReg, ctx->S, ctx->rows_max, h, ng, M, ws, st);
    check_site("dense layer (remapped into S)");
  } else {
    L += dense(ctx, A, M, K, lo, kEpiBetaReg, ctx->I.at(r0), ng, M, st, ws);
  }
  return L;
}

// KGQ_NO_REMAP=1: the last MLP layer writes the scratch I and a scatter kernel moves its rows to S
static bool remap_enabled() {
  static const bool v = [] {
    const char* e = getenv("KGQ_NO_REMAP");
    return !(e && e[0] && e[0] != '0');
  }();
  return v;
}

// KGQ_NO_SPLIT_MLP=1: every hop MLP as one chain of launches on the context's stream
static bool split_mlp_enabled() {
  static const bool v = [] {
    const char* e = getenv("KGQ_NO_SPLIT_MLP");
    return !(e && e[0] && e[0] != '0');
  }();
  return v;
}
// rows from which a batched MLP / attention pair runs as two row halves on two streams
// (KGQ_SPLIT_MLP_ROWS: tuning experiments only)
static int split_mlp_rows() {
  static const int v = env_int("KGQ_SPLIT_MLP_ROWS", 8192);
  return v;
}
static bool side_stream(kgq_ctx* ctx) {  // lazily created; false if CUDA refuses
  if (ctx->side_st && ctx->side_ev[0] && ctx->side_ev[1]) return true;
  if (!ctx->side_st && cudaStreamCreateWithFlags(&ctx->side_st, cudaStreamNonBlocking) != cudaSuccess) {
    ctx->side_st = nullptr;
    cudaGetLastError();
    return false;
  }
  for (auto& e : ctx->side_ev)
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      e = nullptr;
      cudaGetLastError();
      return false;
    }
  return true;
}

// one MLP over a hop batch (segments already describe the batch rows); negated rows are last.
// Large batches (>= 8,192 rows) run as two row halves on two streams (the context's and its
// side stream, each with its own split-K workspace): both halves' GEMMs want the whole GPU, so
// each launch's last, partly filled round of tiles overlaps the other half's tiles instead of
// leaving SMs idle (the per-launch tail), and PDL / graph ordering stays per stream.
static int mix_mlp(kgq_ctx* ctx, const MixSegs& sg, int M, int neg0, cudaStream_t st) {
  const int d = ctx->cfg.dim;
  int L = 0;
  // hop 0 (every row anchor-sourced) with the per-entity precompute: the first layer is a gather
  bool pre = ctx->Hpre != nullptr;
  for (int i = 0; i < sg.n && pre; ++i) pre = sg.s[i].kind == 0;
  if (pre)
    L += launch_mix_h0_pre(sg, M, ctx->Hpre, ctx->RW, ctx->lin1x.out_f, ctx->H[0], ctx->cfg.n_entity,
                           ctx->cfg.n_relation, ctx->d_err, ctx->d_invalid, st);
  else
    L += launch_mix_gather(sg, M, ctx->ent, ctx->S, ctx->M, ctx->Z, ctx->mix_rid, d, ctx->cfg.n_entity,
                           ctx->cfg.n_relation, ctx->d_err, ctx->d_invalid, st);
  // the last layer writes S directly when every segment is whole 32-row boxes (B % 32 == 0 for
  // every group: the TMA store boxes of the epilogue never straddle two segments)
  RowMap rm;
  bool remap = ctx->cfg.terminal == KGQ_TERM_REGULARIZER && sg.n <= kMaxRowMap && remap_enabled();
  for (int i = 0; i < sg.n && remap; ++i) {
    remap = sg.s[i].dst0 % 32 == 0 && sg.s[i].B % 32 == 0;
    rm.dst0[i] = sg.s[i].dst0;
    rm.src0[i] = (int)sg.s[i].src0;
  }
  rm.n = remap ? sg.n : 0;
  const RowMap* rmp = remap ? &rm : nullptr;
  const int half = ((M / 2 + 255) / 256) * 256;  // 256-row (one tile pair) aligned cut
  // (a failing fork / join call leaves its error for the submit's final cudaGetLastError check)
  if (M >= split_mlp_rows() && split_mlp_enabled() && side_stream(ctx) && cudaEventRecord(ctx->side_ev[0], st) == cudaSuccess &&
      cudaStreamWaitEvent(ctx->side_st, ctx->side_ev[0], 0) == cudaSuccess) {
    L += mlp_rows(ctx, 0, half, neg0, st, &ctx->gws, pre, rmp);
    L += mlp_rows(ctx, half, M - half, neg0, ctx->side_st, &ctx->gws2, pre, rmp);
    cudaEventRecord(ctx->side_ev[1], ctx->side_st);
    cudaStreamWaitEvent(st, ctx->side_ev[1], 0);
  } else {
    L += mlp_rows(ctx, 0, M, neg0, st, &ctx->gws, pre, rmp);
  }
  if (!remap) L += launch_mix_scatter(sg, M, ctx->I, ctx->S, 2 * d, st);
  check_site("mixed hop");
  return L;
}

static kgq_status mixed_betae(kgq_ctx* ctx, std::vector<MixGroup>& G, int Q, int32_t k, float* topk_dist,
                              int32_t* topk_id, cudaStream_t st, int64_t* own_map = nullptr) {
  const int d = ctx->cfg.dim;
  int L = 0;
  CK(cudaMemsetAsync(ctx->d_invalid, 0, (size_t)Q * sizeof(int32_t), st), "reset flags");
  // S layout: intersection groups first
  int64_t cur = 0, inter_rows = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (auto& g : G)
      if ((g.P->kind == kInter) == (pass == 0))
        for (int br = 0; br < g.nb; ++br) {
          g.srow[br] = cur;
          cur += g.B;
          if (pass == 0) inter_rows += g.B;
        }
  {
    StageTimer t(ctx, st, kStChain);
    // ---- projection hops, level by level ----
    // Hops of the intersection groups' branches run first (levels [0, H1)), then the attention
    // pair and the combine; every later level batches the remaining branch hops (e.g. 3p's third)
    // TOGETHER with the post-intersection hops of the same depth (ip / inp / up-DM) into one MLP
    // -- the projection weights are shared, so the two small batches (1K + 2K rows at C2) become
    // one launch chain of 3K rows (fewer one-wave launches, one gather / scatter pair).
    int maxh = 0, H1 = 0, maxpost = 0;
    for (auto& g : G) {
      maxh = std::max(maxh, g.maxh);
      if (g.P->kind == kInter) {
        H1 = std::max(H1, g.maxh);
        maxpost = std::max(maxpost, g.P->npost);
      }
    }
    // level h of the branch chains (groups with a branch longer than h) plus, post >= 0, the
    // post-intersection hop `post` of every intersection group that has one; negated rows last
    auto hop = [&](int h, int post) -> kgq_status {
      MixSegs sg;
      int M = 0, neg0 = 0;
      for (int negpass = 0; negpass < 2; ++negpass) {
        if (negpass == 1) neg0 = M;
        for (auto& g : G)
          for (int br = 0; br < g.nb; ++br) {
            if (g.nproj[br] <= h || g.neg_after[br][h] != (negpass == 1)) continue;
            if (sg.n == kMaxMixSegs) return fail(ctx, KGQ_EINVAL, "mixed submit: too many groups");
            MixSeg& m = sg.s[sg.n++];
            m.dst0 = M; m.B = g.B; m.q0 = g.q0;
            m.kind = h == 0 ? 0 : 1;
            m.src0 = g.srow[br];  // gather source = scatter target: the branch's S rows
            m.anchors = g.anchors; m.n_a = g.P->n_anchor; m.aslot = g.P->br[br].anchor;
            m.rels = g.rels; m.n_r = g.P->n_rel; m.rslot = g.proj[br][h];
            M += g.B;
          }
        if (negpass == 0 && post >= 0)  // post-intersection hops are never negated
          for (auto& g : G) {
            if (g.P->kind != kInter || g.P->npost <= post) continue;
            if (sg.n == kMaxMixSegs) return fail(ctx, KGQ_EINVAL, "mixed submit: too many groups");
            MixSeg& m = sg.s[sg.n++];
            m.dst0 = M; m.B = g.B; m.q0 = g.q0;
            m.kind = post == 0 ? 2 : 1;  // 2: the combine's output rows (M at q0); 1: S rows
            m.src0 = g.srow[0];          // the group's branch-0 block holds the embedding
            m.anchors = g.anchors; m.n_a = g.P->n_anchor; m.aslot = 0;
            m.rels = g.rels; m.n_r = g.P->n_rel; m.rslot = g.P->post[post];
            M += g.B;
          }
      }
      if (M > 0) L += mix_mlp(ctx, sg, M, neg0, st);
      return KGQ_OK;
    };
    for (int h = 0; h < H1; ++h) {
      const kgq_status hs = hop(h, -1);
      if (hs != KGQ_OK) return hs;
    }
    // ---- intersections: one attention GEMM pair over every intersection group's branch rows ----
    if (inter_rows > 0) {
      // the attention GEMM pair over rows [r0, r0 + m); >= 8,192 rows: two halves on two streams
      // (as mix_mlp)
      auto attn = [&](int r0, int m, cudaStream_t s2, const GemmWs* w) {
        L += dense(ctx, ctx->S.at(r0), m, 2 * d, ctx->lin[KGQ_LAYER_INTER_1], kEpiRelu, ctx->I.at(r0), 0, 0, s2, w);
        L += dense(ctx, ctx->I.at(r0), m, 2 * d, ctx->lin[KGQ_LAYER_INTER_2], kEpiNone, ctx->T + (int64_t)r0 * ctx->tw,
                   ctx->tw, s2, w);
      };
      const int ir = (int)inter_rows, ih = ((ir / 2 + 255) / 256) * 256;
      if (ir >= split_mlp_rows() && split_mlp_enabled() && side_stream(ctx) &&
          cudaEventRecord(ctx->side_ev[0], st) == cudaSuccess &&
          cudaStreamWaitEvent(ctx->side_st, ctx->side_ev[0], 0) == cudaSuccess) {
        attn(0, ih, st, &ctx->gws);
        attn(ih, ir - ih, ctx->side_st, &ctx->gws2);
        cudaEventRecord(ctx->side_ev[1], ctx->side_st);
        cudaStreamWaitEvent(st, ctx->side_ev[1], 0);
      } else {
        attn(0, ir, st, &ctx->gws);
      }
      MixCombine mc;
      int total = 0;
      for (auto& g : G) {
        if (g.P->kind != kInter) continue;
        MixCombine::Group& mg = mc.g[mc.n++];
        CombineArgs& c = mg.c;
        c = CombineArgs{};
        c.model = KGQ_BETAE; c.nb = g.nb; c.B = g.B; c.d = d; c.ldl = ctx->tw; c.ldg = 0;
        c.rels = g.rels; c.n_r = g.P->n_rel; c.n_relation = ctx->cfg.n_relation; c.post_slot = -1;
        c.negate_out = g.P->neg_inter ? 1 : 0;
        c.err = ctx->d_err; c.invalid = ctx->d_invalid + g.q0;
        mg.q_begin = total;
        mg.q0 = g.q0;
        mg.srow0 = g.srow[0];
        mg.to_m = g.P->npost ? 1 : 0;
        total += g.B;
      }
      L += launch_mix_combine(mc, total, ctx->S, ctx->T, ctx->tw, ctx->M, st);
    }
    // ---- the remaining branch hops and the post-intersection hops, one MLP per depth ----
    const int late = std::max(maxh - H1, maxpost);
    for (int lv = 0; lv < late; ++lv) {
      const kgq_status hs = hop(H1 + lv, lv < maxpost ? lv : -1);
      if (hs != KGQ_OK) return hs;
    }
  }
  // ---- score rows: single-embedding groups first (query order), then the DNF-union groups
  // (rows 2b + branch); out_row maps every dist row back to its global query index ----
  int R1 = 0, R2 = 0;
  for (auto& g : G) (g.P->n_out == 1 ? R1 : R2) += g.B * g.P->n_out;
  const int Q1 = R1, Q2 = R2 / 2;
  // the shared pinned staging buffer is rewritten only after its previous upload finished; a
  // graph capture writes its own pinned copy instead (the graph's memcpy node reads it at replay)
  if (!own_map && ctx->mix_map_ev) CK(cudaEventSynchronize(ctx->mix_map_ev), "mixed staging");
  int64_t* const map_host = own_map ? own_map : ctx->mix_map_host;
  int64_t* srcrow = map_host;
  int64_t* outrow = map_host + (R1 + R2);  // stored as int64 pairs of int32 below
  int32_t* outrow32 = reinterpret_cast<int32_t*>(outrow);
  {
    int r = 0, o = 0;
    for (auto& g : G)
      if (g.P->n_out == 1)
        for (int b = 0; b < g.B; ++b) {
          srcrow[r++] = g.srow[0] + b;
          outrow32[o++] = g.q0 + b;
        }
    for (auto& g : G)
      if (g.P->n_out == 2)
        for (int b = 0; b < g.B; ++b) {
          srcrow[r++] = g.srow[0] + b;
          srcrow[r++] = g.srow[1] + b;
          outrow32[o++] = g.q0 + b;
        }
  }
  const size_t map_bytes = (size_t)(R1 + R2) * sizeof(int64_t) + (size_t)(Q1 + Q2) * sizeof(int32_t);
  CK(cudaMemcpyAsync(ctx->mix_map, map_host, map_bytes, cudaMemcpyHostToDevice, st), "mixed map upload");
  if (!own_map) CK(cudaEventRecord(ctx->mix_map_ev, st), "mixed staging");
  const int64_t* d_srcrow = ctx->mix_map;
  const int32_t* d_outrow = reinterpret_cast<const int32_t*>(ctx->mix_map + (R1 + R2));
  // fused top-k (k <= 16, use_fused_topk): the scorer epilogue keeps per-stripe lists and no
  // distance block is written -- decided per scorer launch (single-branch rows, then union rows)
  const bool f1 = use_fused_topk(ctx, R1, k), f2 = use_fused_topk(ctx, R2, k);
  const int64_t ldc = (int64_t)kFusedTopkLists * k;
  int nl1 = 0, nl2 = 0;
  {
    StageTimer t(ctx, st, kStScore, 2.0 * (R1 + R2) * (double)ctx->ns * 2 * d);
    L += launch_mix_score_prep(d_srcrow, ctx->S, R1 + R2, d, ctx->uvsums, ctx->cfg.n_entity, ctx->Atc, ctx->Ptc, st);
    if (f1)
      L += launch_score_tc_topk(R1, 1, d, ctx->Atc, ctx->Ptc, ctx->uv, ctx->Esum, ctx->np, ctx->ns, k, ctx->cand, ldc,
                                &ctx->gws, st, &nl1, topk_min_tiles(ctx));
    else
      L += launch_score_tc_gemm(R1, 1, d, ctx->Atc, ctx->Ptc, ctx->uv, ctx->Esum, ctx->np, ctx->dist, ctx->np,
                                ctx->cmin, ctx->np / 32, ctx->ns, &ctx->gws, st);
    if (f2)
      L += launch_score_tc_topk(R2, 2, d, ctx->Atc.at(R1), ctx->Ptc + R1, ctx->uv, ctx->Esum, ctx->np, ctx->ns, k,
                                ctx->cand + (int64_t)Q1 * ldc, ldc, &ctx->gws, st, &nl2, topk_min_tiles(ctx));
    else
      L += launch_score_tc_gemm(R2, 2, d, ctx->Atc.at(R1), ctx->Ptc + R1, ctx->uv, ctx->Esum, ctx->np,
                                ctx->dist + (int64_t)Q1 * ctx->np, ctx->np, ctx->cmin + (int64_t)Q1 * (ctx->np / 32),
                                ctx->np / 32, ctx->ns, &ctx->gws, st);
    check_site("mixed scorer");
  }
  {
    StageTimer t(ctx, st, kStTopk);
    PeerPush pp{};
    if (ctx->peers.on()) pp = ctx->peers;  // N2: rows pushed by output row (row0 = 0)
    // score rows [0, Q1): single-branch groups, [Q1, Q1 + Q2): union groups; out_row maps both
    if (f1 && f2) {
      L += launch_topk_lists(ctx->cand, ldc, k, Q1 + Q2, Q1, nl1, nl2, ctx->e0, ctx->d_invalid, d_outrow, topk_dist,
                             topk_id, st, pp);
    } else if (!f1 && !f2) {
      L += launch_topk_cmin_map(ctx->dist, ctx->np, ctx->cmin, ctx->np / 32, Q1 + Q2, ctx->ns, k, ctx->e0,
                                ctx->d_invalid, d_outrow, topk_dist, topk_id, st, pp);
    } else {
      for (int part = 0; part < 2; ++part) {
        const int r0 = part ? Q1 : 0, nr = part ? Q2 : Q1;
        if (nr == 0) continue;
        if (part ? f2 : f1)
          L += launch_topk_lists(ctx->cand + (int64_t)r0 * ldc, ldc, k, nr, nr, part ? nl2 : nl1, part ? nl2 : nl1,
                                 ctx->e0, ctx->d_invalid, d_outrow + r0, topk_dist, topk_id, st, pp);
        else
          L += launch_topk_cmin_map(ctx->dist + (int64_t)r0 * ctx->np, ctx->np, ctx->cmin + (int64_t)r0 * (ctx->np / 32),
                                    ctx->np / 32, nr, ctx->ns, k, ctx->e0, ctx->d_invalid, d_outrow + r0, topk_dist,
                                    topk_id, st, pp);
      }
    }
    check_site("mixed top-k");
  }
  ctx->launches = L;
  CK(cudaGetLastError(), "mixed submit launch");
  return KGQ_OK;
}

static kgq_status submit_mixed_impl(kgq_ctx* ctx, int32_t n_groups, const int32_t* structures,
                                    const int32_t* batches, const int32_t* anchors, const int32_t* rels, int32_t k,
                                    float* topk_dist, int32_t* topk_id, kgq_stream stream) {
  if (n_groups < 0 || (n_groups > 0 && (!structures || !batches)))
    return fail(ctx, KGQ_EINVAL, "mixed submit: bad group arrays");
  int64_t Q = 0;
  for (int i = 0; i < n_groups; ++i) {
    kgq_status st = check_submit(ctx, structures[i], batches[i], k, true);
    if (st) return st;
    Q += batches[i];
  }
  if (Q > ctx->cfg.max_batch)
    return fail(ctx, KGQ_EINVAL, "mixed submit: %lld queries > max_batch %d", (long long)Q, ctx->cfg.max_batch);
  if (Q == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !topk_dist || !topk_id) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  DeviceGuard dg(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  std::vector<MixGroup> G;
  int64_t ao = 0, ro = 0, q0 = 0;
  for (int i = 0; i < n_groups; ++i) {
    MixGroup g{};
    g.s = structures[i];
    g.B = batches[i];
    g.q0 = (int)q0;
    g.P = plan_of(g.s);
    g.anchors = anchors + ao;
    g.rels = rels + ro;
    ao += (int64_t)g.B * g.P->n_anchor;
    ro += (int64_t)g.B * g.P->n_rel;
    q0 += g.B;
    g.nb = g.P->nbranch;
    for (int br = 0; br < g.nb; ++br) {
      g.nproj[br] = 0;
      for (int o = 0; o < g.P->br[br].nops; ++o) {
        const int op = g.P->br[br].ops[o];
        if (op == kOpNeg) {
          g.neg_after[br][g.nproj[br] - 1] = true;
        } else {
          g.proj[br][g.nproj[br]] = op;
          g.neg_after[br][g.nproj[br]] = false;
          g.nproj[br]++;
        }
      }
      g.maxh = std::max(g.maxh, g.nproj[br]);
    }
    if (g.B > 0) G.push_back(g);
  }
  const bool batched = ctx->cfg.model == KGQ_BETAE && ctx->RW && k <= 32 && Q <= ctx->bchunk &&
                       !score_uses_stream(KGQ_BETAE, 1, (int)Q) && (int)G.size() * kMaxBranches <= kMaxMixSegs;
  if (!batched) {  // group by group through the single-structure path (one epoch: rows by q0)
    int L = 0;
    for (auto& g : G) {
      ctx->push_row0 = ctx->peers.on() ? g.q0 : -1;
      kgq_status st = submit_impl(ctx, g.s, g.B, g.anchors, g.rels, k, topk_dist + (int64_t)g.q0 * k,
                                  topk_id + (int64_t)g.q0 * k, nullptr, cs);
      if (st) return st;
      L += ctx->launches;
    }
    ctx->launches = L;
    return KGQ_OK;
  }
  if (!ctx->mix_rid) {
    kgq_status st = dalloc(ctx, &ctx->mix_rid, (size_t)ctx->rows_max, "mixed relation ids");
    if (!st) st = dalloc(ctx, &ctx->mix_map, (size_t)(3 * ctx->cfg.max_batch), "mixed row map");
    if (st) return st;
    CK(cudaMallocHost((void**)&ctx->mix_map_host, (size_t)(3 * ctx->cfg.max_batch) * sizeof(int64_t)), "mixed staging");
    CK(cudaEventCreateWithFlags(&ctx->mix_map_ev, cudaEventDisableTiming), "mixed staging");
  }
  if (!ctx->use_graphs || ctx->profile) return mixed_betae(ctx, G, (int)Q, k, topk_dist, topk_id, cs);
  // ---- graph replay of identical batched mixed submits (first call eager, second captures) ----
  std::vector<int32_t> key;
  for (int i = 0; i < n_groups; ++i) {
    key.push_back(structures[i]);
    key.push_back(batches[i]);
  }
  const void* ptrs[4] = {anchors, rels, topk_dist, topk_id};
  kgq_ctx::MixGraphEntry* e = nullptr;
  for (auto& m : ctx->mgraphs)
    if (m.k == k && m.key == key && std::equal(ptrs, ptrs + 4, m.ptr)) e = &m;
  if (e && e->exec) {
    CK(cudaGraphLaunch(e->exec, cs), "mixed graph launch");
    ctx->launches = e->launches;
    return KGQ_OK;
  }
  if (!e) {
    if (ctx->mgraphs.size() >= 16) clear_mix_graphs(ctx);
    ctx->mgraphs.push_back(kgq_ctx::MixGraphEntry{key, {ptrs[0], ptrs[1], ptrs[2], ptrs[3]}, k, nullptr, 0, 1, nullptr});
    return mixed_betae(ctx, G, (int)Q, k, topk_dist, topk_id, cs);
  }
  if (e->seen != 1) return mixed_betae(ctx, G, (int)Q, k, topk_dist, topk_id, cs);  // capture failed before
  e->seen = 2;
  CK(cudaMallocHost((void**)&e->map_host, (size_t)(3 * ctx->cfg.max_batch) * sizeof(int64_t)), "mixed graph map");
  if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking), "capture stream");
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  kgq_status r = mixed_betae(ctx, G, (int)Q, k, topk_dist, topk_id, ctx->cap_stream, e->map_host);
  cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (r == KGQ_OK && ce == cudaSuccess && graph) ce = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (r != KGQ_OK || ce != cudaSuccess || !exec) {
    cudaGetLastError();
    e->seen = 3;  // never retry this key; run eagerly
    return mixed_betae(ctx, G, (int)Q, k, topk_dist, topk_id, cs);
  }
  e->exec = exec;
  e->launches = ctx->launches;
  CK(cudaGraphLaunch(exec, cs), "mixed graph launch");
  return KGQ_OK;
}

kgq_status kgq_submit_mixed(kgq_ctx* ctx, int32_t n_groups, const int32_t* structures, const int32_t* batches,
                            const int32_t* anchors, const int32_t* rels, int32_t k, float* topk_dist,
                            int32_t* topk_id, kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  kgq_status st = peer_push_check(ctx);
  if (st) return st;
  int64_t Q = 0;
  for (int i = 0; structures && batches && i < n_groups; ++i) Q += batches[i] > 0 ? batches[i] : 0;
  if (!ctx->comm || Q == 0) {
    st = submit_mixed_impl(ctx, n_groups, structures, batches, anchors, rels, k, topk_dist, topk_id, stream);
    return Q > 0 ? peer_push_done(ctx, st) : st;
  }
  // communicator data plane (kgq_comm_init), as submit_comm for one structure
  for (int i = 0; i < n_groups; ++i)
    if ((st = check_submit(ctx, structures[i], batches[i], k, true))) return st;
  if (Q > ctx->cfg.max_batch)
    return fail(ctx, KGQ_EINVAL, "mixed submit: %lld queries > max_batch %d", (long long)Q, ctx->cfg.max_batch);
  if (!anchors || !rels || !topk_dist || !topk_id) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  DeviceGuard dg(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  const int W = ctx->comm_world;
  if (ctx->comm_split == KGQ_SPLIT_ENTITIES) {
    st = submit_mixed_impl(ctx, n_groups, structures, batches, anchors, rels, k, ctx->cm_d, ctx->cm_i, stream);
    if (st) return st;
    int L = ctx->launches;
    if ((st = comm_gather(ctx, (size_t)Q * k, cs))) return st;
    L += launch_merge(W, (int)Q, k, ctx->cg_d, ctx->cg_i, topk_dist, topk_id, cs);
    ctx->launches = L;
    CK(cudaGetLastError(), "merge launch");
    return KGQ_OK;
  }
  // query split: this rank's global rows [lo, hi) cut across the groups; the groups' anchor /
  // relation blocks are concatenated in row order, so the slice's inputs are contiguous
  int32_t lo, hi;
  query_range((int32_t)Q, W, ctx->comm_rank, &lo, &hi);
  const int32_t c = ((int32_t)Q + W - 1) / W;
  std::vector<int32_t> ss, bs;
  const int32_t *a_loc = nullptr, *r_loc = nullptr;
  int64_t q0 = 0, ao = 0, ro = 0;
  for (int i = 0; i < n_groups; ++i) {
    const Plan* P = plan_of(structures[i]);
    const int64_t b0 = std::max<int64_t>(q0, lo), b1 = std::min<int64_t>(q0 + batches[i], hi);
    if (b1 > b0) {
      if (!a_loc) {
        a_loc = anchors + ao + (b0 - q0) * P->n_anchor;
        r_loc = rels + ro + (b0 - q0) * P->n_rel;
      }
      ss.push_back(structures[i]);
      bs.push_back((int32_t)(b1 - b0));
    }
    q0 += batches[i];
    ao += (int64_t)batches[i] * P->n_anchor;
    ro += (int64_t)batches[i] * P->n_rel;
  }
  ctx->launches = 0;
  if (!ss.empty()) {
    st = submit_mixed_impl(ctx, (int32_t)ss.size(), ss.data(), bs.data(), a_loc, r_loc, k, ctx->cm_d, ctx->cm_i,
                           stream);
    if (st) return st;
  }
  if ((st = comm_gather(ctx, (size_t)c * k, cs))) return st;
  CK(cudaMemcpyAsync(topk_dist, ctx->cg_d, (size_t)Q * k * sizeof(float), cudaMemcpyDeviceToDevice, cs), "gather copy");
  CK(cudaMemcpyAsync(topk_id, ctx->cg_i, (size_t)Q * k * sizeof(int32_t), cudaMemcpyDeviceToDevice, cs), "gather copy");
  return KGQ_OK;
}

kgq_status kgq_submit_host(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                           const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                           kgq_stream stream) {
  kgq_status st = kgq_submit_host_async(ctx, s, batch, anchors, rels, k, topk_dist, topk_id, stream);
  if (st || batch == 0) return st;
  CK(cudaStreamSynchronize((cudaStream_t)stream), "submit_host sync");
  return KGQ_OK;
}

kgq_status kgq_submit_host_async(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                                 const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                                 kgq_stream stream) {
  kgq_status st = check_submit(ctx, s, batch, k, true);
  if (st) return st;
  if (batch == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !topk_dist || !topk_id) return fail(ctx, KGQ_EINVAL, "NULL host pointer");
  if ((st = peer_push_check(ctx))) return st;
  DeviceGuard g(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  const Plan* P = plan_of(s);
  CK(cudaMemcpyAsync(ctx->d_anchor_stage, anchors, (size_t)batch * P->n_anchor * sizeof(int32_t),
                     cudaMemcpyHostToDevice, cs), "anchor upload");
  CK(cudaMemcpyAsync(ctx->d_rel_stage, rels, (size_t)batch * P->n_rel * sizeof(int32_t),
                     cudaMemcpyHostToDevice, cs), "relation upload");
  ctx->push_row0 = ctx->peers.on() ? 0 : -1;
  st = submit_dev(ctx, s, batch, ctx->d_anchor_stage, ctx->d_rel_stage, k, ctx->d_topd_stage, ctx->d_topi_stage,
                  nullptr, cs);
  if (st) return st;
  peer_push_done(ctx, st);
  CK(cudaMemcpyAsync(topk_dist, ctx->d_topd_stage, (size_t)batch * k * sizeof(float), cudaMemcpyDeviceToHost, cs),
     "top-k download");
  CK(cudaMemcpyAsync(topk_id, ctx->d_topi_stage, (size_t)batch * k * sizeof(int32_t), cudaMemcpyDeviceToHost, cs),
     "top-k download");
  return KGQ_OK;
}

kgq_status kgq_submit_mixed_host_async(kgq_ctx* ctx, int32_t n_groups, const int32_t* structures,
                                       const int32_t* batches, const int32_t* anchors, const int32_t* rels, int32_t k,
                                       float* topk_dist, int32_t* topk_id, kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (n_groups < 0 || (n_groups > 0 && (!structures || !batches)))
    return fail(ctx, KGQ_EINVAL, "mixed submit: bad group arrays");
  int64_t Q = 0, na = 0, nr = 0;
  for (int i = 0; i < n_groups; ++i) {
    kgq_status st = check_submit(ctx, structures[i], batches[i], k, true);
    if (st) return st;
    const Plan* P = plan_of(structures[i]);
    Q += batches[i];
    na += (int64_t)batches[i] * P->n_anchor;
    nr += (int64_t)batches[i] * P->n_rel;
  }
  if (Q > ctx->cfg.max_batch)
    return fail(ctx, KGQ_EINVAL, "mixed submit: %lld queries > max_batch %d", (long long)Q, ctx->cfg.max_batch);
  if (Q == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !topk_dist || !topk_id) return fail(ctx, KGQ_EINVAL, "NULL host pointer");
  DeviceGuard g(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  // staging holds max_batch x kMaxBranches ids: every structure has <= 3 anchors and relations
  CK(cudaMemcpyAsync(ctx->d_anchor_stage, anchors, (size_t)na * sizeof(int32_t), cudaMemcpyHostToDevice, cs),
     "anchor upload");
  CK(cudaMemcpyAsync(ctx->d_rel_stage, rels, (size_t)nr * sizeof(int32_t), cudaMemcpyHostToDevice, cs),
     "relation upload");
  kgq_status st = kgq_submit_mixed(ctx, n_groups, structures, batches, ctx->d_anchor_stage, ctx->d_rel_stage, k,
                                   ctx->d_topd_stage, ctx->d_topi_stage, stream);
  if (st) return st;
  CK(cudaMemcpyAsync(topk_dist, ctx->d_topd_stage, (size_t)Q * k * sizeof(float), cudaMemcpyDeviceToHost, cs),
     "top-k download");
  CK(cudaMemcpyAsync(topk_id, ctx->d_topi_stage, (size_t)Q * k * sizeof(int32_t), cudaMemcpyDeviceToHost, cs),
     "top-k download");
  return KGQ_OK;
}

kgq_status kgq_set_option(kgq_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (option == KGQ_OPT_FUSED_TOPK) {
    if (value != KGQ_FUSED_OFF && value != KGQ_FUSED_ON && value != KGQ_FUSED_AUTO)
      return fail(ctx, KGQ_EINVAL, "KGQ_OPT_FUSED_TOPK: value %lld is not OFF / ON / AUTO", (long long)value);
    if (ctx->fused_topk != (int)value) {
      ctx->fused_topk = (int)value;
      // captured graphs hold the previous path: re-capture (after the device drained them and
      // their stage events were harvested, as kgq_ktime_enable does)
      DeviceGuard g(ctx->cfg.device);
      CK(cudaDeviceSynchronize(), "set_option");
      for (auto& gr : ctx->graphs) {
        if (gr.pending) harvest(ctx, gr.evs, false);
        destroy_graph_entry(gr);
      }
      ctx->graphs.clear();
      clear_mix_graphs(ctx);
    }
    return KGQ_OK;
  }
  return fail(ctx, KGQ_EINVAL, "unknown option %d", (int)option);
}

kgq_status kgq_query_embedding(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                               const int32_t* rels, float* out, kgq_stream stream) {
  kgq_status st = check_submit(ctx, s, batch, 0, false);
  if (st) return st;
  if (batch == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !out) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  DeviceGuard g(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  CK(cudaMemsetAsync(ctx->d_invalid, 0, (size_t)batch * sizeof(int32_t), cs), "reset flags");
  ctx->launches = run_chain(ctx, s, batch, anchors, rels, cs);
  const Plan* P = plan_of(s);
  CK(cudaMemcpyAsync(out, ctx->Q, (size_t)batch * P->n_out * ctx->qw * sizeof(float),
                     cudaMemcpyDeviceToDevice, cs), "embedding copy");
  CK(cudaGetLastError(), "query_embedding launch");
  return KGQ_OK;
}

kgq_status kgq_merge_topk(kgq_ctx* ctx, int32_t parts, int32_t batch, int32_t k, const float* in_d,
                          const int32_t* in_i, float* out_d, int32_t* out_i, kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (parts < 1 || batch < 0 || k < 1 || k > ctx->cfg.max_k || (int64_t)parts * k > 4096)
    return fail(ctx, KGQ_EINVAL, "merge: parts %d, batch %d, k %d (need parts*k <= 4096, k <= max_k)", parts,
                batch, k);
  if (batch == 0) return KGQ_OK;
  if (!in_d || !in_i || !out_d || !out_i) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  DeviceGuard g(ctx->cfg.device);
  launch_merge(parts, batch, k, in_d, in_i, out_d, out_i, (cudaStream_t)stream);
  ctx->launches = 1;
  CK(cudaGetLastError(), "merge launch");
  return KGQ_OK;
}

int32_t kgq_tensor_mmas_per_fma(void) { return kMmasPerFma; }

kgq_status kgq_check_errors(kgq_ctx* ctx, kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  DeviceGuard g(ctx->cfg.device);
  CK(cudaStreamSynchronize((cudaStream_t)stream), "stream synchronize");
  if (ctx->comm) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = nccl_api().CommGetAsyncError(static_cast<ncclComm_t>(ctx->comm), &ar);
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommGetAsyncError");
    if (ar != ncclSuccess) return nccl_fail(ctx, ar, "communicator (asynchronous)");
  }
  int32_t e[4];
  CK(cudaMemcpy(e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost), "error word");
  if (e[0] == 2) {
    CK(cudaMemset(ctx->d_err, 0, sizeof e), "error reset");
    return fail(ctx, KGQ_EINVAL, "kgq_rank_answers: a query has more than %d answers", kMaxAnswers);
  }
  if (e[0] == 3) {
    CK(cudaMemset(ctx->d_err, 0, sizeof e), "error reset");
    return fail(ctx, KGQ_ESTATE, "kgq_merge_peers: rank %d did not publish row %d within %lld ms; the peer "
                "session is closed (every rank must call kgq_set_peers again)", e[2], e[1],
                ctx->peer_timeout_ns / 1000000);
  }
  if (e[0] == 4) {
    CK(cudaMemset(ctx->d_err, 0, sizeof e), "error reset");
    return fail(ctx, KGQ_ESTATE, "kgq_merge_peers: the peer session was closed by an earlier timeout; every "
                "rank must call kgq_set_peers again");
  }
  if (e[0]) {
    CK(cudaMemset(ctx->d_err, 0, sizeof e), "error reset");
    return fail(ctx, KGQ_ERANGE, "query row %d: %s slot %d out of range", e[1], e[3] ? "relation" : "anchor",
                e[2]);
  }
  if (range_flags_taken())
    return fail(ctx, KGQ_ERANGE, "an operand of the tensor-core GEMMs reached the fp16x2 range (|x| >= 65504): "
                "results since the last check are not exact; use the bf16x3 build (libkgq_bf16x3.so, "
                "KGQ_OPERANDS=bf16x3) for such inputs");
  return KGQ_OK;
}

// ---- N2: fused top-k all-gather over peer memory (peer.cuh) --------------------------------
int64_t kgq_peer_bytes(const kgq_ctx* ctx, int32_t world) {
  if (!ctx || world < 1 || world > kMaxPeers) return -1;
  return peer_flag_bytes(ctx, world) +
         (int64_t)2 * world * ctx->cfg.max_batch * (int64_t)ctx->cfg.max_k * (int64_t)sizeof(unsigned long long);
}

kgq_status kgq_set_peers(kgq_ctx* ctx, int32_t rank, int32_t world, void* const* peer_bufs) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (ctx->comm && world != 0)
    return fail(ctx, KGQ_ESTATE, "kgq_set_peers: the context has a communicator (kgq_comm_destroy first)");
  DeviceGuard g(ctx->cfg.device);
  for (auto& gr : ctx->graphs) {  // captured submits bake in the old push arguments
    if (gr.pending) harvest(ctx, gr.evs, false);
    destroy_graph_entry(gr);
  }
  ctx->graphs.clear();
  clear_mix_graphs(ctx);
  if (world == 0) {
    ctx->peers = PeerPush{};
    ctx->push_outstanding = false;
    return KGQ_OK;
  }
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return fail(ctx, KGQ_EINVAL, "kgq_set_peers: rank %d / world %d (1 <= world <= %d)", rank, world, kMaxPeers);
  if (!peer_bufs) return fail(ctx, KGQ_EINVAL, "kgq_set_peers: peer_bufs is NULL");
  for (int p = 0; p < world; ++p)
    if (!peer_bufs[p] || ((uintptr_t)peer_bufs[p] & 255))
      return fail(ctx, KGQ_EINVAL, "kgq_set_peers: buffer of rank %d is NULL or not 256-byte aligned", p);
  if (!ctx->d_epoch) {
    kgq_status st = dalloc(ctx, &ctx->d_epoch, 2, "peer epoch");
    if (st) return st;
  }
  const char* to = getenv("KGQ_PEER_TIMEOUT_MS");
  if (to && atoll(to) > 0) ctx->peer_timeout_ns = atoll(to) * 1000000LL;
  PeerPush pp{};
  pp.world = world;
  pp.rank = rank;
  pp.max_rows = ctx->cfg.max_batch;
  pp.max_k = ctx->cfg.max_k;
  pp.epoch = ctx->d_epoch;
  const int64_t fb = peer_flag_bytes(ctx, world);
  for (int p = 0; p < world; ++p) {
    pp.hdr[p] = static_cast<uint32_t*>(peer_bufs[p]);
    pp.flag[p] = reinterpret_cast<uint32_t*>(static_cast<char*>(peer_bufs[p]) + kPeerHdrBytes);
    pp.key[p] = reinterpret_cast<unsigned long long*>(static_cast<char*>(peer_bufs[p]) + fb);
  }
  CK(cudaMemset(peer_bufs[rank], 0, (size_t)kgq_peer_bytes(ctx, world)), "peer buffer reset");
  const uint32_t ep0[2] = {1u, 0u};
  CK(cudaMemcpy(ctx->d_epoch, ep0, sizeof ep0, cudaMemcpyHostToDevice), "peer epoch reset");
  CK(cudaDeviceSynchronize(), "kgq_set_peers");
  ctx->peers = pp;
  ctx->push_outstanding = false;
  return KGQ_OK;
}

kgq_status kgq_merge_peers(kgq_ctx* ctx, int32_t batch, int32_t k, float* out_dist, int32_t* out_id,
                           kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (!ctx->peers.on()) return fail(ctx, KGQ_ESTATE, "kgq_merge_peers: no peers registered (kgq_set_peers)");
  if (batch < 0 || batch > ctx->cfg.max_batch) return fail(ctx, KGQ_EINVAL, "batch %d outside [0, max_batch]", batch);
  if (k < 1 || k > ctx->cfg.max_k) return fail(ctx, KGQ_EINVAL, "k %d outside [1, max_k=%d]", k, ctx->cfg.max_k);
  if (batch == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!out_dist || !out_id) return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  if (!ctx->push_outstanding)
    return fail(ctx, KGQ_ESTATE, "kgq_merge_peers: no pushing submit since the last merge on this rank");
  ctx->push_outstanding = false;
  DeviceGuard g(ctx->cfg.device);
  PeerPush pp = ctx->peers;
  pp.row0 = 0;
  ctx->launches = launch_peer_merge(pp, batch, k, out_dist, out_id, ctx->d_err, ctx->peer_timeout_ns,
                                    (cudaStream_t)stream);
  CK(cudaGetLastError(), "kgq_merge_peers launch");
  return KGQ_OK;
}

kgq_status kgq_query_range(int32_t batch, int32_t world, int32_t rank, int32_t* lo, int32_t* hi) {
  if (batch < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi)
    return fail(nullptr, KGQ_EINVAL, "kgq_query_range: batch %d, world %d, rank %d", batch, world, rank);
  query_range(batch, world, rank, lo, hi);
  return KGQ_OK;
}

kgq_status kgq_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(nullptr, KGQ_EINVAL, "kgq_nccl_unique_id: id is NULL");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(nullptr, KGQ_ENCCL, "%s", api.why.c_str());
  ncclUniqueId u;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  ncclResult_t r = api.GetUniqueId(&u);
  if (r != ncclSuccess) return fail(nullptr, KGQ_ENCCL, "ncclGetUniqueId: %s", api.GetErrorString(r));
  memcpy(id, &u, sizeof u);
  return KGQ_OK;
}

kgq_status kgq_comm_init(kgq_ctx* ctx, const uint8_t* id, int32_t world, int32_t rank, int32_t split) {
  if (!ctx || !id) return fail(ctx, KGQ_EINVAL, "kgq_comm_init: NULL argument");
  if (ctx->comm) return fail(ctx, KGQ_ESTATE, "kgq_comm_init: the context already has a communicator");
  if (ctx->peers.on()) return fail(ctx, KGQ_ESTATE, "kgq_comm_init: peers are set (kgq_set_peers(ctx, 0, 0, NULL) first)");
  if (world < 1 || world > 4096 || rank < 0 || rank >= world)
    return fail(ctx, KGQ_EINVAL, "kgq_comm_init: rank %d / world %d", rank, world);
  if (split == KGQ_SPLIT_ENTITIES) {
    if (ctx->cfg.world_size != world || ctx->cfg.rank != rank)
      return fail(ctx, KGQ_EINVAL, "kgq_comm_init: entity split needs cfg.world_size == %d and cfg.rank == %d "
                  "(context: %d / %d)", world, rank, ctx->cfg.world_size, ctx->cfg.rank);
  } else if (split == KGQ_SPLIT_QUERIES) {
    if (ctx->cfg.world_size != 1)
      return fail(ctx, KGQ_EINVAL, "kgq_comm_init: query split needs a context with the whole entity table "
                  "(cfg.world_size == 1)");
  } else {
    return fail(ctx, KGQ_EINVAL, "kgq_comm_init: bad split %d", split);
  }
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(ctx, KGQ_ENCCL, "%s", api.why.c_str());
  DeviceGuard g(ctx->cfg.device);
  const size_t n = (size_t)ctx->cfg.max_batch * ctx->cfg.max_k;
  kgq_status st = KGQ_OK;
  if (!ctx->cm_d) {
    st = dalloc(ctx, &ctx->cm_d, n, "comm top-k");
    if (!st) st = dalloc(ctx, &ctx->cm_i, n, "comm top-k");
  }
  if (!st) {
    if (ctx->cg_d) cudaFree(ctx->cg_d);
    if (ctx->cg_i) cudaFree(ctx->cg_i);
    ctx->cg_d = nullptr;
    ctx->cg_i = nullptr;
    // query split pads each rank's slice to ceil(B / W) rows: W * ceil(B / W) <= B + W - 1
    const size_t ng = (size_t)world * n + (size_t)world * ctx->cfg.max_k;
    st = dalloc(ctx, &ctx->cg_d, ng, "comm gather");
    if (!st) st = dalloc(ctx, &ctx->cg_i, ng, "comm gather");
  }
  if (st) return st;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.CommInitRank(&comm, world, u, rank);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommInitRank");
  for (auto& gr : ctx->graphs) {  // the data plane changed under the captured submits
    if (gr.pending) harvest(ctx, gr.evs, false);
    destroy_graph_entry(gr);
  }
  ctx->graphs.clear();
  clear_mix_graphs(ctx);
  ctx->comm = comm;
  ctx->comm_world = world;
  ctx->comm_rank = rank;
  ctx->comm_split = split;
  return KGQ_OK;
}

kgq_status kgq_comm_destroy(kgq_ctx* ctx) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (!ctx->comm) return KGQ_OK;
  DeviceGuard g(ctx->cfg.device);
  CK(cudaDeviceSynchronize(), "kgq_comm_destroy");
  ncclResult_t r = nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
  ctx->comm = nullptr;
  ctx->comm_world = 0;
  for (auto& gr : ctx->graphs) {
    if (gr.pending) harvest(ctx, gr.evs, false);
    destroy_graph_entry(gr);
  }
  ctx->graphs.clear();
  clear_mix_graphs(ctx);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommDestroy");
  return KGQ_OK;
}

kgq_status kgq_rank_metrics(kgq_ctx* ctx, int32_t batch, const int32_t* ans_off, const int32_t* ranks,
                            const uint8_t* hard, double* metrics, kgq_stream stream) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  if (batch < 0 || !ans_off || !ranks || !metrics) return fail(ctx, KGQ_EINVAL, "kgq_rank_metrics: bad argument");
  DeviceGuard g(ctx->cfg.device);
  ctx->launches = launch_rank_metrics(batch, ans_off, ranks, hard, metrics, (cudaStream_t)stream);
  CK(cudaGetLastError(), "rank metrics launch");
  return KGQ_OK;
}

int32_t kgq_last_launch_count(const kgq_ctx* ctx) { return ctx ? ctx->launches : -1; }

kgq_status kgq_entity_terms(kgq_ctx* ctx, float* out, kgq_stream stream) {
  if (!ctx || !out) return fail(ctx, KGQ_EINVAL, "NULL argument");
  if (!ctx->finalized) return fail(ctx, KGQ_ESTATE, "not finalized");
  if (ctx->cfg.model != KGQ_BETAE) return fail(ctx, KGQ_EUNSUPPORTED, "entity terms exist only for BetaE");
  DeviceGuard g(ctx->cfg.device);
  const int d = ctx->cfg.dim;
  // tab [d][3][np] -> out [3][d][ns]
  for (int p = 0; p < 3; ++p)
    CK(cudaMemcpy2DAsync(out + (int64_t)p * d * ctx->ns, ctx->ns * sizeof(float), ctx->score_tab + p * ctx->np,
                         3 * ctx->np * sizeof(float), ctx->ns * sizeof(float), d, cudaMemcpyDeviceToDevice,
                         (cudaStream_t)stream),
       "entity terms copy");
  return KGQ_OK;
}

kgq_status kgq_rank_answers(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                            const int32_t* rels, const int32_t* ans_off, const int32_t* ans_id,
                            int32_t n_ans, int32_t mode, float* ans_dist, int32_t* count,
                            kgq_stream stream) {
  kgq_status st = check_submit(ctx, s, batch, 0, false);
  if (st) return st;
  if (mode < KGQ_RANK_LOCAL || mode > KGQ_RANK_FILTERED) return fail(ctx, KGQ_EINVAL, "bad rank mode %d", mode);
  const bool sharded = ctx->cfg.world_size > 1;
  if (mode == KGQ_RANK_LOCAL && sharded)
    return fail(ctx, KGQ_EINVAL, "KGQ_RANK_LOCAL needs a single shard; use KGQ_RANK_DIST + min-reduce + KGQ_RANK_COUNT"
                " or KGQ_RANK_FILTERED with a communicator");
  if (mode == KGQ_RANK_FILTERED && sharded && !(ctx->comm && ctx->comm_split == KGQ_SPLIT_ENTITIES))
    return fail(ctx, KGQ_EINVAL, "KGQ_RANK_FILTERED over entity shards needs the communicator (kgq_comm_init)");
  if (batch == 0 || n_ans == 0) { ctx->launches = 0; return KGQ_OK; }
  if (!anchors || !rels || !ans_off || !ans_id || !ans_dist || (mode != KGQ_RANK_DIST && !count))
    return fail(ctx, KGQ_EINVAL, "NULL device pointer");
  DeviceGuard g(ctx->cfg.device);
  cudaStream_t cs = (cudaStream_t)stream;
  const Plan* P = plan_of(s);
  int L = 0;
  // one pass: chain, then per chunk of rows the scorer and the answer-distance / count kernels
  auto pass = [&](int m, bool count_only) {
    if (!count_only) {
      CK(cudaMemsetAsync(ctx->d_invalid, 0, (size_t)batch * sizeof(int32_t), cs), "reset flags");
    }
    const bool from_state = q_in_state(ctx, P, batch);
    if (!count_only) L += run_chain(ctx, s, batch, anchors, rels, cs, !from_state);
    for (int64_t b0 = 0; b0 < batch; b0 += ctx->bchunk) {
      const int nb = (int)std::min<int64_t>(ctx->bchunk, batch - b0);
      if (!count_only) L += score_rows(ctx, P, b0, nb, cs, batch, from_state);
      if (m != KGQ_RANK_COUNT)
        L += launch_answer_dist(ctx->dist, ctx->np, ctx->e0, ctx->ns, (int)b0, nb, ans_off, ans_id, ans_dist, cs);
      if (m != KGQ_RANK_DIST)
        L += launch_filtered_counts(ctx->dist, ctx->np, ctx->e0, ctx->ns, (int)b0, nb, ans_off, ans_id, ans_dist,
                                    count, ctx->d_err, cs);
    }
    return KGQ_OK;
  };
  st = KGQ_OK;
  if (mode != KGQ_RANK_FILTERED) {
    st = pass(mode, false);
  } else if (!sharded) {
    st = pass(KGQ_RANK_LOCAL, false);
    if (!st) L += launch_add_one(count, n_ans, cs);
  } else {  // entity shards: answer distances from their owning shard, then every shard's counts
    const NcclApi& api = nccl_api();
    ncclComm_t comm = static_cast<ncclComm_t>(ctx->comm);
    st = pass(KGQ_RANK_DIST, false);
    if (st) return st;
    ncclResult_t r = api.AllReduce(ans_dist, ans_dist, (size_t)n_ans, ncclFloat32, ncclMin, comm, cs);
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllReduce(min)");
    // one chunk: the distance block of the pass above is still there; else score again
    st = pass(KGQ_RANK_COUNT, batch <= ctx->bchunk);
    if (st) return st;
    r = api.AllReduce(count, count, (size_t)n_ans, ncclInt32, ncclSum, comm, cs);
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllReduce(sum)");
    L += launch_add_one(count, n_ans, cs);
  }
  if (st) return st;
  ctx->launches = L;
  CK(cudaGetLastError(), "rank launch");
  return KGQ_OK;
}

// four span groups (dense / score on the context's stream, dense / score on its side stream:
// tc_gemm.cuh kt_end), the log count at [32], the log from [40]
static const unsigned long long kKtInit[40] = {~0ull, 0, 0, 0, 0, 0, 0, 0, ~0ull, 0, 0, 0, 0, 1, 0, 0,
                                               ~0ull, 0, 0, 0, 0, 2, 0, 0, ~0ull, 0, 0, 0, 0, 3, 0, 0,
                                               0,    0, 0, 0, 0, 0, 0, 0};
constexpr size_t kKtWords = 40 + 3 * kKtLogCap;

kgq_status kgq_ktime_enable(kgq_ctx* ctx, int32_t on) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  DeviceGuard g(ctx->cfg.device);
  if (on && !ctx->kt_buf) {
    kgq_status st = dalloc(ctx, &ctx->kt_buf, kKtWords, "ktime words");
    if (st) return st;
    CK(cudaMemcpy(ctx->kt_buf, kKtInit, sizeof kKtInit, cudaMemcpyHostToDevice), "ktime init");
  }
  unsigned long long* want = on ? ctx->kt_buf : nullptr;
  if (ctx->gws.kt != want) {  // captured graphs carry the old pointer
    CK(cudaDeviceSynchronize(), "ktime toggle");
    for (auto& gr : ctx->graphs) {
      if (gr.pending) harvest(ctx, gr.evs, false);
      destroy_graph_entry(gr);
    }
    ctx->graphs.clear();
    clear_mix_graphs(ctx);
    ctx->gws.kt = want;
    ctx->gws2.kt = want ? want + 16 : nullptr;
  }
  return KGQ_OK;
}

kgq_status kgq_ktime_read(kgq_ctx* ctx, double* ms, int64_t* n) {
  if (!ctx || !ms || !n) return fail(ctx, KGQ_EINVAL, "NULL argument");
  ms[0] = ms[1] = 0.0;
  n[0] = n[1] = 0;
  if (!ctx->kt_buf) return KGQ_OK;
  DeviceGuard g(ctx->cfg.device);
  unsigned long long h[32];  // the four span groups (the log stays: kgq_ktime_log)
  CK(cudaDeviceSynchronize(), "ktime read");
  CK(cudaMemcpy(h, ctx->kt_buf, sizeof h, cudaMemcpyDeviceToHost), "ktime read");
  for (int s = 0; s < 2; ++s) {  // stage s: group s (context stream) + group s + 2 (side stream)
    ms[s] = (double)(h[8 * s + 3] + h[8 * (s + 2) + 3]) * 1e-6;
    n[s] = (int64_t)(h[8 * s + 4] + h[8 * (s + 2) + 4]);
  }
  CK(cudaMemcpy(ctx->kt_buf, kKtInit, 32 * sizeof(unsigned long long), cudaMemcpyHostToDevice), "ktime reset");
  return KGQ_OK;
}

int64_t kgq_ktime_log(kgq_ctx* ctx, uint64_t* out, int64_t cap) {
  if (!ctx || cap < 0 || (cap > 0 && !out)) return -1;
  if (!ctx->kt_buf) return 0;
  DeviceGuard g(ctx->cfg.device);
  unsigned long long n = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpy(&n, ctx->kt_buf + 32, sizeof n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  n = std::min<unsigned long long>(n, kKtLogCap);
  const int64_t m = std::min<int64_t>((int64_t)n, cap);
  if (m > 0 && cudaMemcpy(out, ctx->kt_buf + 40, (size_t)m * 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  const unsigned long long zero = 0;
  if (cudaMemcpy(ctx->kt_buf + 32, &zero, sizeof zero, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
  return (int64_t)n;
}

kgq_status kgq_profile_enable(kgq_ctx* ctx, int32_t on) {
  if (!ctx) return fail(nullptr, KGQ_EINVAL, "ctx is NULL");
  ctx->profile = on != 0;
  return KGQ_OK;
}

kgq_status kgq_profile_read(kgq_ctx* ctx, double* ms, int64_t* n, double* work) {
  if (!ctx || !ms || !n) return fail(ctx, KGQ_EINVAL, "NULL argument");
  DeviceGuard g(ctx->cfg.device);
  harvest(ctx, ctx->prof_recs, true);
  for (auto& gr : ctx->graphs)
    if (gr.pending) {
      harvest(ctx, gr.evs, false);
      gr.pending = false;
    }
  for (int i = 0; i < kStNum; ++i) {
    ms[i] = ctx->prof_acc_ms[i];
    n[i] = ctx->prof_acc_n[i];
    if (work) work[i] = ctx->prof_acc_work[i];
    ctx->prof_acc_ms[i] = ctx->prof_acc_work[i] = 0;
    ctx->prof_acc_n[i] = 0;
  }
  return KGQ_OK;
}

}  // extern "C"
