// Internal declarations of libkgq.so (not part of the ABI; see include/kgq.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/kgq.h"
#include "common.cuh"
#include "peer.cuh"

namespace kgq {

constexpr int kMaxBranches = 3;   // 3i / 3in
constexpr int kMaxOps = 4;        // ops per branch chain
constexpr int kMaxLayers = 32;
constexpr int kMaxK = 256;
constexpr int kMaxAnswers = 2048;  // per query, kgq_rank_answers
constexpr int kEntityPad = 128;   // scorer entity tile; shard tables are padded to it
constexpr int kRowPad = 64;       // scorer query-row tile

// ---------------------------------------------------------------------------------------
// Static per-structure plan (SURVEY §8(b) slot table; Eq. 1 DNF; Eq. 2 mapping).
//   A branch is an anchor slot followed by ops: >= 0 projection with that relation slot,
//   kOpNeg = negation.  kind: single chain, intersection of branches (+ post projections),
//   or union of branches (one query embedding per DNF clause).
// ---------------------------------------------------------------------------------------
constexpr int kOpNeg = -1;
enum PlanKind { kSingle = 0, kInter = 1, kUnion = 2 };
struct BranchPlan {
  int anchor;
  int nops;
  int ops[kMaxOps];
};
struct Plan {
  int kind;
  int nbranch;
  BranchPlan br[kMaxBranches];
  int npost;        // projections applied after the intersection (ip, inp)
  int post[2];
  int n_anchor, n_rel, n_out;  // slot counts; n_out = DNF branches of the final embedding
  bool negation;
  bool neg_inter;   // negate the intersection result (De Morgan unions 2u-DM, up-DM)
};
const Plan* plan_of(int s);

struct Linear {
  float* W = nullptr;     // [out, in] fp32
  Split Wsp{};            // bf16x3 planes of W for the tensor-core path (ld = in)
  float* b = nullptr;     // [out]
  int out_f = 0, in_f = 0;
};

enum Epi { kEpiNone = 0, kEpiRelu = 1, kEpiBetaReg = 2 };

// Per-context scratch of the tensor-core GEMM's split tail (tc_gemm.cuh Sched): fp32 partial
// sums and arrival counters (zeroed once; every launch leaves them zero).
struct GemmWs {
  float* ws = nullptr;
  int* cnt = nullptr;
  // kgq_ktime_enable: in-kernel launch spans of the GEMM, [2 stages: dense, score][8] u64 =
  // {first CTA start (after the PDL wait), last CTA end, CTAs done, summed ns, launches}
  unsigned long long* kt = nullptr;
};
constexpr unsigned long long kKtLogCap = 1ull << 16;  // GEMM launch-span log entries (kgq_ktime_log)
constexpr size_t kGemmWsFloats = (size_t)74 * 256 * 256;  // <= 74 tail units of 256 x 256
constexpr int kGemmCntInts = 74 * 16;                      // <= 74 tail tiles x 16 epilogue warps

// A timed region: CUDA events recorded on the launching stream around one stage.
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
  double work;
};

// Profiling stages (kgq_profile_* in kgq_api.cu).
// kStDense is nested inside kStChain (every dense layer of the operator chain).
enum Stage { kStChain = 0, kStPrep = 1, kStScore = 2, kStTopk = 3, kStDense = 4, kStNum = 5 };

}  // namespace kgq

struct kgq_ctx {
  kgq_config cfg{};
  std::string err;
  int64_t e0 = 0, e1 = 0, ns = 0, np = 0;  // shard [e0, e1), size, padded size
  int ew = 0;                              // entity / state row width (d or 2d)
  int qw = 0;                              // query-embedding row width
  float* ent = nullptr;                    // [N, ew] row-major (BetaE: regularised at finalize)
  std::vector<uint8_t> ent_loaded;         // per-row loaded flags (host)
  int64_t ent_rows_loaded = 0;
  float* rel[2] = {nullptr, nullptr};
  kgq::Linear lin[kgq::kMaxLayers];
  float* score_tab = nullptr;              // GQE/Q2B: [d][np]; BetaE: [d][3][np] (C,U,V)
  bool finalized = false;

  // scratch (sized at finalize for max_batch)
  int64_t rows_max = 0;                    // kMaxBranches * max_batch
  kgq::Split S{}, Z{}, H[2]{}, I{}, M{};   // states, MLP input, hidden ping-pong, inter hidden, q2b mean
  float* T = nullptr;                      // generic fp32 GEMM output [rows_max, tw]
  int64_t tw = 0;
  float* T2 = nullptr;
  float* Q = nullptr;                      // final query embedding [B, 2, qw]
  float* Qt = nullptr;                     // scorer query operand planes [nplanes][d][rpad]
  int64_t rpad = 0;
  float* dist = nullptr;                   // [bchunk, np]
  float* cmin = nullptr;                   // [bchunk, np / 32] block minima (tensor-core scorer)
  unsigned long long* cand = nullptr;      // [bchunk, 128 lists, 16] fused top-k lists (BetaE scorer)
  int64_t bchunk = 0;
  float* topk_tmp_d = nullptr;             // chunked top-k candidates [<= 4096 per row]
  int32_t* topk_tmp_i = nullptr;
  // BetaE tensor-core scoring layout (score_tc.cu)
  kgq::Split uv{};                         // [np][2d] centred (u; v), bf16x3
  kgq::Linear lin1x{};                     // BetaE first projection layer, state columns W1[:, :2d]
  float* RW = nullptr;                     // [n_relation, H] relation term R W1[:, 2d:]^T (fp64 -> fp32)
  float* Hpre = nullptr;                   // [n_entity, H] X W1[:, :2d]^T + b1 of every (regularised) entity row
  int32_t* mix_rid = nullptr;              // mixed batches: per-row relation ids of a hop batch [rows_max]
  int64_t* mix_map = nullptr;              // mixed batches: score-row source rows [2 max_batch] + output rows
  int64_t* mix_map_host = nullptr;         // pinned staging of mix_map
  cudaEvent_t mix_map_ev = nullptr;        // staging reuse guard
  float2* Esum = nullptr;                  // [np] sum_d C_ed as an fp32 (hi, lo) pair
  float* uvT = nullptr;                    // [d][2][np] centred u, v in fp32 (small-batch streaming scorer)
  double* uvsums = nullptr;                // [2][d]
  kgq::GemmWs gws{};                       // tensor-core GEMM split-tail scratch
  kgq::Split Atc{};                        // [2*max_batch][2d] split query rows
  float2* Ptc = nullptr;                   // [2*max_batch] P_q as an fp32 (hi, lo) pair
  int32_t* d_err = nullptr;                // [4]: flag, row, slot, kind
  int32_t* d_invalid = nullptr;            // [max_batch]
  int32_t* d_anchor_stage = nullptr;       // kgq_submit_host staging
  int32_t* d_rel_stage = nullptr;
  float* d_topd_stage = nullptr;
  int32_t* d_topi_stage = nullptr;

  int launches = 0;
  bool profile = false;
  // CUDA graphs of whole submits, keyed by (structure, batch, k, caller pointers); captured on
  // the second identical call and replayed afterwards (kgq_api.cu submit_graphed)
  struct GraphEntry {
    int s, B, k;
    bool prof;  // captured with stage events (replays re-record them)
    const void* ptr[4];
    cudaGraphExec_t exec;
    int launches;
    int seen;
    uint64_t last;
    std::vector<kgq::ProfRec> evs;  // captured stage events (owned)
    bool pending;                   // a replay's events have not been harvested yet
  };
  GraphEntry* capture_entry = nullptr;      // set while capturing: stage events go there
  std::vector<kgq::ProfRec> prof_recs;      // eager stage events (owned until read)
  double prof_acc_ms[kgq::kStNum] = {}, prof_acc_work[kgq::kStNum] = {};
  int64_t prof_acc_n[kgq::kStNum] = {};
  std::vector<GraphEntry> graphs;
  // CUDA graphs of batched mixed submits, keyed by the (structure, batch) list, k and pointers;
  // each owns the pinned copy of its row map that its memcpy node uploads
  struct MixGraphEntry {
    std::vector<int32_t> key;
    const void* ptr[4];
    int k;
    cudaGraphExec_t exec;
    int launches;
    int seen;
    int64_t* map_host;
  };
  std::vector<MixGraphEntry> mgraphs;
  bool use_graphs = true;
  int fused_topk = KGQ_FUSED_AUTO;  // kgq_set_option(KGQ_OPT_FUSED_TOPK)
  uint64_t graph_clock = 0;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t side_st = nullptr;          // mixed path: the second row half of a large MLP hop
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
  kgq::GemmWs gws2{};                      // the side stream's split-K workspace / span group
  // N2: fused top-k all-gather over peer memory (kgq_set_peers); peers.world == 0: off
  kgq::PeerPush peers{};
  uint32_t* d_epoch = nullptr;             // [2]: epoch, merge CTA counter
  bool push_outstanding = false;  // N2: a submit pushed its top-k and kgq_merge_peers has not run yet
  int push_row0 = -1;      // set by the entry points: output-row offset of submit_impl's pushes (-1: none)
  long long peer_timeout_ns = 10000000000LL;  // KGQ_PEER_TIMEOUT_MS
  // multi-GPU data plane (kgq_comm_init): the context's NCCL communicator (ncclComm_t)
  void* comm = nullptr;
  int comm_world = 0, comm_rank = 0, comm_split = 0;
  float* cm_d = nullptr;                   // [max_batch, max_k] this rank's top-k (or row slice)
  int32_t* cm_i = nullptr;
  float* cg_d = nullptr;                   // [world * max_batch, max_k] all-gathered lists
  int32_t* cg_i = nullptr;
  unsigned long long* kt_buf = nullptr;    // kgq_ktime_enable: GEMM launch-span words [2][8]

};

namespace kgq {
// ---- kernel launchers (each returns the number of kernels launched) ---------------------
struct ChainArgs {
  int model;          // kgq_model
  int d;
  int nb;             // branches in this launch
  BranchPlan br[kMaxBranches];
  const int32_t* anchors;
  int n_a;
  const int32_t* rels;
  int n_r;
  int64_t n_entity;
  int n_relation;
  int32_t* err;
  int32_t* invalid;
};
// GQE/Q2B: anchor gather + translation chain for every branch (horizontal + vertical fusion).
// Output: if out_split.hi: split state rows [br*B + b]; else fp32 q[b, br, :] (width ew).
int launch_translate_chain(const ChainArgs& a, const float* ent, const float* rel,
                           const float* rel_off, int B, Split out_split, float* out_q,
                           cudaStream_t st);
// BetaE: build MLP input rows z = [x; R[r]] for a group of branches at one hop.
//   Group member gi -> Z rows [gi*B, gi*B+B); source = regularised anchor row (anchor_slot
//   >= 0) or split state rows [src_row, src_row+B).
struct MlpGroup {
  int n;
  int rel_slot[kMaxBranches];
  int anchor_slot[kMaxBranches];
  int64_t src_row[kMaxBranches];
};
int launch_betae_mlp_input(const ChainArgs& a, const float* ent, const float* rel, int B,
                           const MlpGroup& g, Split src, Split z, cudaStream_t st, bool with_rel = true);
// Dense layer: out = epi(A W^T + b) for rows [0, M), A given as split (K columns).
//   split (bf16x3) output into out_sp if out_sp.valid(), else fp32 into out_f32 (row stride ld_f32).
//   kEpiBetaReg: clamp(y+1, .05, 1e9), then 1/x on rows [neg0, neg1).
int launch_linear(const Split& A, int M, int K, const Linear& L, int epi, const Split& out_sp,
                  float* out_f32, int64_t ld_f32, int neg0, int neg1, const GemmWs* ws, cudaStream_t st);
// First BetaE projection layer with the relation input factored out of Eq. 4's z = [x; R[r]]:
// W1 z + b1 = W1[:, :2d] x + (R W1[:, 2d:]^T)[r] + b1.  RW = R W1[:, 2d:]^T is precomputed once in
// fp64 at finalize ([R, H] fp32); the GEMM runs with K = 2d on the state rows directly and its
// accumulators start at RW[r] of each row (EpiLinear<.., REL> init), r range-checked there.
struct RelTerm {
  const float* RW = nullptr;  // [n_relation, ldrw]
  const int32_t* rid = nullptr;  // optional per-row relation id (already range-checked)
  int64_t ldrw = 0;
  int M = 0, B = 0;           // rows = group member gi * B + query b
  const int32_t* rels = nullptr;
  int n_r = 0, n_relation = 0;
  int rel_slot[kMaxBranches] = {0, 0, 0};
  int32_t* err = nullptr;
  int32_t* invalid = nullptr;
};
int launch_linear_rel(const Split& A, int M, int K, const Linear& L, const RelTerm& rt, const Split& out,
                      const GemmWs* ws, cudaStream_t st);
// Output row remap of a dense layer (the mixed path's last MLP layer writes its rows straight into
// the state S instead of a scratch + scatter): GEMM row r of segment i (dst0[i] <= r, segments
// ascending, every segment a multiple of 32 rows) goes to output row src0[i] + r - dst0[i].
constexpr int kMaxRowMap = 48;
struct RowMap {
  int n = 0;
  int dst0[kMaxRowMap];
  int src0[kMaxRowMap];
};
// launch_linear with the split output rows remapped (out = the whole target, out_rows its rows)
int launch_linear_map(const Split& A, int M, int K, const Linear& L, int epi, const Split& out, int64_t out_rows,
                      const RowMap& rm, int neg0, int neg1, const GemmWs* ws, cudaStream_t st);
// ---- mixed-structure batches (kgq_submit_mixed) ----------------------------
// One block of B query rows inside a batched hop: rows [dst0, dst0 + B) of the batch come from
// anchor slot aslot (kind 0), state rows src0 + b of S (kind 1) or of the combined state Mst
// (kind 2); relation slot rslot; global query index q0 + b (error reporting, invalid flags).
struct MixSeg {
  int32_t dst0, B, q0, kind;
  int64_t src0;
  const int32_t* anchors;
  int32_t n_a, aslot;
  const int32_t* rels;
  int32_t n_r, rslot;
};
constexpr int kMaxMixSegs = 48;
struct MixSegs {
  int32_t n = 0;
  MixSeg s[kMaxMixSegs];
};
// batch rows -> Z [rows, 2d] split (state / regularised anchor rows) and rid[row] (checked)
int launch_mix_gather(const MixSegs& sg, int M, const float* ent, Split S, Split Mst, Split Z, int32_t* rid, int d,
                      int64_t n_entity, int n_relation, int32_t* err, int32_t* invalid, cudaStream_t st);
// hop-0 first projection layer from the per-entity precompute: H0[row] = split(ReLU(Hpre[anchor]
// + RW[rel] + bias)) for batch rows whose segments are anchor-sourced (kind 0); ids range-checked
int launch_mix_h0_pre(const MixSegs& sg, int M, const float* Hpre, const float* RW, int H,
                      Split H0, int64_t n_entity, int n_relation, int32_t* err, int32_t* invalid, cudaStream_t st);
// batch rows [dst0 + b] of src -> S rows src0 + b (width w)
int launch_mix_scatter(const MixSegs& sg, int M, Split src, Split S, int w, cudaStream_t st);
// score rows r: A[r] = S[srcrow[r]] (split copy) and P_q (fp64, as k_score_prep_tc); srcrow
// nullptr: row r of a single-structure chunk = state row (r % nout) * B + b0 + r / nout
int launch_mix_score_prep(const int64_t* srcrow, Split S, int rows, int d, const double* sums, int64_t ns,
                          Split A, float2* P, cudaStream_t st, int64_t B = 0, int64_t b0 = 0, int nout = 1);
// tensor-core score GEMM only (A and P prepared): dist rows = rows / nbq
int launch_score_tc_gemm(int rows, int nbq, int d, Split A, const float2* P, const Split& uv, const float2* Esum,
                         int64_t np, float* dist, int64_t ldd, float* cmin, int64_t ldc, int64_t nvalid,
                         const GemmWs* ws, cudaStream_t st);
// block-minima top-k with an output row map (out_row[b] = output / invalid-flag row of dist row b)
// fused top-k: the BetaE tensor-core scorer keeps per-stripe k-lists in its
// epilogue (no distance block; k <= kFusedTopkMax); *nlists = lists per output row
constexpr int kFusedTopkMax = 16;
constexpr int kFusedTopkLists = 128;  // <= 64 stripes x 2 column halves (the merge's 4 heads per lane)
int launch_score_tc_topk(int rows, int nbq, int d, Split A, const float2* P, const Split& uv, const float2* Esum,
                         int64_t np, int64_t nvalid, int k, unsigned long long* cand, int64_t ldcand,
                         const GemmWs* ws, cudaStream_t st, int* nlists, int min_tiles);
int launch_topk_lists(const unsigned long long* cand, int64_t ldcand, int k, int B, int rows1, int nl1, int nl2,
                      int64_t id_base, const int32_t* invalid, const int32_t* out_row, float* out_d, int32_t* out_i,
                      cudaStream_t st, const PeerPush& pp);
int launch_topk_cmin_map(const float* dist, int64_t ldd, const float* cmin, int64_t ldc, int B, int64_t n,
                         int k, int64_t id_base, const int32_t* invalid, const int32_t* out_row, float* out_d,
                         int32_t* out_i, cudaStream_t st, const PeerPush& pp);
// RW[r, n] = sum_k W[n, col0 + k] R[r, k] (k < d) in fp64 -> fp32
int launch_relation_term(const float* R, int n_relation, int d, const float* W, int64_t ldw, int col0, int H,
                         float* RW, cudaStream_t st);
// BetaE Eq.-4 softmax terminal over rows of T (width w) -> split state rows out_row0 + r,
// with negation on rows r in [neg0, neg1).
int launch_softmax_terminal(const float* T, int64_t ldt, int M, int w, Split out,
                            int64_t out_row0, int neg0, int neg1, cudaStream_t st);
// Negation x -> 1/x on split rows [r0, r1) (width w), in place.
int launch_negate(Split x, int64_t r0, int64_t r1, int w, cudaStream_t st);
// Q2B: mean over nb branches of T[br*B+b, :d] -> split [b, :d].
int launch_branch_mean(const float* T, int64_t ldt, int nb, int B, int d, Split out,
                       cudaStream_t st);
// Attention combine (softmax over branches per dim, weighted sum).  Q2B also applies the
// offset gate o = min_i o_i * sigmoid(G).  Optional post projection (GQE/Q2B only).
// Output split state (rows b) or fp32 q[b, 0, :].
struct CombineArgs {
  int model, nb, B, d;
  int64_t ldl, ldg;
  const float* rel;
  const float* rel_off;
  const int32_t* rels;
  int n_r, n_relation;
  int post_slot;  // -1: none
  int negate_out;  // BetaE: 1/x of the combined embedding (De Morgan union, N4)
  int32_t* err;
  int32_t* invalid;
};
int launch_attention_combine(const CombineArgs& c, Split S, const float* logits,
                             const float* gate, Split out_split, float* out_q, cudaStream_t st);
// attention combine of every intersection group in one launch (blocks = queries of all groups)
struct MixCombine {
  struct Group {
    CombineArgs c;   // per-group args (B, nb, negate_out, err / invalid at the group's queries)
    int32_t q_begin; // first block of this group
    int32_t q0;      // global query index (row of the combined state Mst when to_m)
    int64_t srow0;   // S (and logits) row of the group's branch-0 block
    int32_t to_m;    // 1: write the combined state to Mst rows q0.. (post projections follow);
                     // 0: in place into the branch-0 block
  };
  int32_t n = 0;
  Group g[16];
};
int launch_mix_combine(const MixCombine& mc, int total, Split S, const float* logits, int64_t ldl, Split Mst,
                       cudaStream_t st);
// Copy split state rows (b, branch br) to fp32 q[b, br, :].
int launch_state_to_q(Split S, int nb, int B, int w, float* q, cudaStream_t st);
// Scorer operands: query planes (k-major) from q[B, nbq, qw].
int launch_score_prep(int model, const float* q, int B, int nbq, int d, float* Qt,
                      int64_t rpad, cudaStream_t st);
// Scorer: dist[b, e] = min over DNF branches of distance(q_b,br, entity e0+e).
int launch_score(int model, int nbq, int B, int d, float cen, const float* Qt, int64_t rpad,
                 const float* tab, int64_t np, int64_t ns, float* dist, int64_t ldd,
                 cudaStream_t st);
// Top-k per row of dist (row length n, global id = id_base + index).
// Rows longer than 32k entries are split into chunks (one CTA each) whose candidates
// (tmp_d/tmp_i, <= 4096 per row) are merged by k_merge.
int launch_topk(const float* dist, int64_t ldd, int B, int64_t n, int k, int64_t id_base,
                const int32_t* invalid, float* out_d, int32_t* out_i, float* tmp_d, int32_t* tmp_i,
                cudaStream_t st);
bool score_uses_stream(int model, int nbq, int B);
// N1 filtered ranking (rank.cu)
int launch_add_one(int32_t* v, int n, cudaStream_t st);
int launch_rank_metrics(int B, const int32_t* ans_off, const int32_t* ranks, const uint8_t* hard, double* out,
                        cudaStream_t st);
int launch_answer_dist(const float* dist, int64_t ldd, int64_t e0, int64_t ns, int b0, int nb,
                       const int32_t* ans_off, const int32_t* ans_id, float* ans_dist, cudaStream_t st);
int launch_filtered_counts(const float* dist, int64_t ldd, int64_t e0, int64_t ns, int b0, int nb,
                           const int32_t* ans_off, const int32_t* ans_id, const float* ans_dist,
                           int32_t* count, int32_t* err, cudaStream_t st);
// Tensor-core BetaE scorer (score_tc.cu): finalize builds the centred split table
// uv [np][2d], E_e = sum_d C_ed (fp64) and the per-dim U/V sums; per batch it splits the
// query rows, computes P_q (fp64) and runs the bf16x3 tcgen05 GEMM with the score epilogue.
int launch_betae_uv_table(const float* ent, int64_t n_all, int64_t e0, int64_t ns, int64_t np, int d,
                          double* sums, Split uv, float2* Esum, float* uvT, cudaStream_t st);
// BetaE query prep of the tensor-core / streaming scorers: split [a; b] rows and fp64 P_q
// fp16x2 range flags of the translation units that convert to the operand format (read + clear)
unsigned int range_flag_chain();
unsigned int range_flag_linear();
unsigned int range_flag_score_tc();
int launch_score_prep_tc(const float* q, int rows, int d, const double* sums, int64_t ns, Split A, float2* P,
                         cudaStream_t st);
// BetaE small-batch scorer (<= 16 query rows) streaming the centred fp32 (u, v) table uvT [d][2][np]
int launch_score_betae_stream(const Split& A, const float2* P, const float* uvT, const float2* E, int64_t np, int d,
                              float* dist, int64_t ldd, int B, int nbq, cudaStream_t st);
int launch_score_betae_tc(const float* q, int rows, int nbq, int d, const double* sums, int64_t ns,
                          Split A, float2* P, const Split& uv, const float2* Esum,
                          int64_t np, float* dist, int64_t ldd, float* cmin, int64_t ldc, int64_t nvalid,
                          const GemmWs* ws, cudaStream_t st);
// Top-k of dist rows using the score epilogue's 32-entity block minima cmin [B][ldc] (k <= 32):
// tau = k-th smallest block minimum bounds the k-th best distance (k blocks each hold an
// entry <= tau), so only blocks with minimum <= tau are scanned.  Exact (dist, id) order.
int launch_topk_cmin(const float* dist, int64_t ldd, const float* cmin, int64_t ldc, int B, int64_t n,
                     int k, int64_t id_base, const int32_t* invalid, float* out_d, int32_t* out_i,
                     cudaStream_t st, const PeerPush& pp);
int launch_empty(cudaStream_t st);  // perf probe (KGQ_DBG_EMPTY_NODES)
// N2 (peer.cuh): push of finished output rows [0, B) of (out_d, out_i) (top-k paths without
// the fused push); the waiting merge (advances the epoch; epoch[1] is its CTA counter).
int launch_peer_push(const PeerPush& pp, int B, int k, const float* out_d, const int32_t* out_i, cudaStream_t st);
int launch_peer_merge(const PeerPush& pp, int B, int k, float* out_d, int32_t* out_i, int32_t* err,
                      long long timeout_ns, cudaStream_t st);
int launch_merge(int parts, int B, int k, const float* in_d, const int32_t* in_i, float* out_d,
                 int32_t* out_i, cudaStream_t st);
// Table preparation (finalize).
int launch_beta_regularize(float* ent, int64_t n_elems, cudaStream_t st);
int launch_transpose_shard(const float* ent, int64_t e0, int64_t ns, int d, int ew, float* tab,
                           int64_t np, cudaStream_t st);
int launch_betae_entity_terms(const float* ent, int64_t e0, int64_t ns, int d, float* tab,
                              int64_t np, cudaStream_t st);
int launch_split_copy(const float* src, int64_t n, Split dst, cudaStream_t st);
// fp32 [rows, cols] (row stride lds) -> split planes: the weight (W operand) form, or act = true
// the activation (A operand) form (common.cuh split3 / split3_w)
int launch_split_copy_rows(const float* src, int64_t rows, int cols, Split dst, cudaStream_t st, int64_t lds = 0,
                           bool act = false);
}  // namespace kgq
