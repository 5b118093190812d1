/*
 * kgq.h -- C ABI of libkgq.so: batched CLQA query-embedding inference on B200 (sm_100a).
 *
 * The hot path this library implements is the one
 * KGCompiler (arXiv 2503.02172) accelerates: for a batch of queries of ONE structure,
 * run the FOL operator chain of GQE / Query2Box / BetaE (projection, intersection,
 * negation, DNF union; Eq. 1, Eq. 2, Eq. 4,
 * P:146-150 fusion strategies), score the query embedding against every entity of this
 * rank's shard (the "entity similarity query") and return the k nearest.
 *
 * Conventions (all entry points):
 *  - Ids are int32, everything else fp32, row-major, C order.  Entity ids are GLOBAL.
 *  - Scores are DISTANCES (>= 0; logit = gamma - distance), returned
 *    ascending, ties broken by ascending entity id (Q13).
 *  - "host" pointers are ordinary CPU memory, "device" pointers are CUDA device memory on
 *    cfg.device.  The caller owns every pointer it passes; the library copies tables into
 *    device memory it owns and frees in kgq_destroy().
 *  - Every call returns a kgq_status; on failure kgq_last_error() describes it.  The
 *    library never aborts the process.  A context is not thread-safe; use one per stream.
 *  - Asynchronous calls are stream-ordered on the cudaStream_t passed (0 = legacy default).
 */
#ifndef KGQ_H
#define KGQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KGQ_ABI_VERSION 1u

typedef struct kgq_ctx kgq_ctx; /* opaque */
typedef struct CUstream_st* kgq_stream; /* == cudaStream_t */

typedef enum {
  KGQ_OK = 0,
  KGQ_EINVAL = 1,       /* bad argument (unknown structure, k > max_k, batch > max_batch, ...) */
  KGQ_ERANGE = 2,       /* a query id was out of range (reported by kgq_check_errors)        */
  KGQ_EUNSUPPORTED = 3, /* e.g. negation structure on GQE / Q2B                        */
  KGQ_ESTATE = 4,       /* missing tables, not finalized, finalized twice                     */
  KGQ_ENOMEM = 5,       /* device allocation failed                                           */
  KGQ_ECUDA = 6,        /* CUDA runtime / launch error                                        */
  KGQ_ENCCL = 7         /* NCCL cannot be loaded, or a collective of the communicator failed  */
} kgq_status;

typedef enum { KGQ_GQE = 0, KGQ_Q2B = 1, KGQ_BETAE = 2 } kgq_model;

/* The 14 query structures of P:34 / P:421 (Fig. 1 naming).  Slot layouts
 * (KGReasoning flattened order [ext]) with a_i = anchor slot, r_j = relation
 * slot, P = projection, I = intersection, N = negation, U = union (DNF, Eq. 1):
 *   1p  P(a0,r0)                         2p  P(P(a0,r0),r1)        3p  P(P(P(a0,r0),r1),r2)
 *   2i  I(P(a0,r0),P(a1,r1))             3i  I(P(a0,r0),P(a1,r1),P(a2,r2))
 *   pi  I(P(P(a0,r0),r1),P(a1,r2))       ip  P(I(P(a0,r0),P(a1,r1)),r2)
 *   2u  U(P(a0,r0),P(a1,r1))             up  U(P(P(a0,r0),r2),P(P(a1,r1),r2))
 *   2in I(P(a0,r0),N(P(a1,r1)))          3in I(P(a0,r0),P(a1,r1),N(P(a2,r2)))
 *   inp P(I(P(a0,r0),N(P(a1,r1))),r2)    pin I(P(P(a0,r0),r1),N(P(a1,r2)))
 *   pni I(N(P(P(a0,r0),r1)),P(a1,r2))
 * De Morgan unions (BetaE only -- they use negation; KGReasoning "2u-DM",
 * "up-DM" [ext]): the union as the negation of the intersection of the negated branches, one
 * embedding instead of the DNF min over clauses:
 *   2u-DM N(I(N(P(a0,r0)),N(P(a1,r1))))  up-DM P(N(I(N(P(a0,r0)),N(P(a1,r1)))),r2)          */
typedef enum {
  KGQ_1P = 0, KGQ_2P, KGQ_3P, KGQ_2I, KGQ_3I, KGQ_PI, KGQ_IP, KGQ_2U, KGQ_UP,
  KGQ_2IN, KGQ_3IN, KGQ_INP, KGQ_PIN, KGQ_PNI, KGQ_2U_DM, KGQ_UP_DM, KGQ_NUM_STRUCTURES
} kgq_structure;

/* BetaE projection terminal: KGReasoning regulariser clamp(y+1,0.05,1e9)
 * (default) or the literal Eq. 4 softmax over the 2d outputs followed by max(.,1e-6). */
typedef enum { KGQ_TERM_REGULARIZER = 0, KGQ_TERM_SOFTMAX = 1 } kgq_proj_terminal;

/* Relation tables (kgq_load_relations `which`). */
typedef enum { KGQ_REL_MAIN = 0, KGQ_REL_OFFSET = 1 /* Q2B only */ } kgq_relation_table;

/* nn.Linear layers (kgq_load_linear `layer_id`); W is [out_f, in_f] row-major, b is [out_f].
 *   BetaE projection MLP (Eq. 4; shared weights, input [alpha;beta;r], Q3/Q4):
 *     KGQ_LAYER_PROJ_OUT      = layer0 [2d, H]
 *     KGQ_LAYER_PROJ_HIDDEN+l = layer(l+1), l = 0..n_hidden_layers-1: layer1 [H,3d], others [H,H]
 *   Intersection attention (all models, Q6): KGQ_LAYER_INTER_1 [e,e], KGQ_LAYER_INTER_2 [d,e]
 *     with e = d (GQE, Q2B centre) or 2d (BetaE, input [alpha;beta]).
 *   Q2B offset gate: KGQ_LAYER_OFFSET_1 [d,d], KGQ_LAYER_OFFSET_2 [d,d].                    */
enum {
  KGQ_LAYER_PROJ_OUT = 0,
  KGQ_LAYER_PROJ_HIDDEN = 1, /* .. KGQ_LAYER_PROJ_HIDDEN + 7 */
  KGQ_LAYER_INTER_1 = 16,
  KGQ_LAYER_INTER_2 = 17,
  KGQ_LAYER_OFFSET_1 = 18,
  KGQ_LAYER_OFFSET_2 = 19
};

typedef struct {
  uint32_t abi_version;     /* must be KGQ_ABI_VERSION */
  int32_t model;            /* kgq_model */
  int64_t n_entity;         /* global N */
  int32_t n_relation;       /* R */
  int32_t dim;              /* d (multiple of 4) */
  int32_t hidden;           /* BetaE MLP width H (1600); ignored otherwise */
  int32_t n_hidden_layers;  /* BetaE MLP hidden layers (2), 1..8 */
  float cen;                /* Q2B inside-distance weight (0.02, Q10) */
  int32_t terminal;         /* kgq_proj_terminal (BetaE) */
  int32_t max_batch;        /* upper bound on `batch` in submit calls (scratch sizing) */
  int32_t max_k;            /* upper bound on k, <= 256 */
  int32_t device;           /* CUDA device ordinal */
  int32_t world_size;       /* number of entity shards (ranks), >= 1 */
  int32_t rank;             /* this rank's shard, 0 <= rank < world_size */
} kgq_config;

/* ---- lifetime ------------------------------------------------------------------------- */
/* Validate cfg and create a context on cfg.device.  *out is NULL on failure. */
kgq_status kgq_create(const kgq_config* cfg, kgq_ctx** out);
/* Free all device memory owned by ctx.  NULL-safe.  Synchronises the device. */
void kgq_destroy(kgq_ctx* ctx);
/* Message describing the last failure on ctx (or of the last kgq_create when ctx is NULL).
 * Valid until the next call on ctx. */
const char* kgq_last_error(const kgq_ctx* ctx);
const char* kgq_status_string(kgq_status s);

/* ---- structure metadata (pure host, no GPU needed) ------------------------------------- */
int32_t kgq_num_anchors(int32_t s);   /* -1 if s is not a kgq_structure */
int32_t kgq_num_relations(int32_t s);
int32_t kgq_num_branches(int32_t s);  /* DNF clauses: 2 for 2u/up, else 1 */
int32_t kgq_uses_negation(int32_t s);
const char* kgq_structure_name(int32_t s);       /* "1p" ... "pni", NULL if invalid */
int32_t kgq_structure_from_name(const char* n);  /* -1 if unknown */
/* Width of one query-embedding row: d (GQE), 2d (Q2B [centre;offset]), 2d (BetaE [alpha;beta]). */
int32_t kgq_embedding_width(int32_t model, int32_t dim);
/* Contiguous entity shard of `rank`: [r*ceil(N/W), min(N,(r+1)*ceil(N/W))). */
kgq_status kgq_shard_range(int64_t n_entity, int32_t world_size, int32_t rank,
                           int64_t* begin, int64_t* end);
int64_t kgq_shard_begin(const kgq_ctx* ctx);
int64_t kgq_shard_end(const kgq_ctx* ctx);

/* ---- tables (host pointers, copied synchronously) --------------------------------------- */
/* Rows [first_row, first_row+n_rows) of the GLOBAL entity table, host fp32:
 *   GQE / Q2B: [n_rows, d];  BetaE: raw [n_rows, 2d] = [alpha_raw; beta_raw] (Eq. 3 params
 *   before the regulariser, Q12).  May be called several times to stream a large table.
 * Every rank keeps all rows for anchor gathers (queries are replicated, §8(e)); the scoring
 * layout is built for this rank's shard only, at finalize. */
kgq_status kgq_load_entities(kgq_ctx* ctx, const float* rows, int64_t first_row, int64_t n_rows);
/* Relation table `which` (kgq_relation_table), host fp32 [n, d]; n must equal n_relation. */
kgq_status kgq_load_relations(kgq_ctx* ctx, int32_t which, const float* rows, int32_t n);
/* nn.Linear layer (see KGQ_LAYER_*): host W [out_f, in_f], b [out_f]; shapes are checked. */
kgq_status kgq_load_linear(kgq_ctx* ctx, int32_t layer_id, const float* W, const float* b,
                           int32_t out_f, int32_t in_f);
/* Check completeness, apply the BetaE regulariser to entity rows, build this shard's scoring
 * layout (BetaE: fp64 precompute of C, U, V per entity and dim), allocate
 * scratch for max_batch.  Synchronous.  Required before submit. */
kgq_status kgq_finalize(kgq_ctx* ctx);

/* ---- the hot path (device pointers, asynchronous on `stream`) --------------------------- */
/* anchors: device int32 [batch, kgq_num_anchors(s)]; rels: device int32 [batch,
 * kgq_num_relations(s)]; k in [1, min(max_k, shard size)].
 * Writes topk_dist fp32 [batch, k] and topk_id int32 [batch, k] (global ids, this shard's
 * k nearest, (dist, id) ascending).  shard_dist (optional, may be NULL): fp32
 * [batch, shard_end-shard_begin], the full distance row of every query (debug / parity).
 * Out-of-range ids are detected on the device: that query row gets dist NaN, id -1, and
 * kgq_check_errors() later returns KGQ_ERANGE. */
kgq_status kgq_submit(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                      const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                      float* shard_dist, kgq_stream stream);
/* Same as kgq_submit with HOST pointers: copies anchors/rels host->device, runs the path,
 * copies the top-k back, and synchronises `stream` before returning (end-to-end call). */
kgq_status kgq_submit_host(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                           const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                           kgq_stream stream);
/* kgq_submit_host without the final synchronisation: the copies and kernels are enqueued on
 * `stream` and the call returns; topk_dist / topk_id are valid (and anchors / rels may be
 * reused) once the stream has been synchronised.  With pinned host buffers consecutive calls
 * overlap the host turnaround with the previous submit's kernels; calls on one context are
 * ordered by the stream (the staging buffers are reused in stream order). */
kgq_status kgq_submit_host_async(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                                 const int32_t* rels, int32_t k, float* topk_dist, int32_t* topk_id,
                                 kgq_stream stream);
/* Mixed-structure batch: n_groups groups, group i = batches[i] queries of
 * structure structures[i] (host arrays).  anchors / rels: device int32, the groups' [B_i, n_a(s_i)]
 * and [B_i, n_r(s_i)] blocks concatenated in group order; topk_dist / topk_id: device
 * [sum B_i, k], rows in the same order.  Sum B_i <= max_batch.  BetaE runs the groups
 * level-synchronously (each projection hop of all groups' branches is one MLP, all
 * intersections one attention GEMM pair, the branch hops past the intersections' depth batched
 * with the post-intersection hops of equal depth, one scorer and one top-k for all queries); GQE / Q2B
 * (and BetaE with k > 32) run group by group.  Same results and error behaviour as one
 * kgq_submit per group (global query index in error reports). */
kgq_status kgq_submit_mixed(kgq_ctx* ctx, int32_t n_groups, const int32_t* structures, const int32_t* batches,
                            const int32_t* anchors, const int32_t* rels, int32_t k, float* topk_dist,
                            int32_t* topk_id, kgq_stream stream);
/* kgq_submit_mixed with HOST buffers, asynchronous (the end-to-end form of the mixed batch, as
 * kgq_submit_host_async is for one structure): anchors / rels host int32 in the same packed
 * group order, topk_dist / topk_id host [sum B_i, k]; the H2D copies, the whole path and the
 * D2H copies are enqueued on `stream` and the call returns.  Outputs are valid (and the inputs
 * reusable) once the stream is synchronised; use pinned buffers for overlap.  Errors as
 * kgq_submit_mixed; with a communicator the outputs are the merged / gathered global top-k. */
kgq_status kgq_submit_mixed_host_async(kgq_ctx* ctx, int32_t n_groups, const int32_t* structures,
                                       const int32_t* batches, const int32_t* anchors, const int32_t* rels,
                                       int32_t k, float* topk_dist, int32_t* topk_id, kgq_stream stream);
/* Operator chain only (parity aid): device out fp32 [batch, kgq_num_branches(s),
 * kgq_embedding_width(model, d)]. */
kgq_status kgq_query_embedding(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                               const int32_t* rels, float* out, kgq_stream stream);
/* Cross-shard merge (§8(e), a9): device in_dist fp32 [n_parts, batch, k], in_id int32
 * [n_parts, batch, k] (e.g. the result of an all-gather of every rank's top-k) -> device
 * out_dist/out_id [batch, k], (dist, id) ascending.  NaN rows propagate as NaN/-1. */
kgq_status kgq_merge_topk(kgq_ctx* ctx, int32_t n_parts, int32_t batch, int32_t k,
                          const float* in_dist, const int32_t* in_id, float* out_dist,
                          int32_t* out_id, kgq_stream stream);
/* N2: the all-gather of a9 fused into the top-k kernel over peer memory
 * (NVLink P2P on a multi-GPU node; any device memory for virtual shards on one GPU).
 *   kgq_peer_bytes: size of the per-rank peer buffer for `world` ranks (-1 on bad arguments):
 *     flag uint32 [2][world][max_batch] (256-byte padded), then key uint64
 *     [2][world][max_batch][max_k] = (order key of dist << 32) | global id.
 *   kgq_set_peers: registers the device pointers (host array of `world` entries; each
 *     256-byte aligned, kgq_peer_bytes long, e.g. one symmetric-memory allocation per rank)
 *     of every rank's buffer, this context being `rank`; zero-fills its own buffer and its
 *     epoch (call on every rank, then barrier, before the next submit).  world = 0 turns the
 *     push off.  Invalidates captured submit graphs.
 *   With peers set, every kgq_submit / kgq_submit_host / kgq_submit_mixed starts a new epoch
 *   and its top-k writes each output row's k keys into slot (epoch & 1, rank, row) of EVERY
 *   rank's buffer, then releases the row's flag (= epoch) at system scope.  The local
 *   topk_dist / topk_id outputs are written as before.
 *   kgq_merge_peers: waits (acquire, per row) for all ranks' pushes of the current epoch and
 *     writes the merged global top-k (dist, id ascending; NaN sorts last with id -1) to device
 *     out_dist / out_id [batch, k].  Every rank must issue the same sequence of submits.  A
 *     rank that has not published a row within KGQ_PEER_TIMEOUT_MS (default 10000) is
 *     treated as empty and kgq_check_errors then returns KGQ_ESTATE naming it (no hang). */
int64_t kgq_peer_bytes(const kgq_ctx* ctx, int32_t world);
kgq_status kgq_set_peers(kgq_ctx* ctx, int32_t rank, int32_t world, void* const* peer_bufs);
kgq_status kgq_merge_peers(kgq_ctx* ctx, int32_t batch, int32_t k, float* out_dist, int32_t* out_id,
                           kgq_stream stream);
/* ---- multi-GPU data plane: the library's own NCCL communicator ------
 * One process (one context) per GPU.  NCCL is loaded at run time (the copy the process already
 * uses, else libnccl.so.2); without it these calls return KGQ_ENCCL and nothing else changes.
 *
 * kgq_query_range: the row split of a replicated batch in query-split mode (pure host): rank r
 *   owns rows [lo, hi) = [min(B, r c), min(B, r c + c)), c = ceil(B / world).
 * kgq_nccl_unique_id: ncclGetUniqueId into host id[128] (128 bytes).  Call on one rank, send the
 *   bytes to the others over any channel (e.g. torch.distributed broadcast), then every rank
 *   calls kgq_comm_init with them.
 * kgq_comm_init: ncclCommInitRank(world, id, rank) on cfg.device -- collective, every rank of the
 *   job calls it.  `split` selects the data plane of every later submit (kgq_submit,
 *   kgq_submit_host[_async], kgq_submit_mixed; all on the caller's stream, no host sync):
 *   KGQ_SPLIT_ENTITIES (BASELINE north_star: the 2M-entity table sharded): needs
 *     cfg.world_size == world and cfg.rank == rank.  The batch is replicated; each rank scores
 *     its entity shard, selects its local top-k, one ncclAllGather exchanges the W [batch, k]
 *     lists (distance and id, one NCCL group) and the merge kernel (a9) writes the GLOBAL top-k
 *     to the caller's outputs on every rank.  shard_dist, if given, is this shard's.
 *     kgq_rank_answers with KGQ_RANK_FILTERED reduces over the shards inside (all-reduce min
 *     of the answer distances, all-reduce sum of the counts).
 *   KGQ_SPLIT_QUERIES (small tables, e.g. FB15k-237: the operator chain dominates): needs
 *     cfg.world_size == 1 (every rank holds all entities).  The batch is replicated; each rank
 *     runs only its rows kgq_query_range(batch, world, rank) through the whole path and one
 *     ncclAllGather of the [rows, k] results gives every rank the whole batch's top-k.
 *     shard_dist must be NULL.  Error reports name the row within the rank's slice.
 *   Exclusive with kgq_set_peers (N2).  Invalidates captured submit graphs.  Errors: KGQ_ENCCL
 *   (the NCCL message), KGQ_EINVAL (shape / mode mismatch), KGQ_ESTATE (peers set, or already
 *   initialised).  kgq_check_errors also reports an asynchronous NCCL error (KGQ_ENCCL).
 * kgq_comm_destroy: ncclCommDestroy; submits are local again.  kgq_destroy calls it.          */
typedef enum { KGQ_SPLIT_ENTITIES = 0, KGQ_SPLIT_QUERIES = 1 } kgq_split;
kgq_status kgq_query_range(int32_t batch, int32_t world, int32_t rank, int32_t* lo, int32_t* hi);
kgq_status kgq_nccl_unique_id(uint8_t* id);
kgq_status kgq_comm_init(kgq_ctx* ctx, const uint8_t* id, int32_t world, int32_t rank, int32_t split);
kgq_status kgq_comm_destroy(kgq_ctx* ctx);

/* N1: filtered ranking of given answers (KGReasoning test protocol behind the
 * paper's MRR consistency check).  Query b's answer set (easy and hard, distinct
 * global ids) is ans_id[ans_off[b] .. ans_off[b+1]) (device int32 CSR, ans_off [batch+1],
 * n_ans = ans_off[batch], at most 2048 answers per query).  For answer a of query b:
 *   count[a] = #{entities e of THIS shard, e not in b's answer set : (dist_e, e) < (dist_a, a)}
 * (ties by ascending id, Q13); the filtered rank is 1 + the sum of count over all shards, and
 * MRR / Hits@k follow on the host.  ans_dist (device fp32 [n_ans]) carries dist_a:
 *   KGQ_RANK_LOCAL (single shard): ans_dist is written, then count.
 *   KGQ_RANK_DIST: writes ans_dist for answers inside this shard, +inf for the others
 *                  (min-reduce it across ranks); count is not touched.
 *   KGQ_RANK_COUNT: reads ans_dist (the reduced one), writes count.
 *   KGQ_RANK_FILTERED: writes the filtered RANK (1 + the sum over shards of count) into count:
 *                  one shard, or entity shards with a communicator (kgq_comm_init; the two
 *                  phases and their all-reduces run inside, on `stream`).
 * Runs the operator chain and the scorer like kgq_submit.  A query with more than 2048
 * answers makes kgq_check_errors() return KGQ_EINVAL. */
enum { KGQ_RANK_LOCAL = 0, KGQ_RANK_DIST = 1, KGQ_RANK_COUNT = 2, KGQ_RANK_FILTERED = 3 };
kgq_status kgq_rank_answers(kgq_ctx* ctx, int32_t s, int32_t batch, const int32_t* anchors,
                            const int32_t* rels, const int32_t* ans_off, const int32_t* ans_id,
                            int32_t n_ans, int32_t mode, float* ans_dist, int32_t* count,
                            kgq_stream stream);
/* MRR / Hits@k of filtered ranks (N1; KGReasoning averaging): ranks int32
 * [n_ans] (1-based, e.g. from KGQ_RANK_FILTERED) in the CSR layout of ans_off [batch+1];
 * hard uint8 [n_ans] marks the answers that are scored (the hard answers), NULL = all.  Writes
 * device fp64 metrics[5] = {MRR, Hits@1, Hits@3, Hits@10, number of queries averaged}: the mean
 * over queries with at least one scored answer of the per-query mean of 1/rank and [rank <= k].
 * Device pointers, asynchronous on `stream`, one kernel. */
kgq_status kgq_rank_metrics(kgq_ctx* ctx, int32_t batch, const int32_t* ans_off, const int32_t* ranks,
                            const uint8_t* hard, double* metrics, kgq_stream stream);
/* Synchronise `stream`; KGQ_ERANGE (message names query row and slot) if any submit since
 * the last check saw an out-of-range id, KGQ_ECUDA on an asynchronous CUDA error, KGQ_ENCCL on
 * an asynchronous error of the context's communicator.  KGQ_ERANGE also when a GEMM operand
 * reached the fp16x2 range (|x| >= 65504, see kgq_tensor_mmas_per_fma): that flag is kept per
 * device and process (any context's conversion on this device since the last check reports it),
 * and the affected results are not exact -- rerun with the bf16x3 build. */
kgq_status kgq_check_errors(kgq_ctx* ctx, kgq_stream stream);

/* ---- options -------------------------------------------------------------------------- */
/* KGQ_OPT_FUSED_TOPK (BetaE tensor-core scorer, k <= 16, no shard_dist, not
 * kgq_rank_answers): the scorer's epilogue keeps every query row's k smallest (distance, id) per
 * N stripe of the entity table and a merge kernel returns the top-k -- the [batch, N] distance
 * block is never written.  Values: KGQ_FUSED_OFF (always write the block; block-minima top-k),
 * KGQ_FUSED_ON (fuse whenever eligible), KGQ_FUSED_AUTO (default: fuse scorer launches of >= 8,192
 * query rows, where every stripe spans >= 16 tiles so the lists' warm-up amortises; measured,
 * DESIGN.md §7).  Results are identical either way (same distances, same (dist, id) order).
 * The environment KGQ_NO_FUSED_TOPK=1 makes OFF the default of new contexts.
 * Returns KGQ_EINVAL for an unknown option or value. */
typedef enum { KGQ_OPT_FUSED_TOPK = 1 } kgq_option;
typedef enum { KGQ_FUSED_OFF = 0, KGQ_FUSED_ON = 1, KGQ_FUSED_AUTO = 2 } kgq_fused_mode;
kgq_status kgq_set_option(kgq_ctx* ctx, int32_t option, int64_t value);

/* ---- introspection (parity / bench) ----------------------------------------------------- */
/* Tensor-core MMAs per useful fp32 multiply-add of the GEMMs in this build: 3 for the default
 * fp16x2 operand format (a_hi w_hi' + a_hi w_lo' + a_lo' w_hi, 2^11-scaled lo planes, |x| < 65504,
 * |w| < 32; out-of-range values make kgq_check_errors / kgq_finalize return KGQ_ERANGE), 6 for
 * the bf16x3 build libkgq_bf16x3.so (exact three-plane split, fp32 range).  The roofline divisor. */
int32_t kgq_tensor_mmas_per_fma(void);
/* Number of this library's kernels launched by the last submit/query_embedding call. */
int32_t kgq_last_launch_count(const kgq_ctx* ctx);
/* BetaE only: copy this shard's precomputed entity terms to device out fp32 [3, d, n_shard]
 * (C, U, V planes).  Parity aid for the fp64 precompute. */
kgq_status kgq_entity_terms(kgq_ctx* ctx, float* out, kgq_stream stream);
/* Stage timing with CUDA events recorded on the launching stream (bench roofline).  Stages:
 * 0 operator chain, 1 scorer operand prep, 2 entity scorer, 3 top-k, 4 dense layers (each
 * tcgen05 GEMM of the chain; nested inside stage 0). */
kgq_status kgq_profile_enable(kgq_ctx* ctx, int32_t on);
/* Summed device milliseconds ms[5], timed-region counts n[5] and algorithmic work work[5]
 * (may be NULL; dense: 2MNK FLOPs; scorer: FLOPs of the tensor-core BetaE contraction or FP32
 * lane instructions of the SIMT scorers) since the last read; synchronises, then resets. */
kgq_status kgq_profile_read(kgq_ctx* ctx, double* ms, int64_t* n, double* work);
/* In-kernel launch spans of the tcgen05 GEMM (bench roofline taken from the headline pass
 * itself, no events between kernels).  With it on, every GEMM launch stamps %globaltimer in
 * its first CTA (after the programmatic-dependent-launch wait) and its last CTA, and the last
 * CTA adds the span to a device sum per stage: 0 = dense layers of the operator chain, 1 = the
 * BetaE tensor-core scorer.  Cost: three atomics per CTA.  Toggling re-captures the submit
 * graphs once (the accounting pointer is a kernel argument). */
kgq_status kgq_ktime_enable(kgq_ctx* ctx, int32_t on);
/* Summed spans in ms[2] and launch counts n[2] since the last read; synchronises the device,
 * then resets. */
kgq_status kgq_ktime_read(kgq_ctx* ctx, double* ms, int64_t* n);
/* The launch spans themselves (appended by every GEMM launch while kgq_ktime_enable is on, up to
 * 65,536): copies min(count, cap) entries of three uint64 {start ns, end ns, stage} (%globaltimer,
 * one clock per device, so the logs of several contexts on one GPU can be merged) to host out,
 * returns the count logged since the last call (-1 on error); synchronises, then empties the
 * log.  The union of the spans is the time the GPU spent in GEMMs, also under concurrent
 * streams. */
int64_t kgq_ktime_log(kgq_ctx* ctx, uint64_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* KGQ_H */
