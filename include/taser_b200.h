/*
 * taser_b200.h — C-ABI of the B200-native TASER mini-batch-generation path.
 *
 * This is the drop-in boundary.  The reference (`tgadapt`, /root/reference/pkg)
 * is Python + numba with no FFI of its own; every entry point below replaces
 * one reference function (cited file:line, paths relative to
 * pkg/src/tgadapt/).  The Python host mirror (paper_2402_05396_b200/*.py) binds
 * these symbols with ctypes and keeps the reference's Python signatures.
 *
 * Conventions
 *  - Every buffer argument is a DEVICE pointer owned by the caller unless the
 *    comment says "host".  The library never frees caller memory.  It may
 *    allocate stream-ordered temporaries (cudaMallocAsync) and frees them on
 *    the same stream before returning.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on
 *    that stream unless marked SYNC (those read results back to the host).
 *  - Return value: TG_OK (0) or a negative status; the shim maps them to the
 *    reference's exception types.  tg_last_error() gives the message
 *    (thread-local).
 *  - Index widths: node ids / eids in query and output arrays are int64 and
 *    timestamps f64, exactly the reference dtypes.  The device T-CSR stores
 *    neighbor ids and eids as int32 (2E < 2^31 for every configured shape).
 */
#ifndef TASER_B200_H
#define TASER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 4  /* 4: tg_graph coarse index fields, batched finder, multi-segment K5, graph launch */

enum tg_status {
  TG_OK = 0,
  TG_EVALUE = -1,   /* ValueError   (finder.py:167-172, 200-202)           */
  TG_EINDEX = -2,   /* IndexError   (cache.py:76-77)                       */
  TG_EDATA = -3,    /* DataError    (graph.py:20, 103-128)                 */
  TG_ECONFIG = -4,  /* ConfigError  (sampler.py:36-40)                     */
  TG_ECUDA = -5,    /* RuntimeError: a CUDA call failed                    */
  TG_EFLOAT = -6    /* FloatingPointError (sampler.py:202-203)             */
};

enum tg_policy { TG_RECENT = 0, TG_UNIFORM = 1 };

/* Global row index of local query i: i < split ? base0 + i : base1 + (i - split).
 * Keeps the counter RNG keyed by the reference's row index when roots are
 * sharded across GPUs (finder.py:99 keys draws by the query's row). */
typedef struct tg_rowmap {
  int64_t split;
  int64_t base0;
  int64_t base1;
} tg_rowmap;

/* Device T-CSR (graph.py:50-91 TemporalGraph.tcsr_*). */
typedef struct tg_graph {
  const int64_t* offsets;  /* [V+1]                                        */
  const int32_t* nbr;      /* [2E] peer node per adjacency entry            */
  const double* adj_ts;    /* [2E] timestamp per entry, per-node ascending  */
  const int32_t* adj_eid;  /* [2E] event id per entry                       */
  int64_t num_nodes;
  int64_t num_adj;
  /* optional coarse time index (tg_tcsr_coarse; NULL: none): every
   * 2^coarse_shift-th timestamp of each node's list, coarse_ts[coarse_off[v]
   * + i] = adj_ts[offsets[v] + (i << coarse_shift)] -- small enough to stay
   * in L2, so a hub's pivot search costs L2 probes + one short DRAM sweep */
  const int64_t* coarse_off; /* [V+1] */
  const double* coarse_ts;
  int32_t coarse_shift;
  int32_t reserved;
} tg_graph;

/* Feature tiers.  Row r of the logical table (eid or node id) is served from
 *   hot   + slot*hot_ld   if cache slot_of[r] >= 0 and hot != NULL,
 *   peers[r / shard_rows] + (r % shard_rows)*ld   if n_peers > 0,
 *   table + r*ld          otherwise.
 * peers[] entries may be local or peer-mapped (tg_ipc_open) device pointers;
 * each must be 16-byte aligned and use the row stride ld.
 * Values never depend on the tier (cache.py:85: features always come from the
 * full array), so parity is unaffected by the placement. */
typedef struct tg_feat_store {
  const float* table;
  const float* hot;
  const float* const* peers; /* device array of n_peers device pointers */
  int64_t shard_rows;
  int32_t n_peers;
  int32_t d;                 /* feature width (floats)                  */
  int64_t ld;                /* row stride of table/peers (floats)      */
  int64_t hot_ld;            /* row stride of hot (floats)              */
  int64_t num_rows;
} tg_feat_store;

/* Edge-feature cache state (cache.py:32-55 CacheState). */
typedef struct tg_cache_dev {
  int32_t* slot_of;          /* [E]; >= 0 iff resident (CacheState.resident) */
  int32_t* counters;         /* [E]; per-epoch accesses (CacheState.counters) */
  unsigned long long* stats; /* [2]; hits, misses of the open epoch           */
  int64_t num_edges;
} tg_cache_dev;

/* One neighbor-finding pass over a query batch, fused with the
 * materialisation of training.py:246-252, the hop expansion of
 * training.py:311-314 and (optionally) the edge-feature slice of
 * training.py:207-221 through the cache (cache.py:72-86).
 * Every output pointer may be NULL (not written). */
typedef struct tg_find_args {
  const int64_t* qv;      /* [B] query nodes                                */
  const double* qt;       /* [B] query times                                */
  int64_t B;
  int32_t m;              /* budget                                        */
  int32_t policy;         /* TG_RECENT | TG_UNIFORM                        */
  uint64_t seed;          /* finder seed (training.py:242)                 */
  tg_rowmap rows;
  int64_t* idx;           /* [B,m] adjacency positions, -1 fill (finder.py:173) */
  int64_t* cnt;           /* [B]                                            */
  int64_t* ids;           /* [B,m] neighbor ids, 0 on padded slots          */
  int64_t* eids;          /* [B,m] event ids, 0 on padded slots             */
  double* dts;            /* [B,m] t - ts, 0.0 on padded slots              */
  double* tss;            /* [B,m] ts, 0.0 on padded slots                  */
  uint8_t* mask;          /* [B,m] slot < cnt                               */
  int64_t* next_v;        /* [B + B*m] next-hop nodes  [targets || children] */
  double* next_t;         /* [B + B*m] next-hop times  [t || t - dt]          */
  float* feat_out;        /* [B*m, feat_ld] edge rows, +0.0 on padded slots  */
  int64_t feat_ld;
  unsigned long long* valid_count; /* += sum(cnt) (sampled neighbors)      */
  int64_t* window;        /* [B] pivot - lo = #entries with ts < t (finder.py:152-155) */
  const uint64_t* seed_ptr; /* device; when non-NULL the finder seed is *seed_ptr (not `seed`),
                               so a CUDA-graph replay of a step takes each batch's seed from
                               memory the caller refreshes before the replay */
} tg_find_args;

int tg_abi_version(void);
/* Replay an executable CUDA graph (cudaGraphExec_t, e.g. from torch's
 * CUDAGraph.raw_cuda_graph_exec()) on `stream` via cuGraphLaunch. */
int tg_graph_launch(void* graph_exec, void* stream);
/* cuGraphUpload: stage an executable graph on the device before its first launch. */
int tg_graph_upload(void* graph_exec, void* stream);
const char* tg_last_error(void);
/* Number of kernels this library has launched since load (host counter). */
unsigned long long tg_launch_count(void);
/* SM count of the current device (grid sizing), SYNC. */
int tg_device_sms(int* out);

/* ---- K1: T-CSR construction (graph.py:94-152 build_graph) ---------------- */
/* SYNC.  Validates the event arrays like graph.py:103-110 and reports
 * host_info[0] = max node id (or -1 if E == 0), host_info[1] = 1 if ts is
 * already non-decreasing (so the stable ts sort is the identity). */
int tg_tcsr_check(const int64_t* src, const int64_t* dst, const double* ts, int64_t E,
                  int64_t* host_info, void* stream);
/* Stable sort of the events by ts (graph.py:112-113), both-direction entries
 * ordered by (node, ts, eid) (graph.py:131-137) and CSR offsets
 * (graph.py:139-141).  order[E] receives the stable ts permutation (may be
 * NULL); src_s/dst_s/ts_s the events in eid order.  ts_sorted = host_info[1]
 * of tg_tcsr_check (skips the identity sort). */
int tg_tcsr_build(const int64_t* src, const int64_t* dst, const double* ts, int64_t E,
                  int64_t V, int32_t ts_sorted, int64_t* order, int64_t* src_s, int64_t* dst_s, double* ts_s,
                  int64_t* offsets, int32_t* nbr, double* adj_ts, int32_t* adj_eid,
                  void* stream);
/* Coarse time index of a built T-CSR (see tg_graph.coarse_*): coarse_off
 * [V+1] and coarse_ts [(num_adj >> shift) + V] (capacity), 1 <= shift <= 16.
 * Does not change any result: the finder's pivot is the same strict-<
 * count (finder.py:69-77), found through the index. */
int tg_tcsr_coarse(const tg_graph* g, int32_t shift, int64_t* coarse_off, double* coarse_ts, void* stream);
/* out[i, :] = in[order[i], :] for f32 rows (graph.py:118 edge_features[order]). */
int tg_gather_rows_f32(const float* in, int64_t in_ld, const int64_t* order, int64_t n,
                       int32_t d, float* out, int64_t out_ld, void* stream);

/* ---- K2+K3(+K4/K5): finder (finder.py:85-149, 162-179) -------------------- */
/* store/cache may be NULL; feat_out requires store.  m <= 2048. */
int tg_find(const tg_graph* g, const tg_find_args* a, const tg_feat_store* store,
            const tg_cache_dev* cache, void* stream);
/* nb finder passes of one layer (same m and policy, feat_out NULL) as one
 * launch per 16 of them: the per-layer finder of several mini-batches
 * (training.py:241-253 for each), bit-identical to nb tg_find calls. */
int tg_find_batch(const tg_graph* g, const tg_find_args* args, int32_t nb, const tg_cache_dev* cache,
                  void* stream);

/* ---- K4+K5: feature slice through the cache (training.py:207-230) ---------- */
/* For n slots: rows[i] valid iff mask==NULL or mask[i]; valid rows are copied
 * from the store (and counted by the cache when cache != NULL, cache.py:78-82);
 * invalid rows are +0.0 (mask_mode 0, edge rows, training.py:218) or
 * row(ids[i]) * 0.0 (mask_mode 1, node rows, training.py:227-229). */
int tg_lookup_gather(const int64_t* ids, const uint8_t* mask, int64_t n,
                     const tg_feat_store* store, const tg_cache_dev* cache, int32_t mask_mode,
                     float* out, int64_t out_ld, void* stream);
/* K5 alone: the row copy of tg_lookup_gather without cache accounting
 * (training.py:217-219 / 227-229 layout).  slot_of (may be NULL) routes rows
 * resident in the cache to store->hot. */
int tg_gather_rows(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                   const int32_t* slot_of, int32_t mask_mode, float* out, int64_t out_ld, void* stream);

/* K5 over several row lists in ONE launch per 32 of them (e.g. every layer of a mini-batch:
 * training.py:264-267 for each layer of :297-315).  Segment i copies rows
 * ids[0..n) (valid iff mask == NULL or mask[j]) to out + j*out_ld; all
 * segments share the store, the cache's slot map and out_ld.  Same row
 * semantics as tg_gather_rows. */
typedef struct tg_gather_seg {
  const int64_t* ids;
  const uint8_t* mask;
  int64_t n;
  float* out;
} tg_gather_seg;
int tg_gather_rows_multi(const tg_gather_seg* segs, int32_t nseg, const tg_feat_store* store,
                         const int32_t* slot_of, int32_t mask_mode, int64_t out_ld, void* stream);
/* cache.py:72-86 lookup(): count every id, hits[i] = resident[ids[i]];
 * feat_out (may be NULL) receives all rows. */
int tg_cache_lookup(const int64_t* ids, int64_t n, const tg_cache_dev* cache, uint8_t* hits,
                    const tg_feat_store* store, float* feat_out, int64_t out_ld, void* stream);
/* SYNC.  Range check for lookup (cache.py:76-77): TG_EINDEX if any id is
 * outside [0, num_edges). */
int tg_check_range(const int64_t* ids, int64_t n, int64_t limit, void* stream);

/* Selection gather + hop expansion after K8 (training.py:281-291, 311-314):
 * sel_*[b,k] = cand_*[b, selected[b,k]] (0 / 0.0 where !sel_mask); next_v/t
 * (may be NULL) = [qv || sel_ids], [qt || qt[b] - sel_dts]. */
int tg_select_expand(const int64_t* ids, const int64_t* eids, const double* dts, const int64_t* selected,
                     const uint8_t* sel_mask, const int64_t* qv, const double* qt, int64_t B, int32_t m, int32_t n,
                     int64_t* sel_ids, int64_t* sel_eids, double* sel_dts, int64_t* next_v, double* next_t,
                     void* stream);

/* ---- K6: epoch-boundary replacement (cache.py:89-118) --------------------- */
/* SYNC.  Top-k of the touched counters by (count desc, eid asc); replace the
 * resident set iff overlap < epsilon; reset counters and stats.  When
 * store != NULL && hot != NULL the hot-tier rows are refilled from the cold
 * tier.  host_out[0] = replaced, [1] = overlap, [2] = touched, [3] = selected. */
int tg_cache_replace(const tg_cache_dev* cache, int64_t k, int64_t epsilon,
                     const tg_feat_store* store, float* hot, int64_t hot_ld,
                     int64_t* host_out, void* stream);
/* SYNC.  Per-edge key order used by the clairvoyant oracle (cache.py:89-104):
 * writes into topk_mask[E] (uint8) the top-k touched entries of `counts`. */
int tg_topk_mask(const int32_t* counts, int64_t E, int64_t k, uint8_t* topk_mask,
                 int64_t* host_selected, void* stream);


/* ---- K7: adaptive-sampler scoring (encoders.py:152-200, mixer.py:31-51,
 *      sampler.py:69-135, autodiff.py:421-464) ------------------------------ */
enum tg_decoder { TG_DEC_LINEAR = 0, TG_DEC_GAT = 1, TG_DEC_GATV2 = 2, TG_DEC_TRANS = 3 };

/* Sampler parameters resident on the device, all in `dtype` (0 f32, 1 f64),
 * row-major exactly as the reference ParamStore holds them (params.py:24-61;
 * names in the comments).  Unused decoder weights may be NULL. */
typedef struct tg_score_model {
  int32_t dtype;
  int32_t decoder;   /* tg_decoder (SamplerConfig.decoder, sampler.py:29-40)     */
  int32_t m;         /* candidate scope (<= 64)                                   */
  int32_t F;         /* enc_dim = d_feat = d_time = d_freq (RunConfig.enc_dim)    */
  int32_t d_v, d_e;  /* node / edge feature widths (0 = absent)                   */
  int32_t d_enc;     /* encoded_width (encoders.py:116-119)                       */
  int32_t d_tv;      /* target_width (encoders.py:122-123)                        */
  int32_t gemm_path; /* f32 GEMMs: 0 = tcgen05 3xTF32 tensor cores, 1 = CUDA-core FFMA */
  double slope;      /* SamplerConfig.negative_slope                              */
  const void *W_node, *W_edge;                  /* encoder/W_node [d_v,F], W_edge [d_e,F] */
  const void *ln1_g, *ln1_b, *Wc1, *bc1, *Wc2, *bc2;   /* sampler/mixer/...          */
  const void *ln2_g, *ln2_b, *Wt1, *bt1, *Wt2, *bt2;
  const void* w_linear;                         /* sampler/w_linear [d_enc,1]        */
  const void *W_gat, *a_gat;                    /* sampler/W_gat [d,d], a_gat [2d,1] */
  const void *W_gatv2, *a_gatv2;                /* [2d,d], [d,1]                     */
  const void *W_trans_target, *W_trans_nbr;     /* [d_tv,d], [d,d]                   */
  const double* omega;     /* [F] alpha^(-(i-1)/beta) (encoders.py:57-59)            */
  const double* fe_table;  /* [(m+1), F] freq_encode_array(0..m) (encoders.py:75-85) */
} tg_score_model;

/* Bytes of device workspace tg_score needs for B roots. */
int tg_score_workspace(const tg_score_model* model, int64_t B, size_t* bytes);
/* q, log_q [B, m] in model->dtype for the candidate block of B roots:
 * ids int64 [B,m], dts f64 [B,m], mask u8 [B,m]; node_rows / edge_rows f32
 * [B*m, d] (row stride *_ld floats; masked slots as training.py:218/227);
 * tgt_rows f32 [B, d_v] (target node rows, encoders.py:186). */
int tg_score(const tg_score_model* model, const int64_t* ids, const double* dts, const uint8_t* mask,
             const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld,
             const float* tgt_rows, int64_t tgt_ld, int64_t B, void* q, void* log_q, void* workspace,
             size_t ws_bytes, void* stream);

/* Sampler backward: parameter gradients of the scoring
 * network from dlogits = d loss / d logits [B, m] (model dtype; K10's
 * tg_logq_surrogate_grad output), through decode_policy (sampler.py:91-135),
 * mixer_transform (sampler.py:69-72, mixer.py:31-51) and the encoders
 * (encoders.py:152-200) -- ad.backward's vjps (autodiff.py:495) from the
 * logits down.  Same candidate-block inputs as tg_score.  Every non-NULL
 * gradient buffer (model dtype, the parameter's shape) is ACCUMULATED into
 * (+=, like .grad across a multi-layer loss, training.py:411-436); NULL
 * skips that parameter.  Forward intermediates are recomputed into the
 * workspace (tg_score_backward_workspace bytes). */
typedef struct tg_score_grads {
  void *W_node, *W_edge;
  void *ln1_g, *ln1_b, *Wc1, *bc1, *Wc2, *bc2;
  void *ln2_g, *ln2_b, *Wt1, *bt1, *Wt2, *bt2;
  void* w_linear;
  void *W_gat, *a_gat;
  void *W_gatv2, *a_gatv2;
  void *W_trans_target, *W_trans_nbr;
} tg_score_grads;
int tg_score_backward_workspace(const tg_score_model* model, int64_t B, size_t* bytes);
int tg_score_backward(const tg_score_model* model, const int64_t* ids, const double* dts, const uint8_t* mask,
                      const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld,
                      const float* tgt_rows, int64_t tgt_ld, int64_t B, const void* dlogits,
                      const tg_score_grads* grads, void* workspace, size_t ws_bytes, void* stream);

/* The same forward, stage by stage, behind the reference's own function
 * boundaries (the drop-ins for code that composes them itself); each stage
 * reads and writes caller tensors in the model dtype with their own row
 * strides.  Workspace: tg_score_stage_workspace bytes.  tg_score fuses the
 * four for the pipeline.
 *   tg_encode_neighborhood  encode_neighborhood_batch  encoders.py:152-183
 *                           z [B*m, d_enc]
 *   tg_encode_target        encode_target_batch        encoders.py:186-200
 *                           zt [B, d_tv] ([GeLU(x W_node) | TE(0) | FE(1)])
 *   tg_mixer_transform      mixer_transform            sampler.py:69-72
 *                           out [B*m, d_enc] = mixer(z) * mask
 *   tg_decode_policy        decode_policy              sampler.py:91-135
 *                           q, log_q [B, m]; z_raw read by gat / gatv2,
 *                           z_mixed by linear / trans, z_target by all but linear */
int tg_score_stage_workspace(const tg_score_model* model, int64_t B, size_t* bytes);
int tg_encode_neighborhood(const tg_score_model* model, const int64_t* ids, const double* dts, const uint8_t* mask,
                           const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld,
                           int64_t B, void* z, int64_t ldz, void* workspace, size_t ws_bytes, void* stream);
int tg_encode_target(const tg_score_model* model, const float* tgt_rows, int64_t tgt_ld, int64_t B, void* zt,
                     int64_t ldt, void* workspace, size_t ws_bytes, void* stream);
int tg_mixer_transform(const tg_score_model* model, const void* z, int64_t ldz, const uint8_t* mask, int64_t B,
                       void* out, int64_t ldo, void* workspace, size_t ws_bytes, void* stream);
int tg_decode_policy(const tg_score_model* model, const void* z_raw, int64_t ldr, const void* z_mixed, int64_t ldm,
                     const void* z_target, int64_t ldt, const uint8_t* mask, int64_t B, void* q, void* log_q,
                     void* workspace, size_t ws_bytes, void* stream);

/* Diagnostics for K7's tensor-core GEMM: C[M,N] = A[M,K] @ W[K,N] (+ bias[N])
 * with 3xTF32 tcgen05 MMAs (A rows 16-byte aligned, lda % 4 == 0). */
int tg_tc_gemm_workspace(int64_t M, int N, int K, size_t* bytes);
int tg_tc_gemm(const float* A, int64_t lda, int64_t M, int K, const float* W, int64_t ldw, int N,
               const float* bias, float* C, int64_t ldc, void* workspace, void* stream);

/* ---- GraphMixer aggregator forward (aggregators.py:58-71, 140-145;
 *      mixer.py:31-51; called at training.py:318-330) ------------------- */
/* Model parameters (ParamStore names model/time_w, model/time_b,
 * model/gmixer/...), row-major, all in `dtype` (0 f32, 1 f64). */
typedef struct tg_gmixer_model {
  int32_t dtype;
  int32_t n;          /* slots = the layer's selection width                */
  int32_t d_v, d_e;   /* node / edge feature widths (0 = absent)            */
  int32_t d_time;     /* ModelConfig.d_time                                 */
  int32_t gemm_path;  /* f32 channel MLP: 0 = tcgen05 3xTF32, 1 = FFMA       */
  const void *time_w, *time_b;                  /* [d_time]                  */
  const void *ln1_g, *ln1_b, *Wc1, *bc1, *Wc2, *bc2;   /* d_msg = d_v+d_e+d_time */
  const void *ln2_g, *ln2_b, *Wt1, *bt1, *Wt2, *bt2;   /* token MLP [n, n]      */
} tg_gmixer_model;
int tg_graphmixer_workspace(const tg_gmixer_model* model, int64_t B, size_t* bytes);
/* h [B, d_msg] (row stride h_ld, model dtype) = mean over slots of
 * mixer(messages); node_rows / edge_rows f32 [B*n, *] as the generator
 * writes them, dts f64 [B, n], mask u8 [B, n]. */
int tg_graphmixer_forward(const tg_gmixer_model* model, const float* node_rows, int64_t node_ld,
                          const float* edge_rows, int64_t edge_ld, const double* dts, const uint8_t* mask,
                          int64_t B, void* h, int64_t h_ld, void* workspace, size_t ws_bytes, void* stream);

/* ---- TGAT attention layer forward (aggregators.py:74-132, build_messages
 *      :58-71; training.py:333-356) ------------------------------------- */
typedef struct tg_tgat_layer {
  int32_t dtype;       /* 0 f32, 1 f64 (the model store dtype)                 */
  int32_t gemm_path;   /* f32: 0 = tcgen05 3xTF32, 1 = FFMA                      */
  int32_t d_in;        /* embedding width of targets / neighbors (layer 1: d_v) */
  int32_t d_e, d_time, d_out;
  int32_t s;           /* slots (<= 64)                                         */
  const void *time_w, *time_b;                      /* model/time_w, time_b    */
  const void *W_q, *b_s, *W_k, *b_k, *W_v, *b_v;    /* model/tgat{l}/...       */
} tg_tgat_layer;
int tg_tgat_workspace(const tg_tgat_layer* layer, int64_t B, size_t* bytes);
/* h [B, d_out] (stride h_ld) and tau [B, s] (may be NULL) in the layer dtype.
 * h_tgt [B, d_in] / h_nbr [B*s, d_in]: f32 feature rows when *_f32 != 0,
 * else the layer dtype (the previous layer's h). */
int tg_tgat_forward(const tg_tgat_layer* layer, const void* h_tgt, int64_t tgt_ld, int32_t tgt_f32,
                    const void* h_nbr, int64_t nbr_ld, int32_t nbr_f32, const float* edge_rows, int64_t edge_ld,
                    const double* dts, const uint8_t* mask, int64_t B, void* h, int64_t h_ld, void* tau,
                    void* workspace, size_t ws_bytes, void* stream);

/* ---- K8: sampling without replacement (sampler.py:138-176) ---------------- */
/* q/log_q: [B,m] f64 (dtype 1) or f32 (dtype 0).  The draw of round k for
 * global row g is PCG64 output number k*B_global + g of the stream whose state
 * is (state_hi, state_lo, inc_hi, inc_lo) (numpy random(B) per round).
 * jump_mul/jump_add: the LCG constants that advance the state by B_global
 * steps (host precomputed, 128-bit as hi/lo pairs). */
typedef struct tg_pcg64 {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint64_t jmul_hi, jmul_lo;   /* M^B_global mod 2^128            */
  uint64_t jadd_hi, jadd_lo;   /* inc*(M^B_global-1)/(M-1)        */
} tg_pcg64;
int tg_sample_wor(const void* q, const void* log_q, int32_t dtype, int64_t B, int32_t m,
                  int32_t n, const tg_pcg64* rng, tg_rowmap rows, int64_t* selected,
                  uint8_t* sel_mask, void* sel_log_q, void* stream);

/* ---- K10: surrogate-loss head of the sampler update (sampler.py:183-250,
 * training.py:409-436).  Float arrays in `dtype` (0 f32, 1 f64), row-major;
 * masks u8.  c, sel_mask: [B, n]; contrib: [B].  Reductions run in f64. ---- */
/* tgat_sample_coefficients (sampler.py:191-213): dL_dh [B, d] (row stride
 * dh_ld), tau [B, n], V [B, n, d].  TG_EFLOAT if an active row (contrib and at
 * least one pick) has lam <= 0, like the reference's FloatingPointError.
 * SYNC (reads the error flag back). */
int tg_tgat_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d, const void* dL_dh, int64_t dh_ld,
                          const void* tau, const void* V, const uint8_t* sel_mask, const uint8_t* contrib,
                          void* c, void* stream);
/* graphmixer coefficients as training.py:423-431 composes them: mu = msgs @
 * Wc1, w'_j = 1 + rowsum(Wt1 @ Wt2)_j, then graphmixer_sample_coefficients
 * (sampler.py:230-239).  msgs [B, n, d_msg] (slot row stride msg_ld), Wc1
 * [d_msg, d], Wt1 [n, ht], Wt2 [ht, n]. */
int tg_graphmixer_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d_msg, int32_t d, int32_t ht,
                                const void* dL_dh, int64_t dh_ld, const void* msgs, int64_t msg_ld, const void* Wc1,
                                const void* Wt1, const void* Wt2, const uint8_t* sel_mask, const uint8_t* contrib,
                                void* c, void* stream);
/* graphmixer_sample_coefficients (sampler.py:230-239) in its general form:
 * w_prime [n, d] (wp_bstride 0) or [B, n, d] (wp_bstride n*d), mu [B, n, d]. */
int tg_mixer_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d, const void* dL_dh, int64_t dh_ld,
                           const void* w_prime, int64_t wp_bstride, const void* mu, const uint8_t* sel_mask,
                           const uint8_t* contrib, void* c, void* stream);
/* loss = sum(c * selected_log_q) (sample_loss_*, sampler.py:216-227, 242-250)
 * and its gradient with respect to the scoring logits through index and
 * log_softmax_masked (autodiff.py:257-271, 447-464): dlogits [B, m] (dtype).
 * q / log_q / mask [B, m] as K7 produced them, selected [B, n] int64 (-1 pad).
 * row_loss [B] f64 scratch (may be NULL when loss is NULL); loss: one f64. */
int tg_logq_surrogate_grad(int32_t dtype, int64_t B, int32_t m, int32_t n, const void* q, const void* log_q,
                           const uint8_t* mask, const int64_t* selected, const uint8_t* sel_mask, const void* c,
                           void* dlogits, double* row_loss, double* loss, void* stream);

/* One Adam step over every tensor of the sampler's store (params.py:80-99,
 * update_sampler sampler.py:253-256), bit-identical to the reference's numpy
 * update.  p/m/v in `dtype`; g in g_dtype (0 f32, 1 f64; -1: no gradient,
 * the moments still decay).  bc1 = 1 - beta1**t, bc2 = 1 - beta2**t as the
 * host computes them.  `tensors` is a host array; SYNC. */
typedef struct tg_adam_tensor {
  void* p;
  const void* g;
  void* m;
  void* v;
  int64_t n;
  int32_t g_dtype;
} tg_adam_tensor;
int tg_adam_step(int32_t dtype, const tg_adam_tensor* tensors, int32_t count, double lr, double beta1,
                 double beta2, double eps, double bc1, double bc2, void* stream);

/* ---- K9: importance-weighted mini-batch selection (selector.py:46-61) ----- */
/* SYNC.  out[b] = sort(rng.choice(n, b, replace=False, p=scores/scores.sum()))
 * + base, bit-exact with numpy: the PCG64 stream (state, inc of `rng`; the
 * jump fields are unused) is consumed from its next output on, exactly as
 * Generator.choice does.  TG_EVALUE like numpy/selector.py: b > n, NaN or
 * negative probabilities, fewer non-zero entries than b.  host_draws (may be
 * NULL) receives the number of doubles consumed (to advance the caller's
 * generator). */
int tg_select_batch(const double* scores, int64_t n, int64_t b, const tg_pcg64* rng, int64_t base,
                    int64_t* out, int64_t* host_draws, void* stream);
/* SYNC.  scores[eids[i] - base] = sigmoid(logits[i]) + gamma (Eq. 10,
 * selector.py:56-61) with the device exp (within 1 ulp of numpy's); for a
 * repeated eid the last position wins (numpy fancy assignment); TG_EINDEX if
 * an eid is outside [base, base + n). */
int tg_update_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                     const double* logits, double gamma, void* stream);
/* SYNC.  The same scatter with finished values: scores[eids[i] - base] =
 * values[i] (the caller evaluated Eq. 10, e.g. with the reference's numpy
 * expression on host logits -- selector.py:61 -- so scores stay bit-exact). */
int tg_scatter_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                      const double* values, void* stream);

/* ---- event-file ingest (graph.py:159-205 ingest_events) ------------------ */
/* Device-resident file bytes -> events.  All SYNC.
 * tg_ingest_lines: host_info[0] = line terminators ("\n", "\r\n", lone
 *   "\r"), [1] = lines; ends (may be NULL) = terminator offsets in order.
 * tg_ingest_classify: per line isdata / field count nf / output row (prefix
 *   of isdata); host_info[0] = data lines, [1] = first data line or -1,
 *   [2] = its field count.
 * tg_ingest_parse: src/dst (int()), ts (float()), feats [rows, feat_ld] f32
 *   (float() then f32) for rows of `width` features; host_err[0] = first
 *   failing line (0-based, -1 if none), [1] = check: failing field index,
 *   or 0xFFEF too few fields, 0xFFF0 non-finite ts, 0xFFF1 width,
 *   0xFFF4 int outside int64.  A value of more than 19 significant digits
 *   whose rounding the device cannot settle is not an error (Python parses
 *   it): its line index goes to unsup[0..unsup_cap) and host_err[2] counts
 *   such lines, for the caller to re-parse on the host (ABI 2). */
int tg_ingest_lines(const char* text, int64_t nbytes, int64_t* ends, int64_t* host_info, void* stream);
int tg_ingest_classify(const char* text, int64_t nbytes, const int64_t* ends, int64_t nterm, int64_t nlines,
                       int* isdata, int* nf, int* row, int64_t* host_info, void* stream);
int tg_ingest_parse(const char* text, int64_t nbytes, const int64_t* ends, int64_t nterm, int64_t nlines,
                    const int* isdata, const int* nf, const int* row, int32_t width, int64_t* src, int64_t* dst,
                    double* ts, float* feats, int64_t feat_ld, int64_t* unsup, int64_t unsup_cap,
                    int64_t* host_err, void* stream);

/* ---- peer memory for the sharded feature table ------------- */
/* No reference counterpart (the reference is single-process): rank r exports
 * its shard, the other ranks map it and list it in tg_feat_store.peers, so K5
 * reads remote rows over NVLink inside the gather.  SYNC. */
int tg_ipc_handle_size(void);
/* handle_out (tg_ipc_handle_size() bytes) names the allocation containing
 * dptr; offset_out = dptr - allocation base. */
int tg_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out);
/* Map a handle exported by another process (base of its allocation). */
int tg_ipc_open(const void* handle, void** base_out);
int tg_ipc_close(void* base);
/* Enable direct access from the current device to peer_device (no-op if it
 * is the same device); can_access = cudaDeviceCanAccessPeer. */
int tg_peer_access(int peer_device, int* can_access);

/* ---- synthetic shapes (bench inputs) ------------------------ */
/* Events e in [e0, e0+n): src = node_at_rank[lower_bound(cdf, u1)], dst uniform,
 * ts per ts_mode (0 sorted-uniform over span, 1 tie-heavy floor, 2 integer 1..E). */
int tg_synth_events(int64_t e0, int64_t n, int64_t E, int64_t V, uint64_t seed,
                    const double* zipf_cdf, const int64_t* node_at_rank, int32_t ts_mode,
                    double span, int64_t* src, int64_t* dst, double* ts, void* stream);
/* rows [r0, r0+n) of a hash-defined f32 table in [-1, 1). */
int tg_synth_features(int64_t r0, int64_t n, int32_t d, uint64_t seed, float* out,
                      int64_t ld, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TASER_B200_H */
