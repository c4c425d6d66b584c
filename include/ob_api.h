/*
 * ob_api.h -- C ABI of libomega_b200.so, the B200-native Omega serving hot path.
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams travel as uint64 handles).  Every call returns an ob_status;
 * ob_last_error() gives the thread-local message of the last failure.
 *
 * Each entry point replaces one piece of the reference's Python serving API
 * (paths relative to /root/reference/pkg/src/gnnserve):
 *
 *   ob_engine_create      ServingEngine.__init__ + ServeConfig      runtime.py:62-82, 258-288
 *   ob_load_graph         GraphDataset / build_csr (device resident) graphstore.py:40-88
 *   ob_load_pe            PeStore (device resident)                 graphstore.py:122-171
 *   ob_load_model         ModelSpec + Weights (weight_matrix_names)  models.py:47-133
 *   ob_precompute_pe      precompute_embeddings                      graphstore.py:330-365
 *   ob_read_pe            PeStore.layers[l-1] readback               graphstore.py:143-152
 *   ob_serve              ServingEngine.serve -> (emb, breakdown)    runtime.py:308-358
 *   ob_serve_device       same, request already in device memory     (bench: HBM-resident inputs)
 *   ob_last_plan          RecomputationPlan / CandidateSet (parity)  policy.py:38-61, 64-135
 *   ob_last_block_sizes   ComputationBlock sizes (parity hook)       compgraph.py:33-57
 *   ob_last_block         ComputationBlock arrays (parity hook)      compgraph.py:33-57
 *   ob_nccl_unique_id     bootstrap for one-process-per-GPU CGP      collectives.py:94-137 (World)
 *   ob_reserve / ob_profile / ob_profile_read   measurement support (no reference counterpart;
 *                         the reference only has perf_counter phase timers, runtime.py:312-334)
 *
 * Status -> Python exception mapping:
 *   OB_EINVAL -> ValueError, OB_ENOTFOUND -> KeyError, OB_ECOMM -> TransportError,
 *   OB_ECUDA / OB_ENOMEM / OB_ESTATE -> RuntimeError.
 */
#ifndef OB_API_H
#define OB_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OB_API_VERSION 1

typedef struct ob_engine ob_engine;

enum ob_status {
  OB_OK = 0,
  OB_EINVAL = 1,     /* bad argument / request / config          -> ValueError     */
  OB_ENOTFOUND = 2,  /* row not stored locally                    -> KeyError       */
  OB_ECOMM = 3,      /* collective failure                        -> TransportError */
  OB_ECUDA = 4,      /* CUDA runtime error                        -> RuntimeError   */
  OB_ENOMEM = 5,     /* device allocation failure                 -> RuntimeError   */
  OB_ESTATE = 6      /* call out of order (e.g. serve before load) -> RuntimeError  */
};

/* ServeConfig.strategy (runtime.py:51).  "sampled" is build_sampled
   (compgraph.py:248-284): build_full_k_hop with each destination's sources cut to
   fanouts[l-1] by numpy's SeedSequence(seed, (l, v)) -> PCG64 -> choice stream,
   reproduced per destination on the device (fanouts <= OB_MAX_FANOUT). */
enum ob_strategy { OB_STRATEGY_FULL = 0, OB_STRATEGY_SAMPLED = 1, OB_STRATEGY_SRPE = 2, OB_STRATEGY_SRPE_CGP = 3 };
#define OB_MAX_FANOUT 200
#define OB_MAX_LAYERS 8

/* ServeConfig.policy (policy.py:29-32): ratio (policy.py:77-81) and importance
   (policy.py:84-107; under srpe-cgp the per-partition numerators are summed in
   rank order, runtime.py:168-175). */
/* ratio: query-edge ratio (policy.py:77-81); is: importance (policy.py:84-107);
 * random: default_rng(seed).permutation of the candidates (policy.py:122-124) */
enum ob_policy { OB_POLICY_RATIO = 0, OB_POLICY_IS = 1, OB_POLICY_RANDOM = 2 };

/* Layer kinds use the reference's on-disk tags (models.py:36 KIND_TAGS). */
enum ob_kind {
  OB_KIND_GCN = 0,
  OB_KIND_SAGE_MEAN = 1,
  OB_KIND_GAT = 2,
  OB_KIND_POWER_MEAN = 3,
  OB_KIND_MOMENTS = 4,
  OB_KIND_SAGE_MAX = 5
};

typedef struct {
  int32_t device;          /* CUDA ordinal                                       */
  int32_t strategy;        /* enum ob_strategy                                   */
  double gamma;            /* recompute budget in [0, 1]                         */
  int32_t policy;          /* enum ob_policy                                     */
  int32_t num_partitions;  /* CGP partitions P (1 for centralized strategies)    */
  int32_t rank;            /* this process's partition when nccl_id != NULL      */
  uint64_t seed;           /* partition hash seed (ServeConfig.seed)             */
  uint64_t stream;         /* cudaStream_t to launch on; 0 = engine-owned stream */
  const void* nccl_id;     /* 128-byte ncclUniqueId: one process per GPU / rank;
                              NULL with P > 1 = all P partitions on this device  */
  int32_t num_fanouts;     /* sampled: one fanout per layer (== k), else 0      */
  int32_t fanouts[OB_MAX_LAYERS]; /* ServeConfig.fanouts, outermost hop first     */
} ob_config;

typedef struct {
  int32_t kind;     /* enum ob_kind */
  int32_t in_dim;
  int32_t out_dim;
  float p;          /* power_mean exponent */
  int32_t n;        /* moments order */
} ob_layer;

/* LatencyBreakdown (runtime.py:85-95) plus device-side counters. */
typedef struct {
  double fetch_ms;          /* selection + graph construction (device time)          */
  double transfer_ms;       /* fetch_bytes / bandwidth, as the reference models it   */
  double compute_ms;        /* per-layer execution (device time)                     */
  int64_t collective_bytes; /* CGP: bytes moved between GPUs for the request, all ranks
                               (NVLink exchange: from the request's actual sizes)      */
  int64_t fetch_bytes;      /* graph_fetch_bytes (runtime.py:105-120)                */
  int64_t num_candidates;
  int64_t num_targets;
  int64_t h2d_bytes;        /* request bytes copied host -> device                   */
  int64_t d2h_bytes;        /* result bytes copied device -> host                    */
  double total_device_ms;   /* whole request on the device                           */
  int64_t allgather_bytes;  /* CGP: the all-gather-of-source-rows alternative,
                               sum_l (P-1) S_l row_bytes_l           */
} ob_breakdown;

const char* ob_last_error(void);
int ob_version(void);

int ob_engine_create(const ob_config* cfg, ob_engine** out);
int ob_engine_destroy(ob_engine* e);

/* In-CSR graph: offsets[N+1], neighbours[E] (sources ascending per destination
 * after load; duplicates kept), features N x F row-major float32. */
int ob_load_graph(ob_engine* e, int64_t num_nodes, const int64_t* in_offsets,
                  const int64_t* in_neighbors, int64_t num_edges, const float* features,
                  int32_t feature_dim);

/* Device-generated synthetic graph (the power law of
 * workload.py:119-168, drawn on the GPU -- not the numpy stream): N nodes,
 * average in-degree avg_degree, degree exponent, F-wide N(0,1) features.  An
 * NCCL-mode CGP engine builds only its rank's share (source-split CSR, owned
 * feature rows); other engines build the whole in-CSR.  Replaces
 * ob_load_graph for graphs that cannot exist on the host. */
int ob_generate_graph(ob_engine* e, int64_t num_nodes, double avg_degree, double exponent,
                      int32_t feature_dim, uint64_t seed);
/* Synthetic N(0,1) stored embeddings for layer `layer` (rows this engine stores). */
int ob_generate_pe(ob_engine* e, int32_t layer, int32_t dim, uint64_t seed);
/* Sizes of the loaded graph: global nodes/edges, rows and edges held here. */
int ob_graph_info(ob_engine* e, int64_t* num_nodes, int64_t* num_edges, int64_t* local_rows,
                  int64_t* local_edges);
/* Copy out the whole in-CSR (partition < 0) or partition p's source-split CSR,
 * plus the global in-degrees; any pointer may be NULL. */
int ob_graph_csr(ob_engine* e, int32_t partition, int64_t* offsets, int64_t* neighbors,
                 int32_t* in_degree);
/* Copy out rows of the feature table (table 0) or stored layer `table` for
 * global ids; OB_ENOTFOUND for rows another rank stores. */
int ob_read_rows(ob_engine* e, int32_t table, int64_t n, const int64_t* ids, float* out);

/* Stored embeddings for layer `layer` (1-based), N x dim float32. */
int ob_load_pe(ob_engine* e, int32_t layer, const float* rows, int64_t num_rows, int32_t dim);

/* k layers; mats lists every matrix in weight_matrix_names order per layer
 * (gcn: w; sage_*: w_self, w_neigh; gat: w, a_src, a_dst; power_mean/moments:
 * w_self, w), each row-major float32 in_dim x out_dim (a_* are out_dim). */
int ob_load_model(ob_engine* e, int32_t k, const ob_layer* layers, const float* const* mats);

/* precompute_embeddings on the device: PE layers 1..k-1 from the loaded graph. */
int ob_precompute_pe(ob_engine* e);
int ob_read_pe(ob_engine* e, int32_t layer, float* out_rows);

/* Serve one query batch.  Host pointers: query_features B x F, edges m x 2
 * int64 (src, dst) global ids with queries numbered N..N+B-1.  out: B x H_k
 * float32 in query-id order.  bd may be NULL.  Under CGP with one process per
 * GPU every rank calls this with the full request; rank 0 receives `out`. */
int ob_serve(ob_engine* e, int32_t num_queries, const float* query_features, int64_t num_edges,
             const int64_t* edges, float* out, ob_breakdown* bd);
/* Same with int32 (src, dst) pairs (valid whenever N + B < 2^31, which the engine
 * requires anyway): half the request's PCIe bytes; widened on the device. */
int ob_serve_i32(ob_engine* e, int32_t num_queries, const float* query_features, int64_t num_edges,
                 const int32_t* edges, float* out, ob_breakdown* bd);

/* Same with device pointers (request already resident in HBM); `out` is a
 * device pointer.  Work is enqueued on the engine stream; with bd == NULL the
 * call does not synchronise (errors are reported by the next call). */
int ob_serve_device(ob_engine* e, int32_t num_queries, const float* d_query_features,
                    int64_t num_edges, const int64_t* d_edges, float* d_out, ob_breakdown* bd);

/* Pipelined host path (production serving loop): submit copies the request's
 * host inputs to one of four device staging slots on a copy stream and enqueues
 * the request; the rows come back on a second copy stream.  While request t
 * runs, request t+1's inputs cross PCIe and request t-1's rows return (with
 * request lanes, slot s runs on lane s % lanes).  At most four requests are
 * outstanding (OB_ESTATE otherwise); ob_serve_wait(ticket)
 * blocks until request `ticket`'s rows are in its `out` and reports its errors
 * and breakdown (compute_ms = device time of the request).  Host buffers must
 * stay valid until the wait; pinned buffers give full overlap. */
int ob_serve_submit(ob_engine* e, int32_t num_queries, const float* query_features, int64_t num_edges,
                    const int64_t* edges, float* out, int64_t* ticket);
int ob_serve_submit_i32(ob_engine* e, int32_t num_queries, const float* query_features, int64_t num_edges,
                        const int32_t* edges, float* out, int64_t* ticket);
int ob_serve_wait(ob_engine* e, int64_t ticket, ob_breakdown* bd);

/* Request lanes: with n > 1, consecutive ob_serve_device calls (and the
 * slots of ob_serve_submit) rotate over n independent request workspaces on n
 * streams, so one request's graph construction (many small
 * latency-bound kernels) overlaps the other's aggregation gathers.  Lane 0 uses
 * the engine stream; ob_lanes_fork orders the other lanes after lane 0's
 * enqueued work and ob_lanes_join orders lane 0 after theirs (bracket a batch
 * of device serves with them to time it on lane 0's stream).  Not for CGP. */
int ob_set_lanes(ob_engine* e, int32_t n);
int ob_lanes_fork(ob_engine* e);
int ob_lanes_join(ob_engine* e);

/* Parity hooks over the last served request (synchronising). */
int ob_last_plan(ob_engine* e, int64_t* num_candidates, int64_t* num_targets, int64_t* cand_ids,
                 int64_t* cand_nq, int64_t* cand_total, double* cand_scores, int64_t* targets);
int ob_last_block_sizes(ob_engine* e, int32_t partition, int32_t layer, int64_t* num_src,
                        int64_t* num_dst, int64_t* num_edges);
int ob_last_block(ob_engine* e, int32_t partition, int32_t layer, int64_t* src_ids,
                  int64_t* dst_ids, int64_t* edge_src, int64_t* edge_dst, uint8_t* bind_kind,
                  int32_t* bind_pe_layer, int64_t* src_degree, int64_t* dst_self_src);

/* Size the request workspace for batches up to (num_queries, num_edges) so
 * later serves never allocate, and plan every later request at that edge
 * bound so all of them replay one captured graph (serving warm-up). */
int ob_reserve(ob_engine* e, int32_t num_queries, int64_t num_edges);

/* In-library kernel profiler: CUDA events around the hot launches on the
 * engine stream.  enable != 0 resets the records.  ob_profile_read sums the
 * launches of one class since enabling: device time, count, algorithmic bytes
 * (aggregation: 4*E + 4*w*S + 4*pw*items; finalize: partials in + rows out;
 * gemm: operands + result) and flops (gemm; for the aggregation class this slot returns the
 * gathered row bytes 4*w*E, i.e. the traffic the gather actually serves). */
enum ob_prof_class { OB_PROF_AGG = 0, OB_PROF_GEMM = 1, OB_PROF_FINALIZE = 2, OB_PROF_BUILD = 3,
                     OB_PROF_SELECT = 4, OB_PROF_RESOLVE = 5, OB_PROF_REQUEST = 6, OB_PROF_CSR = 7,
                     OB_PROF_COMM = 8 };
int ob_profile(ob_engine* e, int32_t enable);
/* Request graphs: by default each (B, edge-count bucket) request shape is
 * captured once into a CUDA graph and replayed (the request itself is read
 * from a device parameter block, so any request of that shape reuses it).
 * enable == 0 launches every stage eagerly; profiling always runs eagerly.
 * The environment variable OB_NO_GRAPHS=1 sets the default to off. */
int ob_set_graphs(ob_engine* e, int32_t enable);
int ob_profile_read(ob_engine* e, int32_t kernel_class, double* total_ms, int64_t* launches,
                    double* alg_bytes, double* flops);

/* Partition map of a CGP engine (owner per node), for parity checks. */
int ob_partition_owner(ob_engine* e, int64_t* owner);

/* Kernel-launch counter (own kernels only), for the bench's gpu_launches. */
int64_t ob_launch_count(ob_engine* e);

/* Fill a 128-byte buffer with a fresh ncclUniqueId (rank 0 of a CGP group). */
int ob_nccl_unique_id(void* out128);

#ifdef __cplusplus
}
#endif

#endif /* OB_API_H */
