/*
 * figaro_cuda.h -- C ABI of the B200-native FiGaRo hot path.
 *
 * Drop-in boundary for the reference pipeline entry
 *   figaro::run_pipeline(std::vector<Relation>, const JoinTree&,
 *                        const PipelineOptions&, bool keep_r0)
 *   (/root/reference/proj/include/figaro/driver.hpp:47-85)
 * and its phases
 *   compute_counts      (counts.hpp:92-224)
 *   figaro_r0           (figaro.hpp:319-329)
 *   postprocess_thin    (postprocess.hpp:261-273) + normalize_signs (:173-190)
 *
 * Plain C types only: int64 keys and FP64 data, row-major, exactly the memory
 * of figaro::Relation::keys (one int64 per key attribute, relation.hpp:27-28)
 * and figaro::Matrix (row-major, matrix.hpp:37,53-54).  Strings never reach
 * the device: attribute names are used on the host side of this library to
 * derive the join tree exactly as build_join_tree (join_tree.hpp:72-97) does.
 *
 * Every entry returns an fg_status.  Error codes map one-to-one onto the
 * reference's exception taxonomy (error.hpp:9-46); fg_last_error() gives the
 * message.  Device work is stream-ordered on the context's stream.
 *
 * There is no CPU fallback: if no sm_100 device is present every entry that
 * computes returns FG_E_CUDA.
 */
#ifndef FIGARO_CUDA_H_
#define FIGARO_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIGARO_CUDA_VERSION 1

#if defined(__GNUC__)
#define FG_API __attribute__((visibility("default")))
#else
#define FG_API
#endif

typedef int32_t fg_status;
enum {
  FG_OK = 0,
  FG_E_ARG = 1,         /* figaro::error: bad argument                    */
  FG_E_SCHEMA = 2,      /* figaro::schema_error                           */
  FG_E_TREE = 3,        /* figaro::tree_error                             */
  FG_E_INTEGRITY = 4,   /* figaro::integrity_error (unreduced input)      */
  FG_E_SIZE = 5,        /* figaro::size_error (u64 count overflow)        */
  FG_E_EMPTY_JOIN = 6,  /* figaro::empty_join_error                       */
  FG_E_UNSUPPORTED = 7, /* input shape this build does not handle         */
  FG_E_CUDA = 8,        /* CUDA runtime / launch failure                  */
  FG_E_RANK = 9,        /* figaro::rank_error (singular R in recover_q)   */
  FG_E_NCCL = 10        /* NCCL failure in fg_gather_r                    */
};

typedef struct fg_ctx fg_ctx;

/* ---- context ----------------------------------------------------------- */

/* One context per GPU.  Owns a stream, a stream-ordered memory pool and the
 * results of the last fg_run_pipeline call. */
FG_API fg_status fg_ctx_create(int32_t device, fg_ctx** out);
FG_API fg_status fg_ctx_destroy(fg_ctx* ctx);
/* Use an external stream (cudaStream_t passed as void*); NULL = own stream. */
FG_API fg_status fg_ctx_set_stream(fg_ctx* ctx, void* cuda_stream);
FG_API void* fg_ctx_stream(fg_ctx* ctx);
/* Message of the last failing call on this context (never NULL). */
FG_API const char* fg_last_error(fg_ctx* ctx);
FG_API int32_t fg_version(void);
/* Number of kernels this context launched since creation (evidence counter). */
FG_API int64_t fg_kernel_launches(fg_ctx* ctx);

/* ---- pipeline ---------------------------------------------------------- */

typedef struct fg_relation {
  const char* name;
  int32_t n_key;
  const char* const* key_attrs;  /* n_key names, declaration order         */
  int32_t n_data;
  const char* const* data_attrs; /* n_data names                           */
  int64_t rows;
  const int64_t* keys;           /* rows * n_key, row-major                 */
  const double* data;            /* rows * n_data, row-major                */
} fg_relation;

enum { FG_MEM_DEVICE = 0, FG_MEM_HOST = 1 };
enum { FG_ENGINE_THIN = 0, FG_ENGINE_HOUSEHOLDER = 1 };

typedef struct fg_options {
  int32_t assume_reduced; /* PipelineOptions::assume_reduced (driver.hpp:30) */
  int32_t engine;         /* PipelineOptions::engine (driver.hpp:29); both
                             engines run the device TSQR                    */
  int32_t memory;         /* where keys/data/R live: FG_MEM_DEVICE|HOST      */
  int32_t keep_r0;        /* keep R0 spans on the device for fg_get_r0_*     */
  int32_t fuse;           /* 1: tails go straight into the TSQR leaf         */
  int32_t reserved[3];
} fg_options;

/* Zero-initialised options are the reference defaults except memory. */
FG_API void fg_options_default(fg_options* o);

typedef struct fg_result {
  int64_t data_columns;   /* N   (PipelineResult::data_columns)            */
  int64_t input_rows;     /* M   (PipelineResult::input_rows)              */
  int64_t r0_rows;        /* rows(R0) (PipelineResult::r0_rows)            */
  double seconds_group;   /* device time per phase (CUDA events)           */
  double seconds_counts;
  double seconds_figaro;
  double seconds_postprocess;
  double seconds_total;   /* whole call incl. host<->device copies         */
  int64_t kernels;        /* kernels launched by this call                  */
  double seconds_headtail_kernels; /* device time of the heads/tails (or  */
                          /* fused heads/tails->TSQR) kernels of the call  */
  double seconds_tsqr_kernels;     /* device time of the TSQR stage        */
  int64_t headtail_launches;
  /* Algorithmic units of the timed launches (SURVEY
   * 8(d)): bytes = 8 x (input data elements read + summary elements read
   * + head/summary elements written + tail elements written to HBM) of the
   * heads/tails launches; flops = 2 m w^2 - 2/3 w^3 per column span, split
   * between the spans absorbed inside the fused heads/tails kernels and the
   * spans (plus the 2/3 N^3 final merge) factored in the TSQR stage.     */
  double headtail_bytes;
  double headtail_fused_flops;
  double tsqr_stage_flops;
  int64_t fused_launches;         /* heads/tails launches that were fused  */
  int64_t host_syncs;             /* host<->device synchronisations       */
  int64_t device_mallocs;         /* cudaMalloc calls (caching-allocator misses) */
  int64_t reserved[2];
} fg_result;

/* Runs validate_join_tree, counts, the FiGaRo transform and the TSQR
 * post-processing; writes the sign-normalised N x N R (row-major, strict
 * lower triangle exactly 0) to R_out (device or host per options->memory).
 * `parent[i]` is the parent relation index of relation i, -1 at `root`
 * (build_join_tree's arguments, join_tree.hpp:72-73). */
FG_API fg_status fg_run_pipeline(fg_ctx* ctx, int32_t n_rel, const fg_relation* rels,
                          int32_t root, const int32_t* parent,
                          const fg_options* options, double* R_out,
                          fg_result* result);

/* ---- results of the last pipeline run (host copies) -------------------- */

/* Kinds of per-node tables; order = NodeCounts fields (counts.hpp:24-31). */
enum {
  FG_ROWS_PER_KEY = 0,  /* own keys   */
  FG_THETA_DOWN = 1,    /* own keys   */
  FG_FULL_JOIN_SIZE = 2,/* own keys   */
  FG_PHI_CIRC = 3,      /* own keys   */
  FG_PHI_DOWN = 4,      /* parent keys */
  FG_PHI_UP = 5         /* parent keys */
};

/* Number of distinct own keys (G) and distinct parent-shared keys (P). */
FG_API fg_status fg_get_sizes(fg_ctx* ctx, int32_t node, int64_t* G, int64_t* P);
/* Relation::key_groups() begins in canonical (sorted) row order, G+1 values
 * (last = rows).  relation.hpp:56-66 */
FG_API fg_status fg_get_segments(fg_ctx* ctx, int32_t node, int64_t* begins);
/* Distinct own keys (G x n_key) or parent keys (P x n_pattr), ascending. */
FG_API fg_status fg_get_keys(fg_ctx* ctx, int32_t node, int32_t parent_keys,
                      int64_t* out);
/* One count table (G or P u64 values, ascending key order). */
FG_API fg_status fg_get_counts(fg_ctx* ctx, int32_t node, int32_t kind,
                        uint64_t* out);
/* Stable sort permutation of the node's rows (rows int32 values). */
FG_API fg_status fg_get_permutation(fg_ctx* ctx, int32_t node, int32_t* out);

/* R0 spans (only with keep_r0 and fuse == 0).  Span order follows
 * figaro()'s block order (figaro.hpp:166-316): each span is the vertical
 * concatenation of the reference's OutBlocks of one (node, col_begin). */
FG_API fg_status fg_get_r0_span_count(fg_ctx* ctx, int32_t* n_spans);
FG_API fg_status fg_get_r0_span(fg_ctx* ctx, int32_t idx, int32_t* node,
                         int64_t* col_begin, int64_t* rows, int64_t* cols,
                         double* out /* host, rows*cols, may be NULL */);

/* ---- phase-level kernels (device pointers, context stream) ------------- */

/* K1: stable grouping of packed keys; every keys[i] < 2^bits (bits <= 32 runs
 * the 32-bit key path the pipeline uses for narrow keys).
 * Writes perm[n] (stable sort permutation), begins[G+1] and uniq[G]
 * (capacity n+1 / n), and *G (host).  relation.hpp:56-66,127-167 */
FG_API fg_status fg_group_keys(fg_ctx* ctx, const uint64_t* keys, int64_t n,
                        int32_t bits, int32_t* perm, int32_t* begins,
                        uint64_t* uniq, int64_t* G);

/* K3/K5: heads and tails of n_seg row groups.  Row p of the sorted order is
 * data[(perm ? perm[p] : p) * ld + c], c < w.  Group g spans sorted rows
 * [begins[g], begins[g+1]).  weights (per source row, optional) select the
 * generalized transform (givens.hpp:106-148) instead of head/tail
 * (givens.hpp:59-92).  Tails of group g are multiplied by
 * sqrt(tail_count[g]) (optional) and written densely: tail row index
 * begins[g] - g + j - 1 for j = 1..m-1, stride ldt.  heads[g*ldh + c] get
 * the (generalized) head; scales[g] = sqrt(m) or, with weights, ||v_g||. */
FG_API fg_status fg_heads_tails(fg_ctx* ctx, const double* data, int64_t ld,
                         int32_t w, const int32_t* perm, const int32_t* begins,
                         int64_t n_seg, const double* weights,
                         const uint64_t* tail_count, double* heads,
                         int64_t ldh, double* tails, int64_t ldt,
                         double* scales);

/* K6/K7: R factor of a stack of row blocks.  Block b holds rows x cols
 * values at data (row stride ld) placed at columns [col_begin,
 * col_begin+cols) of an n-column matrix, zeros elsewhere.  Writes the
 * sign-normalised n x n R (device).  postprocess.hpp:35-190 */
typedef struct fg_block {
  const double* data;
  int64_t rows;
  int64_t ld;
  int32_t cols;
  int32_t col_begin;
} fg_block;
FG_API fg_status fg_tsqr(fg_ctx* ctx, int32_t n_blocks, const fg_block* blocks,
                  int32_t n, double* R_out);

/* ---- join rows and Q = A R^-1 (the steps after R) ---------------------- */

/* The join rows in the reference's depth-first order (for_each_join_row,
 * join.hpp:47-92): root rows in input order, then for every node in
 * pre-order the rows of that relation whose parent-shared key equals its
 * parent's current row's, in input order.  Relations are used as given (not
 * canonicalised, not reduced); dangling tuples yield no rows.  A row has
 * n = sum of n_data values in the pre-order column layout (make_layout,
 * join_tree.hpp:186-219).  More than `cap` rows -> FG_E_SIZE (join.hpp:77-79;
 * the reference's default cap is 1,000,000).  `memory` says where keys/data,
 * R, A_out and Q_out live (FG_MEM_DEVICE | FG_MEM_HOST); output buffers hold
 * rows x n doubles, row-major -- size them with fg_join_size. */

/* Number of join rows (for_each_join_row with an empty sink, join.hpp:63). */
FG_API fg_status fg_join_size(fg_ctx* ctx, int32_t n_rel, const fg_relation* rels,
                              int32_t root, const int32_t* parent, int32_t memory,
                              uint64_t cap, int64_t* rows);
/* A = the dense join (materialize_join, join.hpp:96-112). */
FG_API fg_status fg_materialize_join(fg_ctx* ctx, int32_t n_rel,
                                     const fg_relation* rels, int32_t root,
                                     const int32_t* parent, int32_t memory,
                                     uint64_t cap, double* A_out, int64_t* rows);
/* Q = A R^{-1} row by row (recover_q, postprocess.hpp:293-321): R is the
 * n x n upper-triangular factor (row-major); q solves q R = a by forward
 * substitution in the reference's operation order.  |R_ii| <= 1e-12 ||R||_F
 * -> FG_E_RANK before any work.  A_out (the streamed a_row) may be NULL;
 * with Q_out and A_out both NULL only the checks run and *rows is set.
 * n <= 128. */
FG_API fg_status fg_recover_q(fg_ctx* ctx, int32_t n_rel, const fg_relation* rels,
                              int32_t root, const int32_t* parent, int32_t memory,
                              uint64_t cap, const double* R, double* A_out,
                              double* Q_out, int64_t* rows);

/* ---- multi-GPU ------------------------------------------- */

/* One process (or host thread) per GPU, one context each.  Attach the rank's
 * NCCL communicator (an ncclComm_t passed as void*; NULL detaches).  NCCL is
 * resolved from the calling process at run time. */
FG_API fg_status fg_ctx_set_nccl(fg_ctx* ctx, void* nccl_comm);
/* All-gathers every rank's n x n factor R_local (row-major; device or host
 * per `memory`) over the communicator and writes the merged, sign-normalised
 * global R (one more TSQR of the P stacked factors) to R_out.  Every rank
 * calls it collectively with the same n; every rank gets the same R. */
FG_API fg_status fg_gather_r(fg_ctx* ctx, const double* R_local, int32_t n,
                             int32_t memory, double* R_out);

#ifdef __cplusplus
}
#endif

#endif /* FIGARO_CUDA_H_ */
