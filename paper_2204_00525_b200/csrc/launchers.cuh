// Host-side launchers of the device kernels (one per kernel family).
#pragma once

#include "fg_internal.cuh"

namespace fg {

constexpr int kMaxKeyCols = 16;
constexpr int kMaxChildren = 16;

// Field layout of a packed key: field f takes `bits[f]` bits at `shift[f]`
// and encodes the attribute value v as (u64)(v - min[f]).
struct PackSpec {
  int n;
  int col[kMaxKeyCols];  // source key column (pack) / source field (project)
  int shift[kMaxKeyCols];
  int bits[kMaxKeyCols];
  long long min[kMaxKeyCols];
};

// ---- group.cu -------------------------------------------------------------
// Per key column min/max over rows (atomics into mins/maxs[attr_of_col]).
void launch_key_minmax(Context& ctx, const int64_t* keys, int64_t rows,
                       int n_key, const int* attr_of_col_dev,
                       long long* mins, long long* maxs);
// Packs int64 key tuples into u64 keys (declaration order, MSB first) and
// writes the identity permutation.
template <class KeyT>
void launch_pack_keys(Context& ctx, const int64_t* keys, int64_t rows,
                      int n_key, const PackSpec& spec, KeyT* out, int* iota);
// Re-packs already packed keys into another field layout (projection).
// n_dev (optional): the real element count, device-resident; n is then the
// host's upper bound (grid sizing only).
void launch_project(Context& ctx, const uint64_t* in, int64_t n,
                    const PackSpec& from_to, uint64_t* out, const int64_t* n_dev = nullptr);
// Stable radix sort of (key, perm) on the low `bits` bits + segment
// extraction.  perm_in == null means the identity permutation.
struct GroupOut {
  DevArray<int> perm;       // n
  DevArray<int> begins;     // G + 1 (allocated with n + 1 entries)
  DevArray<uint64_t> uniq;  // G (allocated with n entries)
  int64_t G = 0;
};
// Returns G on the host (synchronises).
void group_sorted(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                  const int* perm_in, GroupOut& out);
void group_sorted32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                    const int* perm_in, GroupOut& out);
// Split form: begin (sort + segments, no sync) for several inputs, one sync
// reading every pend.nr, then finish with the counts.  `hist` = the digit
// histograms from launch_pack_hist (null: computed here); `pidx` (optional,
// n entries) receives the run id of every input element.
struct GroupPending {
  int64_t n = 0;
  DevArray<int> begins;
  DevArray<uint64_t> uniq;
  DevArray<int64_t> nr;  // device: number of runs
};
void group_begin(Context& ctx, const uint64_t* keys, int64_t n, int bits,
                 const int* perm_in, GroupOut& out, GroupPending& pend,
                 const uint32_t* hist = nullptr, int* pidx = nullptr);
void group_begin32(Context& ctx, const uint32_t* keys, int64_t n, int bits,
                   const int* perm_in, GroupOut& out, GroupPending& pend,
                   const uint32_t* hist = nullptr, int* pidx = nullptr);
void group_finish(Context& ctx, int64_t G, GroupOut& out, GroupPending& pend);
// Same for keys already in ascending order (no sort; perm_in is kept).
// n_dev: as launch_project (buffers are sized for n); want_perm = false
// skips the (identity) permutation output.
void group_begin_presorted(Context& ctx, const uint64_t* keys, int64_t n,
                           const int* perm_in, GroupOut& out, GroupPending& pend,
                           int* pidx = nullptr, const int64_t* n_dev = nullptr,
                           bool want_perm = true);
void exclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n);
void inclusive_sum_int(Context& ctx, const int* in, int* out, int64_t n);

// ---- radix.cu ---------------------------------------------------------------
// Entries of the digit-histogram buffer of a `bits`-bit sort.
size_t radix_hist_size(int bits);
int radix_passes(int bits);
// Key packing fused with the digit histograms of the sort that follows.
template <class KeyT>
void launch_pack_hist(Context& ctx, const int64_t* keys, int64_t rows, int n_key,
                      const PackSpec& spec, int bits, KeyT* out, uint32_t* hist);
// Stable LSD onesweep sort of (key, val); vals_in == null sorts row ids.
template <class KeyT>
void radix_sort_pairs(Context& ctx, const KeyT* keys_in, KeyT* keys_out, const int* vals_in,
                      int* vals_out, int64_t n, int bits, const uint32_t* hist = nullptr);
// Runs of a sorted key array: begins[0..G] (begins[G] = n), uniq[0..G),
// *n_runs = G (device); pidx[perm ? perm[p] : p] = run of position p.
template <class KeyT>
void launch_segments(Context& ctx, const KeyT* sorted, int64_t n, int* begins, uint64_t* uniq,
                     int64_t* n_runs, const int* perm, int* pidx,
                     const int64_t* n_dev = nullptr);
void scan_int(Context& ctx, const int* in, int* out, int64_t n, bool inclusive);
// out[0..*count) = in[i] for keep[i] != 0, in order (device count).
void compact_flagged(Context& ctx, const int* in, const char* keep, int* out, int64_t n,
                     int64_t* count);

// For each of n packed keys (projected to the child's parent-key layout by
// `proj`), binary search it in sorted `table` (size m); write the index or
// flag ST_MISSING_CHILD and write -1.
void launch_lookup(Context& ctx, const uint64_t* own_keys, int64_t n,
                   const PackSpec& proj, const uint64_t* table, int64_t m,
                   int* out, unsigned* status);
// Same with the table's key width: keys of <= 24 bits use a direct-address
// table (one gather instead of a binary search).
void launch_lookup_bits(Context& ctx, const uint64_t* own_keys, int64_t n,
                        const PackSpec& proj, const uint64_t* table, int64_t m,
                        int bits, int* out, unsigned* status);
// Decodes packed keys back to int64 tuples (n x spec.n).
void launch_unpack(Context& ctx, const uint64_t* in, int64_t n,
                   const PackSpec& spec, int64_t* out);
void launch_iota(Context& ctx, int* out, int64_t n);
// out[i] = low 32 bits of in[i].
void launch_narrow(Context& ctx, const uint64_t* in, int64_t n, uint32_t* out);
// counts[g] = begins[g+1] - begins[g]
void launch_seg_sizes(Context& ctx, const int* begins, int64_t G,
                      uint64_t* sizes);

// ---- counts.cu ------------------------------------------------------------
struct ChildLinks {
  int n;
  const int* lidx[kMaxChildren];       // own segment -> child parent-key idx
  uint64_t* phi_down[kMaxChildren];
  uint64_t* phi_up[kMaxChildren];  // 2 P entries each (split accumulation)
  int64_t P[kMaxChildren];
};
// phi_down (own parent-key table) has 2 P entries, zeroed by the caller.
void launch_theta(Context& ctx, const uint64_t* sizes, int64_t G,
                  const ChildLinks& ch, const int* pidx, uint64_t* phi_down, int64_t P,
                  uint64_t* theta, unsigned* status);
void launch_fjs(Context& ctx, const uint64_t* sizes, const uint64_t* theta,
                int64_t G, const int* pidx, const uint64_t* phi_up,
                const ChildLinks& ch, const int64_t* child_P, uint64_t* fjs,
                uint64_t* circ, unsigned* status);
void launch_up_div(Context& ctx, uint64_t* phi_up, const uint64_t* phi_down,
                   int64_t P, unsigned* status);

// ---- headtail.cu ----------------------------------------------------------
struct JoinArgs;
struct HeadTailArgs {
  const double* data = nullptr;
  int64_t ld = 0;
  int w = 0;
  const int* perm = nullptr;        // sorted pos -> source row (null = id)
  const int* begins = nullptr;      // G + 1
  int64_t n_seg = 0;
  int64_t n_rows = 0;               // begins[G]
  const double* weights = nullptr;  // per source row (generalized mode)
  const uint64_t* tail_count = nullptr;   // tails *= sqrt(tail_count[g])
  const uint64_t* scale_count = nullptr;  // scale = sqrt(scale_count[g])
  const int* head_index = nullptr;  // output row of head/scale (null = g)
  double* heads = nullptr;
  int64_t ldh = 0;
  double* tails = nullptr;
  int64_t ldt = 0;
  double* scales = nullptr;
  // Join-on-read (project-away of a joined node, K4 folded into K5): rows
  // are the join of own heads (join_heads, row stride join_ldh) and the
  // children's summaries described by *join (S and scale of *join unused);
  // `data`/`ld` are ignored and `weights` are the own (pre-join) scales.
  const JoinArgs* join = nullptr;
  const double* join_heads = nullptr;
  int64_t join_ldh = 0;
  // Join-on-write (K4 folded into K3's head emission): the head row of group
  // g is written as the joined summary row -- own columns times prod_c s_c,
  // child columns from the children's summaries -- and `scales` receives the
  // joined scale sqrt(m_g) * prod_c s_c.  Uses join->n_children, lidx,
  // child_S, child_scale, child_w, child_off; `heads`/`ldh` is the summary.
  const JoinArgs* join_write = nullptr;
  // Per-group multiplier of the heads (the join's own-column factor), or null.
  const double* head_mul = nullptr;
};
// Runs the segmented (generalized) head/tail transform.  Needs the max
// segment size only to decide whether the heavy-segment pre-pass runs.
void run_heads_tails(Context& ctx, const HeadTailArgs& a);
// Fused K3 -> K6 for own tails (plain transform, w <= 32): heads/scales as
// run_heads_tails, tails absorbed per warp; writes count = return value
// partial factors of fused_width(w) x fused_width(w) to `partials`;
// returns -1 (nothing launched) when no fused kernel fits this width.
int fused_width(int w);
int run_heads_tails_fused(Context& ctx, const HeadTailArgs& a,
                          DevArray<double>& partials);

struct JoinArgs {
  int64_t G = 0;
  int own_w = 0;
  double* S = nullptr;  // G x width, own head in [0, own_w)
  int64_t width = 0;
  double* scale = nullptr;  // G (read)
  double* scale_out = nullptr;  // G (new scales, must not alias scale)
  int n_children = 0;
  const int* lidx[kMaxChildren];
  const double* child_S[kMaxChildren];
  const double* child_scale[kMaxChildren];
  int child_w[kMaxChildren];
  int child_off[kMaxChildren];  // local column offset in S
  // The own columns already carry prod_c s_c (heads/tails with head_mul):
  // only the children's columns and the scales are written.
  bool own_done = false;
};
void launch_join(Context& ctx, const JoinArgs& a);
// all_out[g] = product of the children's scales of summary row g.
void launch_join_all(Context& ctx, const JoinArgs& a, double* all_out);

// ---- tsqr.cu ----------------------------------------------------------------
struct Span {
  const double* data;
  int64_t rows;
  int64_t ld;
  int cols;
  int col_begin;
  // Already factored span (fused kernel): `count` partial W x W factors.
  const double* partials = nullptr;
  int count = 0;
  int W = 0;
};
// R (n x n, row-major, device) of the stacked spans, sign-normalised.
void tsqr(Context& ctx, const std::vector<Span>& spans, int n, double* R_out);

// ---- gather.cu -------------------------------------------------------------
void set_nccl(Context& ctx, void* comm);
// All-gather of the ranks' n x n factors + device TSQR merge (syncs).
void gather_r(Context& ctx, const double* R_local, int n, int memory, double* R_out);

// ---- join.cu ---------------------------------------------------------------
// Join rows in for_each_join_row order; count only when A_out and Q_out are
// null; Q = A R^-1 when Q_out is set (R host or device per `memory`).
void join_rows(Context& ctx, int32_t n_rel, const fg_relation* rels, int32_t root,
               const int32_t* parent, int32_t memory, uint64_t cap, const double* R,
               double* A_out, double* Q_out, int64_t* rows_out);

}  // namespace fg
