// Host orchestration of the device pipeline and the C ABI (figaro_cuda.h).
//
// fg_run_pipeline restates figaro::run_pipeline (driver.hpp:47-85):
//   validate_join_tree + build_join_tree   -> host (join_tree.hpp:72-180)
//   semi_join_reduce (unless assume_reduced) -> device selection vectors
//                                               (reduce.hpp:47-74)
//   make_layout                            -> host (join_tree.hpp:186-219)
//   canonical grouping                     -> K1 (group.cu)
//   compute_counts                         -> K2 (counts.cu)
//   figaro_r0                              -> K3/K4/K5 (headtail.cu)
//   postprocess_thin + normalize_signs     -> K6/K7 (tsqr.cu)
// Device phases are timed with CUDA events on the context stream.
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>


#include "host_tree.hpp"
#include "launchers.cuh"

namespace fg {

struct NodeState {
  std::string name;
  int n_key = 0, w = 0;
  int64_t rows_in = 0;   // rows as passed in
  int64_t rows = 0;      // rows after reduction
  std::vector<std::string> key_names, data_names;
  std::vector<int> key_attr;    // global attribute ids, declaration order
  std::vector<int> pattr;       // parent-shared attribute ids, name order
  std::vector<std::string> pattr_names;
  int parent = -1;
  std::vector<int> children;
  const int64_t* keys = nullptr;
  const double* data = nullptr;
  DevArray<int64_t> keys_own;
  DevArray<double> data_own;
  DevArray<int> sel;            // selected rows after reduction (or empty)
  bool has_sel = false;
  PackSpec own{};               // int64 key columns -> packed own key
  int own_bits = 0;
  GroupOut grp;
  DevArray<uint64_t> sizes;
  // parent-key grouping of own segments
  DevArray<int> pa_perm, pa_begins, pidx;
  bool pa_identity = false;  // parent-key order == own-key order (prefix case)
  DevArray<uint64_t> upk;
  int64_t P = 0;
  PackSpec par{};               // own packed -> parent key (pattr order)
  std::vector<DevArray<int>> lidx;  // per child
  DevArray<uint64_t> theta, fjs, circ, phi_down, phi_up;
  // summaries
  int64_t width = 0;
  DevArray<double> S, scale, scale_j, Sq, scale_q;
  const double* sum_S = nullptr;
  const double* sum_scale = nullptr;
  DevArray<double> tails, ptails;
  DevArray<double> fused;  // partial R factors of the own tails (fused path)
  int fused_count = 0, fused_W = 0;
  DevArray<double> pfused;  // ... and of the project-away tails
  int pfused_count = 0, pfused_W = 0;
};

struct SpanInfo {
  int node;
  int64_t col_begin;
  int64_t rows;
  int64_t cols;
  const double* data;
};

struct Context::Saved {
  std::vector<std::unique_ptr<NodeState>> nodes;
  std::vector<SpanInfo> spans;
  bool have_r0 = false;
};

namespace {

// --------------------------------------------------------------- reduction

__global__ void k_pack_sel(const int64_t* __restrict__ keys, int n_key,
                           const int* __restrict__ sel, int64_t n,
                           PackSpec spec, uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = sel ? sel[t] : t;
    uint64_t k = 0;
    for (int f = 0; f < spec.n; ++f) {
      const long long v = keys[i * n_key + spec.col[f]];
      if (spec.bits[f]) k |= ((uint64_t)v - (uint64_t)spec.min[f]) << spec.shift[f];
    }
    out[t] = k;
  }
}

__global__ void k_member(const uint64_t* __restrict__ q, int64_t n,
                         const uint64_t* __restrict__ table, int64_t m,
                         char* __restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = q[t];
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (table[mid] < key) lo = mid + 1; else hi = mid;
    }
    keep[t] = (lo < m && table[lo] == key) ? 1 : 0;
  }
}

int grid1d(const Context& ctx, int64_t n) {
  int64_t g = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx.sm_count * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

// Packs the projection of node `i`'s selected rows onto `attrs`.
void pack_projection(Context& ctx, NodeState& n, const std::vector<int>& attrs,
                     const std::vector<AttrCode>& code, DevArray<uint64_t>& out) {
  PackSpec s = make_spec(attrs, code,
                         [&](int a) {
                           return (int)(std::find(n.key_attr.begin(),
                                                  n.key_attr.end(), a) -
                                        n.key_attr.begin());
                         },
                         nullptr, "semi-join");
  out.alloc(n.rows, ctx.stream);
  if (n.rows == 0) return;
  k_pack_sel<<<grid1d(ctx, n.rows), 256, 0, ctx.stream>>>(
      n.keys, n.n_key, n.has_sel ? n.sel.get() : nullptr, n.rows, s,
      out.get());
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
}

// semi_join (reduce.hpp:20-43): keep rows of `a` whose projection onto
// `attrs` occurs in `b`.  Row order is preserved (selection vector).
void semi_join(Context& ctx, NodeState& a, NodeState& b,
               const std::vector<int>& attrs, const std::vector<AttrCode>& code) {
  if (attrs.empty()) return;
  DevArray<uint64_t> qa, qb;
  pack_projection(ctx, a, attrs, code, qa);
  pack_projection(ctx, b, attrs, code, qb);
  DevArray<uint64_t> tb(b.rows, ctx.stream);
  if (b.rows) {
    int bits = 0;
    for (int x : attrs) bits += code[x].bits;
    DevArray<int> tv(b.rows, ctx.stream);
    radix_sort_pairs<uint64_t>(ctx, qb.get(), tb.get(), nullptr, tv.get(), b.rows,
                               std::max(bits, 1));
  }
  DevArray<char> keep(a.rows, ctx.stream);
  if (a.rows) {
    k_member<<<grid1d(ctx, a.rows), 256, 0, ctx.stream>>>(
        qa.get(), a.rows, tb.get(), b.rows, keep.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
  }
  DevArray<int> cur;
  if (!a.has_sel) {
    cur.alloc(a.rows, ctx.stream);
    launch_iota(ctx, cur.get(), a.rows);
  } else {
    cur = std::move(a.sel);
  }
  DevArray<int> next(a.rows, ctx.stream);
  DevArray<int64_t> nsel(1, ctx.stream);
  compact_flagged(ctx, cur.get(), keep.get(), next.get(), a.rows, nsel.get());
  int64_t m = 0;
  FG_CUDA(cudaMemcpyAsync(&m, nsel.get(), sizeof m, cudaMemcpyDeviceToHost,
                          ctx.stream));
  sync_stream(ctx);
  a.sel = std::move(next);
  a.has_sel = true;
  a.rows = m;
}

void check_nonempty(const NodeState& n) {
  if (n.rows == 0)
    fail(FG_E_EMPTY_JOIN, "relation " + n.name +
                              " reduced to empty: the join result is empty");
}

// --------------------------------------------------------------- status

// Maps the device status word read back with the final synchronisation to
// the reference's exceptions.  The transform and TSQR kernels tolerate the
// flagged states (a missing child is a zero row, inexact counts are 0), so
// the word is read once at the end instead of stalling the stream after K2.
void raise_status(unsigned st, const char* phase) {
  if (!st) return;
  const std::string p = phase;
  if (st & ST_MISSING_CHILD)
    fail(FG_E_INTEGRITY, p + ": a key has no match in a child relation; is the "
                             "database fully reduced?");
  if (st & ST_OVERFLOW)
    fail(FG_E_SIZE, "count aggregate overflow (64-bit)");
  if (st & ST_UP_UNMATCHED)
    fail(FG_E_INTEGRITY, p + ": a child has keys unmatched in its parent; is "
                             "the database fully reduced?");
  if (st & ST_CIRC_INEXACT)
    fail(FG_E_INTEGRITY, p + ": phi_circ: counts are inconsistent; is the "
                             "database fully reduced?");
  if (st & ST_UP_INEXACT)
    fail(FG_E_INTEGRITY, p + ": phi_up: counts are inconsistent; is the "
                             "database fully reduced?");
  fail(FG_E_INTEGRITY, p + ": inconsistent counts");
}

// Host-side stage timer, enabled with FG_TRACE=1 (prints to stderr).
struct Trace {
  bool on = getenv("FG_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[fg] %-28s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Event pairs bracketing individual launches (per-kernel device time).
struct KernelTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  cudaStream_t st;
  explicit KernelTimer(cudaStream_t s) : st(s) {}
  ~KernelTimer() {
    for (auto& e : ev) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  }
  void begin() {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ev.push_back({a, b});
    cudaEventRecord(a, st);
  }
  void end() { cudaEventRecord(ev.back().second, st); }
  double seconds() const {
    double s = 0;
    for (auto& e : ev) {
      float t = 0;
      cudaEventElapsedTime(&t, e.first, e.second);
      s += t * 1e-3;
    }
    return s;
  }
};

// Events of the overlapped host upload (copy stream -> compute stream).
struct UploadEvents {
  cudaEvent_t ready = nullptr, keys = nullptr;
  std::vector<cudaEvent_t> data;
  cudaStream_t copy = nullptr;  // drained before the buffers are released
  void init(int n, cudaStream_t s) {
    copy = s;
    FG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    FG_CUDA(cudaEventCreateWithFlags(&keys, cudaEventDisableTiming));
    data.assign(n, nullptr);
    for (auto& e : data) FG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~UploadEvents() {
    if (copy) cudaStreamSynchronize(copy);
    if (ready) cudaEventDestroy(ready);
    if (keys) cudaEventDestroy(keys);
    for (auto e : data) if (e) cudaEventDestroy(e);
  }
};

struct Events {
  cudaEvent_t e[6];
  Events() { for (auto& x : e) cudaEventCreate(&x); }
  ~Events() { for (auto& x : e) cudaEventDestroy(x); }
  double ms(int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, e[a], e[b]);
    return t * 1e-3;
  }
};

// ---------------------------------------------------------------- pipeline

void run(Context& ctx, int32_t n_rel, const fg_relation* rels, int32_t root,
         const int32_t* parent, const fg_options& opt, double* R_out,
         fg_result* res) {
  if (n_rel <= 0 || !rels || !parent) fail(FG_E_ARG, "no relations");
  cudaStream_t st = ctx.stream;
  const int64_t launches0 = ctx.launches;
  auto saved = std::make_unique<Context::Saved>();
  auto& nodes = saved->nodes;
  for (int i = 0; i < n_rel; ++i) {
    const fg_relation& r = rels[i];
    auto n = std::make_unique<NodeState>();
    n->name = r.name ? r.name : ("R" + std::to_string(i));
    n->n_key = r.n_key;
    n->w = r.n_data;
    n->rows_in = n->rows = r.rows;
    if (r.n_key < 0 || r.n_data < 0 || r.rows < 0)
      fail(FG_E_ARG, "relation " + n->name + ": negative size");
    if (r.rows > INT_MAX)
      fail(FG_E_UNSUPPORTED, "relation " + n->name + ": more than 2^31-1 rows");
    if ((r.rows && r.n_key && !r.keys) || (r.rows && r.n_data && !r.data))
      fail(FG_E_ARG, "relation " + n->name + ": null keys/data");
    for (int k = 0; k < r.n_key; ++k)
      n->key_names.push_back(r.key_attrs && r.key_attrs[k] ? r.key_attrs[k] : "");
    for (int k = 0; k < r.n_data; ++k)
      n->data_names.push_back(r.data_attrs && r.data_attrs[k] ? r.data_attrs[k]
                                                              : "");
    nodes.push_back(std::move(n));
  }
  std::vector<int> preorder;
  build_tree(nodes, root, parent, preorder);
  validate(nodes);
  const Layout lay = make_layout(nodes, preorder, root);
  if (lay.total > 128)
    fail(FG_E_UNSUPPORTED, "more than 128 data columns in total");

  Trace tr;
  Events ev;
  KernelTimer kt_ht(st), kt_tsqr(st);
  // Algorithmic units of the timed launches.
  double ht_bytes = 0, fused_flops = 0, tsqr_flops = 0;
  int64_t fused_launches = 0;
  const int64_t syncs0 = ctx.syncs;
  const int64_t mallocs0 = ctx.cache.mallocs();
  auto span_flops = [](double m, double w) {
    return m > 0 && w > 0 ? 2.0 * m * w * w - 2.0 / 3.0 * w * w * w : 0.0;
  };
  FG_CUDA(cudaEventRecord(ev.e[0], st));

  // Inputs on the device.  Host inputs are uploaded on the context's copy
  // stream -- all keys first, then the data in the order the transform reads
  // it (reverse pre-order) -- so grouping and counts run while the data is
  // still crossing PCIe; the compute stream waits per relation.
  UploadEvents up;
  const bool host_in = opt.memory == FG_MEM_HOST;
  if (host_in) {
    for (int i = 0; i < n_rel; ++i) {
      nodes[i]->keys_own.alloc(rels[i].rows * rels[i].n_key, st);
      nodes[i]->data_own.alloc(rels[i].rows * rels[i].n_data, st);
    }
    up.init(n_rel, ctx.copy_stream);
    FG_CUDA(cudaEventRecord(up.ready, st));  // buffers free on the compute stream
    FG_CUDA(cudaStreamWaitEvent(ctx.copy_stream, up.ready, 0));
  }
  for (int i = 0; i < n_rel; ++i) {
    NodeState& n = *nodes[i];
    const fg_relation& r = rels[i];
    if (host_in) {
      if (n.keys_own.size())
        FG_CUDA(cudaMemcpyAsync(n.keys_own.get(), r.keys, n.keys_own.bytes(),
                                cudaMemcpyHostToDevice, ctx.copy_stream));
      n.keys = n.keys_own.get();
      n.data = n.data_own.get();
    } else {
      n.keys = r.keys;
      n.data = r.data;
    }
  }
  if (host_in) {
    FG_CUDA(cudaEventRecord(up.keys, ctx.copy_stream));
    for (auto it = preorder.rbegin(); it != preorder.rend(); ++it) {
      NodeState& n = *nodes[*it];
      if (n.data_own.size())
        FG_CUDA(cudaMemcpyAsync(n.data_own.get(), rels[*it].data, n.data_own.bytes(),
                                cudaMemcpyHostToDevice, ctx.copy_stream));
      FG_CUDA(cudaEventRecord(up.data[*it], ctx.copy_stream));
    }
    FG_CUDA(cudaStreamWaitEvent(st, up.keys, 0));
  }
  FG_CUDA(cudaEventRecord(ev.e[1], st));
  // The status word outlives streams bound with fg_ctx_set_stream: clear it
  // on the stream this call runs on.
  FG_CUDA(cudaMemsetAsync(ctx.status.get(), 0, sizeof(unsigned), st));
  tr.mark("setup+upload");

  // ---- attribute encodings (global, per attribute name)
  std::vector<AttrCode> code = encode_attributes(ctx, nodes);
  tr.mark("encode (minmax sync)");
  // ---- semi-join reduction (reduce.hpp:47-74)
  if (!opt.assume_reduced) {
    for (int i : preorder) check_nonempty(*nodes[i]);
    for (auto it = preorder.rbegin(); it != preorder.rend(); ++it)
      for (int c : nodes[*it]->children) {
        semi_join(ctx, *nodes[*it], *nodes[c], nodes[c]->pattr, code);
        check_nonempty(*nodes[*it]);
      }
    for (int i : preorder)
      for (int c : nodes[i]->children) {
        semi_join(ctx, *nodes[c], *nodes[i], nodes[c]->pattr, code);
        check_nonempty(*nodes[c]);
      }
  }

  // ---- K1: own-key grouping per relation.  All sorts are enqueued first;
  // one synchronisation reads every relation's group count.
  std::vector<GroupPending> pend(nodes.size());
  std::vector<DevArray<uint32_t>> pk32(nodes.size());
  std::vector<DevArray<uint64_t>> pk64(nodes.size());
  std::vector<DevArray<uint32_t>> hists(nodes.size());
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    NodeState& n = *nodes[ni];
    n.own = make_spec(n.key_attr, code,
                      [&](int a) {
                        return (int)(std::find(n.key_attr.begin(),
                                               n.key_attr.end(), a) -
                                     n.key_attr.begin());
                      },
                      &n.own_bits, "relation " + n.name);
    hists[ni].alloc(radix_hist_size(n.own_bits), st);
    if (n.own_bits <= 32 && !n.has_sel) {
      // Narrow packed keys: 8 instead of 12 bytes per element per radix pass.
      // Packing also builds every pass's digit histogram; the first pass
      // generates the row ids itself.
      pk32[ni].alloc(n.rows, st);
      launch_pack_hist<uint32_t>(ctx, n.keys, n.rows, n.n_key, n.own, n.own_bits,
                                 pk32[ni].get(), hists[ni].get());
      group_begin32(ctx, pk32[ni].get(), n.rows, n.own_bits, nullptr, n.grp, pend[ni],
                    hists[ni].get());
    } else if (!n.has_sel) {
      pk64[ni].alloc(n.rows, st);
      launch_pack_hist<uint64_t>(ctx, n.keys, n.rows, n.n_key, n.own, n.own_bits,
                                 pk64[ni].get(), hists[ni].get());
      group_begin(ctx, pk64[ni].get(), n.rows, n.own_bits, nullptr, n.grp, pend[ni],
                  hists[ni].get());
    } else {
      pk64[ni].alloc(n.rows, st);
      if (n.rows) {
        k_pack_sel<<<grid1d(ctx, n.rows), 256, 0, st>>>(n.keys, n.n_key,
                                                        n.sel.get(), n.rows,
                                                        n.own, pk64[ni].get());
        FG_LAUNCHED(ctx);
        FG_KERNEL_CHECK();
      }
      group_begin(ctx, pk64[ni].get(), n.rows, n.own_bits, n.sel.get(), n.grp, pend[ni]);
    }
  }
  // Parent-key grouping of own segments (the std::map regroupings of
  // counts.hpp:121-130 and figaro.hpp:236-239).  Parent attributes that are
  // the leading own-key attributes (in the same order) project the ascending
  // own keys to ascending parent keys -- no sort (C3's F under D1, C4's R2
  // under R1, every leaf, 2-way joins): those regroupings are enqueued right
  // behind the own grouping with the group count G still on the device, so
  // one synchronisation reads every G and P.  Other nodes sort their G
  // projected keys after it (a second synchronisation for their P).
  std::vector<GroupPending> ppend(nodes.size());
  std::vector<GroupOut> pgs(nodes.size());
  std::vector<DevArray<uint64_t>> ppks(nodes.size());
  auto parent_spec = [&](NodeState& n, int* pbits) {
    n.par = make_spec(n.pattr, code,
                      [&](int a) {
                        const int f = (int)(std::find(n.key_attr.begin(),
                                                      n.key_attr.end(), a) -
                                            n.key_attr.begin());
                        return n.own.shift[f];
                      },
                      pbits, "relation " + n.name + " (parent key)");
  };
  bool any_sorted_parent = false;
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    NodeState& n = *nodes[ni];
    if (n.parent < 0) continue;
    const bool prefix = n.pattr.size() <= n.key_attr.size() &&
                        std::equal(n.pattr.begin(), n.pattr.end(), n.key_attr.begin());
    n.pa_identity = prefix;
    if (!prefix) {
      any_sorted_parent = true;
      continue;
    }
    int pbits = 0;
    parent_spec(n, &pbits);
    // upper bound: G <= rows
    ppks[ni].alloc(n.rows, st);
    n.pidx.alloc(n.rows, st);
    launch_project(ctx, pend[ni].uniq.get(), n.rows, n.par, ppks[ni].get(), pend[ni].nr.get());
    // pidx[g] = parent-key run of own segment g, written by the segment
    // extraction of the parent-key grouping.
    group_begin_presorted(ctx, ppks[ni].get(), n.rows, nullptr, pgs[ni], ppend[ni],
                          n.pidx.get(), pend[ni].nr.get(), /*want_perm=*/false);
  }
  std::vector<int64_t> Gs(nodes.size(), 0), Ps(nodes.size(), 0);
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    FG_CUDA(cudaMemcpyAsync(&Gs[ni], pend[ni].nr.get(), sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    if (nodes[ni]->parent >= 0 && nodes[ni]->pa_identity)
      FG_CUDA(cudaMemcpyAsync(&Ps[ni], ppend[ni].nr.get(), sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
  }
  sync_stream(ctx);
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    NodeState& n = *nodes[ni];
    group_finish(ctx, Gs[ni], n.grp, pend[ni]);
    pk32[ni].release();
    pk64[ni].release();
    hists[ni].release();
    n.sizes.alloc(n.grp.G, st);
    launch_seg_sizes(ctx, n.grp.begins.get(), n.grp.G, n.sizes.get());
  }
  tr.mark("own grouping");
  if (any_sorted_parent) {
    for (size_t ni = 0; ni < nodes.size(); ++ni) {
      NodeState& n = *nodes[ni];
      if (n.parent < 0 || n.pa_identity) continue;
      int pbits = 0;
      parent_spec(n, &pbits);
      const int64_t G = n.grp.G;
      ppks[ni].alloc(G, st);
      launch_project(ctx, n.grp.uniq.get(), G, n.par, ppks[ni].get());
      n.pidx.alloc(G, st);
      group_begin(ctx, ppks[ni].get(), G, pbits, nullptr, pgs[ni], ppend[ni], nullptr,
                  n.pidx.get());
      FG_CUDA(cudaMemcpyAsync(&Ps[ni], ppend[ni].nr.get(), sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    }
    sync_stream(ctx);
  }
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    NodeState& n = *nodes[ni];
    if (n.parent < 0) continue;
    const int64_t G = n.grp.G;
    GroupOut& pg = pgs[ni];
    group_finish(ctx, Ps[ni], pg, ppend[ni]);
    n.P = pg.G;
    n.pa_perm = std::move(pg.perm);
    n.pa_begins = std::move(pg.begins);
    n.upk = std::move(pg.uniq);
    ppks[ni].release();
    if (n.children.empty() && n.P != G)
      fail(FG_E_INTEGRITY, "relation " + n.name +
                               ": leaf keys do not match its parent attributes");
  }
  tr.mark("parent grouping");
  // Edge lookups: own segment of i -> parent-key index of child c.
  for (auto& np : nodes) {
    NodeState& n = *np;
    for (int c : n.children) {
      NodeState& ch = *nodes[c];
      int pbits = 0;
      PackSpec proj = make_spec(ch.pattr, code,
                                [&](int a) {
                                  const int f = (int)(std::find(n.key_attr.begin(),
                                                                n.key_attr.end(), a) -
                                                      n.key_attr.begin());
                                  return n.own.shift[f];
                                },
                                &pbits, "edge " + n.name + "-" + ch.name);
      DevArray<int> l(n.grp.G, st);
      launch_lookup_bits(ctx, n.grp.uniq.get(), n.grp.G, proj, ch.upk.get(), ch.P,
                         pbits, l.get(), ctx.status.get());
      n.lidx.push_back(std::move(l));
    }
  }
  FG_CUDA(cudaEventRecord(ev.e[2], st));

  // ---- K2: counts (counts.hpp:92-224)
  for (auto& np : nodes) {
    NodeState& n = *np;
    n.theta.alloc(n.grp.G, st);
    n.fjs.alloc(n.grp.G, st);
    n.circ.alloc(n.grp.G, st);
    // 2 P: low/high-word accumulators of the split sums (counts.cu add_split)
    n.phi_down.alloc(2 * n.P, st);
    n.phi_up.alloc(2 * n.P, st);
    n.phi_down.zero();
    n.phi_up.zero();
  }
  auto links = [&](NodeState& n) {
    ChildLinks ch{};
    ch.n = (int)n.children.size();
    if (ch.n > kMaxChildren) fail(FG_E_UNSUPPORTED, "more than 16 children");
    for (int k = 0; k < ch.n; ++k) {
      NodeState& c = *nodes[n.children[k]];
      ch.lidx[k] = n.lidx[k].get();
      ch.phi_down[k] = c.phi_down.get();
      ch.phi_up[k] = c.phi_up.get();
      ch.P[k] = c.P;
    }
    return ch;
  };
  for (auto it = preorder.rbegin(); it != preorder.rend(); ++it) {
    NodeState& n = *nodes[*it];
    launch_theta(ctx, n.sizes.get(), n.grp.G, links(n),
                 n.parent >= 0 ? n.pidx.get() : nullptr, n.phi_down.get(), n.P,
                 n.theta.get(), ctx.status.get());
  }
  for (int i : preorder) {
    NodeState& n = *nodes[i];
    std::vector<int64_t> child_P;
    for (int c : n.children) child_P.push_back(nodes[c]->P);
    launch_fjs(ctx, n.sizes.get(), n.theta.get(), n.grp.G,
               n.parent >= 0 ? n.pidx.get() : nullptr, n.phi_up.get(), links(n),
               child_P.data(), n.fjs.get(), n.circ.get(), ctx.status.get());
    for (int c : n.children)
      launch_up_div(ctx, nodes[c]->phi_up.get(), nodes[c]->phi_down.get(),
                    nodes[c]->P, ctx.status.get());
  }
  FG_CUDA(cudaEventRecord(ev.e[3], st));
  tr.mark("lookups+counts enqueue");

  // ---- K3/K4/K5: the FiGaRo transform (figaro.hpp:166-329)
  for (auto it = preorder.rbegin(); it != preorder.rend(); ++it) {
    const int i = *it;
    NodeState& n = *nodes[i];
    const bool is_root = n.parent < 0;
    const bool is_leaf = n.children.empty();
    const int64_t G = n.grp.G;
    n.width = lay.sub_end[i] - lay.sub_begin[i];
    // Join-on-read: an inner node's joined summary rows are consumed only
    // by its project-away, which builds them on the fly from the own heads
    // and the children's summaries -- S holds just the heads (C3's fact
    // node: 54 M x 8 instead of 54 M x 20 written, read and re-read).
    // Measured slower than materialising S (C3: figaro 19.0 -> 27.7 ms; the
    // per-row factor loads dominate), so it is opt-in (FG_JOIN_ON_READ=1).
    const bool vj = !is_root && !is_leaf && n.width > 0 &&
                    (int)n.children.size() <= 4 && getenv("FG_JOIN_ON_READ") != nullptr;
    const int64_t ldS = vj ? n.w : n.width;
    // Every element of S is written: own columns by the heads (one per
    // group), child columns by the join (zero for a missing child), so no
    // memset (8.6 GB on C3's fact node).
    n.S.alloc(G * std::max<int64_t>(ldS, 1), st);
    n.scale.alloc(G, st);
    const int64_t n_tails = n.rows - G;
    // The fused kernel absorbs a zero row per group start; when groups are
    // short (tails < 70% of the rows) writing the tails densely and factoring
    // only them is cheaper (measured on C3's F: 9.1 ms fused vs 6.7 ms).
    const bool fuse = opt.fuse && !opt.keep_r0 && fused_width(n.w) > 0 && n_tails > 0 &&
                      n_tails * 10 >= n.rows * 7;
    if (n.w > 0 && n_tails > 0 && !fuse) n.tails.alloc(n_tails * n.w, st);
    JoinArgs j{};
    if (!is_leaf) {
      j.G = G;
      j.own_w = n.w;
      j.S = n.S.get();
      j.width = n.width;
      j.scale = n.scale.get();
      j.n_children = (int)n.children.size();
      for (int k = 0; k < j.n_children; ++k) {
        NodeState& c = *nodes[n.children[k]];
        j.lidx[k] = n.lidx[k].get();
        j.child_S[k] = c.sum_S;
        j.child_scale[k] = c.sum_scale;
        j.child_w[k] = (int)c.width;
        j.child_off[k] = (int)(lay.sub_begin[n.children[k]] - lay.sub_begin[i]);
      }
    }
    // Join-on-write: the unfused own heads/tails kernel emits the joined
    // summary rows and scales itself (no separate K4 pass over S).  Measured
    // slower on C3 (figaro 18.9 -> 20.5 ms: the child lookups stall the
    // head emission), so it is opt-in (FG_JOIN_ON_WRITE=1).
    const bool jw = !is_leaf && !vj && !fuse && n.w > 0 && n.w <= 16 && G > 0 &&
                    (int)n.children.size() <= 4 && getenv("FG_JOIN_ON_WRITE") != nullptr;
    if (host_in) FG_CUDA(cudaStreamWaitEvent(st, up.data[i], 0));
    HeadTailArgs a;
    a.data = n.data;
    a.ld = n.w;
    a.w = n.w;
    a.perm = n.grp.perm.get();
    a.begins = n.grp.begins.get();
    a.n_seg = G;
    a.n_rows = n.rows;
    a.tail_count = n.circ.get();
    a.head_index = (is_leaf && !is_root) ? n.pidx.get() : nullptr;
    a.heads = n.w > 0 ? n.S.get() : nullptr;
    a.ldh = ldS;
    a.tails = n.tails.get();
    a.ldt = n.w;
    a.scales = n.scale.get();
    a.join_write = jw ? &j : nullptr;
    // The join's own-column factor prod_c s_c is applied by the heads/tails
    // kernel as it writes the heads (no read-modify-write pass over S's own
    // columns); the join then writes only the children's columns.
    DevArray<double> hmul;
    const bool own_mul = !is_leaf && !vj && !jw && n.w > 0 && G > 0 &&
                         getenv("FG_JOIN_OWN_PASS") == nullptr;
    if (own_mul) {
      hmul.alloc(G, st);
      launch_join_all(ctx, j, hmul.get());
      a.head_mul = hmul.get();
      j.own_done = true;
    }
    kt_ht.begin();
    if (fuse) {
      n.fused_count = run_heads_tails_fused(ctx, a, n.fused);
      n.fused_W = fused_width(n.w);
    }
    if (!fuse || n.fused_count < 0) {
      n.fused_count = 0;
      if (n.w > 0 && n_tails > 0 && !n.tails.size()) n.tails.alloc(n_tails * n.w, st);
      a.tails = n.tails.get();
      run_heads_tails(ctx, a);
    }
    kt_ht.end();
    // input elements read once + heads written once (+ tails written once
    // when they go to HBM; fused tails stay on chip)
    // (+ the children's summary columns of the joined rows with join-on-write)
    ht_bytes += 8.0 * ((double)n.rows * n.w + (double)G * n.w +
                       (n.fused_count ? 0.0 : (double)n_tails * n.w) +
                       (jw ? (double)G * (n.width - n.w) : 0.0));
    if (n.fused_count) {
      ++fused_launches;
      fused_flops += span_flops((double)n_tails, n.w);
    }
    if (!is_leaf && !vj && !jw) {
      n.scale_j.alloc(G, st);
      j.scale_out = n.scale_j.get();
      launch_join(ctx, j);
      std::swap(n.scale, n.scale_j);  // joined scales replace the head scales
    }
    if (!is_root && !is_leaf) {
      n.Sq.alloc(n.P * n.width, st);
      n.scale_q.alloc(n.P, st);
      // The generalized (weighted) transform is not fused: measured slower
      // (C3, width 20) than the separate heads/tails + warp TSQR.
      const bool pfuse = false;
      if (n.width > 0 && G > n.P && !pfuse) n.ptails.alloc((G - n.P) * n.width, st);
      HeadTailArgs b;
      b.data = n.S.get();
      b.ld = n.width;
      b.w = (int)n.width;
      if (vj) {
        b.data = nullptr;
        b.join = &j;
        b.join_heads = n.S.get();
        b.join_ldh = ldS;
      }
      // identity order (prefix case): rows read in place, no index loads
      b.perm = n.pa_identity ? nullptr : n.pa_perm.get();
      b.begins = n.pa_begins.get();
      b.n_seg = n.P;
      b.n_rows = G;
      b.weights = n.scale.get();
      b.tail_count = n.phi_up.get();
      b.scale_count = n.phi_down.get();
      b.heads = n.width > 0 ? n.Sq.get() : nullptr;
      b.ldh = n.width;
      b.tails = n.ptails.get();
      b.ldt = n.width;
      b.scales = n.scale_q.get();
      if (pfuse) {
        n.pfused_count = run_heads_tails_fused(ctx, b, n.pfused);
        n.pfused_W = fused_width((int)n.width);
      }
      if (!pfuse || n.pfused_count < 0) {
        n.pfused_count = 0;
        if (n.width > 0 && G > n.P && !n.ptails.size()) n.ptails.alloc((G - n.P) * n.width, st);
        b.tails = n.ptails.get();
        kt_ht.begin();
        run_heads_tails(ctx, b);
        kt_ht.end();
        // summary rows read once (join-on-read: the own heads; the
        // children's summaries are L2-resident lookups), parent-key heads
        // and projection tails written once
        double child_rows = 0;
        if (vj)
          for (int c : n.children) child_rows += (double)nodes[c]->P * nodes[c]->width;
        ht_bytes += 8.0 * ((double)G * (vj ? n.w : n.width) + child_rows +
                           (double)n.P * n.width + (double)(G - n.P) * n.width);
      }
      n.sum_S = n.Sq.get();
      n.sum_scale = n.scale_q.get();
    } else {
      n.sum_S = n.S.get();
      n.sum_scale = n.scale.get();
    }
  }
  FG_CUDA(cudaEventRecord(ev.e[4], st));
  tr.mark("figaro enqueue");

  // ---- R0 spans in figaro()'s block order, then K6/K7
  std::vector<SpanInfo>& spans = saved->spans;
  std::function<void(int)> collect = [&](int i) {
    NodeState& n = *nodes[i];
    if (n.tails.size() || n.fused_count)
      spans.push_back({i, lay.node_offset[i], n.rows - n.grp.G, n.w,
                       n.tails.get()});
    for (int c : n.children) collect(c);
    if (n.ptails.size() || n.pfused_count)
      spans.push_back({i, lay.sub_begin[i], n.grp.G - n.P, n.width,
                       n.ptails.get()});
    if (n.parent < 0 && n.width > 0 && n.grp.G > 0)
      spans.push_back({i, lay.sub_begin[i], n.grp.G, n.width, n.S.get()});
  };
  collect(root);
  int64_t r0_rows = 0;
  std::vector<Span> tsq;
  for (const auto& s : spans) {
    r0_rows += s.rows;
    Span sp{s.data, s.rows, s.cols, (int)s.cols, (int)s.col_begin};
    NodeState& sn = *nodes[s.node];
    if (!s.data && s.rows > 0) {
      // Fused spans: own tails are span (node_offset, w); project-away tails
      // are (subtree_begin, width).  Both can share col_begin, so match the
      // row count too.
      const bool own = sn.fused_count && s.col_begin == lay.node_offset[s.node] &&
                       s.cols == sn.w && s.rows == sn.rows - sn.grp.G;
      if (own) {
        sp.partials = sn.fused.get();
        sp.count = sn.fused_count;
        sp.W = sn.fused_W;
      } else if (sn.pfused_count) {
        sp.partials = sn.pfused.get();
        sp.count = sn.pfused_count;
        sp.W = sn.pfused_W;
      }
    }
    if (!sp.partials) tsqr_flops += span_flops((double)s.rows, (double)s.cols);
    tsq.push_back(sp);
  }
  const int N = (int)lay.total;
  tsqr_flops += 2.0 / 3.0 * (double)N * N * N;  // final merge of span factors
  DevArray<double> Rdev;
  double* Rd = R_out;
  if (opt.memory == FG_MEM_HOST) {
    Rdev.alloc((size_t)N * N, st);
    Rd = Rdev.get();
  }
  kt_tsqr.begin();
  tsqr(ctx, tsq, N, Rd);
  kt_tsqr.end();
  tr.mark("tsqr enqueue");
  FG_CUDA(cudaEventRecord(ev.e[5], st));
  if (opt.memory == FG_MEM_HOST && N > 0)
    FG_CUDA(cudaMemcpyAsync(R_out, Rd, sizeof(double) * N * N,
                            cudaMemcpyDeviceToHost, st));
  unsigned status_word = 0;
  FG_CUDA(cudaMemcpyAsync(&status_word, ctx.status.get(), sizeof status_word,
                          cudaMemcpyDeviceToHost, st));
  sync_stream(ctx);
  FG_CUDA(cudaGetLastError());
  tr.mark("final sync");
  raise_status(status_word, "compute_counts");

  if (res) {
    res->data_columns = N;
    int64_t m = 0;
    for (auto& n : nodes) m += n->rows;
    res->input_rows = m;
    res->r0_rows = r0_rows;
    res->seconds_group = ev.ms(1, 2);
    res->seconds_counts = ev.ms(2, 3);
    res->seconds_figaro = ev.ms(3, 4);
    res->seconds_postprocess = ev.ms(4, 5);
    res->seconds_total = ev.ms(0, 5);
    res->kernels = ctx.launches - launches0;
    res->seconds_headtail_kernels = kt_ht.seconds();
    res->seconds_tsqr_kernels = kt_tsqr.seconds();
    res->headtail_launches = (int64_t)kt_ht.ev.size();
    res->headtail_bytes = ht_bytes;
    res->headtail_fused_flops = fused_flops;
    res->tsqr_stage_flops = tsqr_flops;
    res->fused_launches = fused_launches;
    res->host_syncs = ctx.syncs - syncs0;
    res->device_mallocs = ctx.cache.mallocs() - mallocs0;
  }
  // Keep the inspection state; drop the bulky buffers unless R0 is wanted.
  saved->have_r0 = opt.keep_r0 != 0;
  for (auto& n : nodes) {
    n->keys_own.release();
    n->data_own.release();
    n->sel.release();
    if (!opt.keep_r0) {
      n->S.release();
      n->Sq.release();
      n->tails.release();
      n->ptails.release();
      n->fused.release();
      n->pfused.release();
    }
  }
  if (!opt.keep_r0) spans.clear();
  delete ctx.saved;
  ctx.saved = saved.release();
}

// RAII: makes ctx's BlockCache the allocation source of this thread.
struct CacheScope {
  BlockCache* prev;
  explicit CacheScope(Context* c) : prev(current_cache()) { current_cache() = &c->cache; }
  ~CacheScope() { current_cache() = prev; }
};

fg_status guard(fg_ctx* c, const std::function<void()>& f) {
  Context* ctx = reinterpret_cast<Context*>(c);
  if (!ctx) return FG_E_ARG;
  CacheScope scope(ctx);
  try {
    FG_CUDA(cudaSetDevice(ctx->device));
    f();
    ctx->last_error = "ok";
    return FG_OK;
  } catch (const Failure& e) {
    ctx->last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return FG_E_ARG;
  }
}

NodeState& node_at(Context& ctx, int32_t node) {
  if (!ctx.saved) fail(FG_E_ARG, "no pipeline result");
  if (node < 0 || node >= (int)ctx.saved->nodes.size())
    fail(FG_E_ARG, "node index out of range");
  return *ctx.saved->nodes[node];
}

}  // namespace

BlockCache*& current_cache() {
  static thread_local BlockCache* c = nullptr;
  return c;
}

}  // namespace fg

using fg::Context;
using fg::fail;

extern "C" {

int32_t fg_version(void) { return FIGARO_CUDA_VERSION; }

void fg_options_default(fg_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->assume_reduced = 0;
  o->engine = FG_ENGINE_THIN;
  o->memory = FG_MEM_DEVICE;
  o->keep_r0 = 0;
  o->fuse = 1;
}

fg_status fg_ctx_create(int32_t device, fg_ctx** out) {
  if (!out) return FG_E_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return FG_E_CUDA;
  if (device < 0 || device >= n) return FG_E_ARG;
  auto* ctx = new Context();
  ctx->device = device;
  fg::current_cache() = &ctx->cache;
  try {
    FG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    FG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      delete ctx;
      return FG_E_CUDA;  // built for sm_100a only
    }
    ctx->sm_count = prop.multiProcessorCount;
    ctx->smem_optin = prop.sharedMemPerBlockOptin;
    // FG_L2_FETCH=32|64|128: L2 fetch granularity hint (experiments with the
    // permuted 64-byte row gathers); the device default otherwise.
    if (const char* e = getenv("FG_L2_FETCH")) {
      size_t before = 0, after = 0;
      cudaDeviceGetLimit(&before, cudaLimitMaxL2FetchGranularity);
      cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e));
      cudaDeviceGetLimit(&after, cudaLimitMaxL2FetchGranularity);
      fprintf(stderr, "[fg] L2 fetch granularity %zu -> %zu\n", before, after);
    }
    FG_CUDA(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    ctx->stream = ctx->own;
    FG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    // Keep freed pool memory: no OS round trips in steady state.
    cudaMemPool_t pool;
    FG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    FG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    ctx->status.alloc(1, ctx->stream);
    ctx->status.zero();
    FG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (const fg::Failure&) {
    fg::current_cache() = nullptr;
    delete ctx;
    return FG_E_CUDA;
  }
  fg::current_cache() = nullptr;
  *out = reinterpret_cast<fg_ctx*>(ctx);
  return FG_OK;
}

fg_status fg_ctx_destroy(fg_ctx* c) {
  Context* ctx = reinterpret_cast<Context*>(c);
  if (!ctx) return FG_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  fg::current_cache() = &ctx->cache;
  delete ctx->saved;
  ctx->saved = nullptr;
  ctx->status.release();
  ctx->cache.trim();
  fg::current_cache() = nullptr;
  if (ctx->own) {
    cudaStreamSynchronize(ctx->own);
    cudaStreamDestroy(ctx->own);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  delete ctx;
  return FG_OK;
}

fg_status fg_ctx_set_stream(fg_ctx* c, void* s) {
  return fg::guard(c, [&] {
    Context* ctx = reinterpret_cast<Context*>(c);
    // Work already queued on the old stream completes before the switch;
    // the context's own stream lives until fg_ctx_destroy.
    FG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  });
}

void* fg_ctx_stream(fg_ctx* c) {
  Context* ctx = reinterpret_cast<Context*>(c);
  return ctx ? ctx->stream : nullptr;
}

const char* fg_last_error(fg_ctx* c) {
  Context* ctx = reinterpret_cast<Context*>(c);
  return ctx ? ctx->last_error.c_str() : "null context";
}

int64_t fg_kernel_launches(fg_ctx* c) {
  Context* ctx = reinterpret_cast<Context*>(c);
  return ctx ? ctx->launches : 0;
}

fg_status fg_run_pipeline(fg_ctx* c, int32_t n_rel, const fg_relation* rels,
                          int32_t root, const int32_t* parent,
                          const fg_options* options, double* R_out,
                          fg_result* result) {
  return fg::guard(c, [&] {
    fg_options o;
    fg_options_default(&o);
    if (options) o = *options;
    if (!R_out) fail(FG_E_ARG, "R_out is null");
    fg::run(*reinterpret_cast<Context*>(c), n_rel, rels, root, parent, o,
            R_out, result);
  });
}

fg_status fg_get_sizes(fg_ctx* c, int32_t node, int64_t* G, int64_t* P) {
  return fg::guard(c, [&] {
    auto& n = fg::node_at(*reinterpret_cast<Context*>(c), node);
    if (G) *G = n.grp.G;
    if (P) *P = n.parent >= 0 ? n.P : 0;
  });
}

fg_status fg_get_segments(fg_ctx* c, int32_t node, int64_t* begins) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    auto& n = fg::node_at(ctx, node);
    std::vector<int> h(n.grp.G + 1, 0);
    if (n.grp.begins.size())
      FG_CUDA(cudaMemcpy(h.data(), n.grp.begins.get(), h.size() * sizeof(int),
                         cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h.size(); ++i) begins[i] = h[i];
  });
}

fg_status fg_get_keys(fg_ctx* c, int32_t node, int32_t parent_keys,
                      int64_t* out) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    auto& n = fg::node_at(ctx, node);
    const bool par = parent_keys != 0;
    if (par && n.parent < 0) return;
    const int64_t cnt = par ? n.P : n.grp.G;
    fg::PackSpec spec = par ? n.par : n.own;
    if (spec.n == 0 || cnt == 0) return;
    fg::DevArray<int64_t> d(cnt * spec.n, ctx.stream);
    fg::launch_unpack(ctx, par ? n.upk.get() : n.grp.uniq.get(), cnt, spec,
                      d.get());
    FG_CUDA(cudaMemcpyAsync(out, d.get(), d.bytes(), cudaMemcpyDeviceToHost,
                            ctx.stream));
    sync_stream(ctx);
  });
}

fg_status fg_get_counts(fg_ctx* c, int32_t node, int32_t kind, uint64_t* out) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    auto& n = fg::node_at(ctx, node);
    const fg::DevArray<uint64_t>* src = nullptr;
    switch (kind) {
      case FG_ROWS_PER_KEY: src = &n.sizes; break;
      case FG_THETA_DOWN: src = &n.theta; break;
      case FG_FULL_JOIN_SIZE: src = &n.fjs; break;
      case FG_PHI_CIRC: src = &n.circ; break;
      case FG_PHI_DOWN: src = &n.phi_down; break;
      case FG_PHI_UP: src = &n.phi_up; break;
      default: fail(FG_E_ARG, "unknown count kind");
    }
    if (kind >= FG_PHI_DOWN && n.parent < 0) return;
    // phi tables carry 2 P entries (split accumulation, counts.cu): the
    // first P are the final values.
    const int64_t cnt = kind >= FG_PHI_DOWN ? n.P : n.grp.G;
    if (cnt > (int64_t)src->size()) fail(FG_E_ARG, "count table shorter than its keys");
    if (cnt) FG_CUDA(cudaMemcpy(out, src->get(), cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  });
}

fg_status fg_get_permutation(fg_ctx* c, int32_t node, int32_t* out) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    auto& n = fg::node_at(ctx, node);
    if (n.grp.perm.size())
      FG_CUDA(cudaMemcpy(out, n.grp.perm.get(), n.grp.perm.bytes(),
                         cudaMemcpyDeviceToHost));
  });
}

fg_status fg_get_r0_span_count(fg_ctx* c, int32_t* n_spans) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    if (!ctx.saved || !ctx.saved->have_r0) fail(FG_E_ARG, "R0 was not kept");
    *n_spans = (int32_t)ctx.saved->spans.size();
  });
}

fg_status fg_get_r0_span(fg_ctx* c, int32_t idx, int32_t* node,
                         int64_t* col_begin, int64_t* rows, int64_t* cols,
                         double* out) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    if (!ctx.saved || !ctx.saved->have_r0) fail(FG_E_ARG, "R0 was not kept");
    if (idx < 0 || idx >= (int)ctx.saved->spans.size())
      fail(FG_E_ARG, "span index out of range");
    const auto& s = ctx.saved->spans[idx];
    if (node) *node = s.node;
    if (col_begin) *col_begin = s.col_begin;
    if (rows) *rows = s.rows;
    if (cols) *cols = s.cols;
    if (out && s.rows * s.cols) {
      if (!s.data) fail(FG_E_ARG, "final span is not kept");
      FG_CUDA(cudaMemcpy(out, s.data, sizeof(double) * s.rows * s.cols,
                         cudaMemcpyDeviceToHost));
    }
  });
}

fg_status fg_group_keys(fg_ctx* c, const uint64_t* keys, int64_t n,
                        int32_t bits, int32_t* perm, int32_t* begins,
                        uint64_t* uniq, int64_t* G) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    if (bits < 0 || bits > 64) fail(FG_E_ARG, "bits out of range");
    if (n > INT_MAX) fail(FG_E_UNSUPPORTED, "more than 2^31-1 keys");
    fg::GroupOut g;
    if (bits <= 32) {  // the pipeline's narrow-key path (8 bytes per element per pass)
      fg::DevArray<uint32_t> k32(n, ctx.stream);
      fg::launch_narrow(ctx, keys, n, k32.get());
      fg::group_sorted32(ctx, k32.get(), n, bits, nullptr, g);
    } else {
      fg::group_sorted(ctx, keys, n, bits, nullptr, g);
    }
    if (n) {
      FG_CUDA(cudaMemcpyAsync(perm, g.perm.get(), n * sizeof(int),
                              cudaMemcpyDeviceToDevice, ctx.stream));
    }
    FG_CUDA(cudaMemcpyAsync(begins, g.begins.get(), (g.G + 1) * sizeof(int),
                            cudaMemcpyDeviceToDevice, ctx.stream));
    if (g.G)
      FG_CUDA(cudaMemcpyAsync(uniq, g.uniq.get(), g.G * sizeof(uint64_t),
                              cudaMemcpyDeviceToDevice, ctx.stream));
    sync_stream(ctx);
    *G = g.G;
  });
}

fg_status fg_heads_tails(fg_ctx* c, const double* data, int64_t ld, int32_t w,
                         const int32_t* perm, const int32_t* begins,
                         int64_t n_seg, const double* weights,
                         const uint64_t* tail_count, double* heads,
                         int64_t ldh, double* tails, int64_t ldt,
                         double* scales) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    if (n_seg < 0 || w < 0) fail(FG_E_ARG, "negative size");
    int n_rows = 0;
    if (n_seg > 0)
      FG_CUDA(cudaMemcpy(&n_rows, begins + n_seg, sizeof(int),
                         cudaMemcpyDeviceToHost));
    fg::HeadTailArgs a;
    a.data = data;
    a.ld = ld;
    a.w = w;
    a.perm = perm;
    a.begins = begins;
    a.n_seg = n_seg;
    a.n_rows = n_rows;
    a.weights = weights;
    a.tail_count = tail_count;
    a.heads = heads;
    a.ldh = ldh;
    a.tails = tails;
    a.ldt = ldt;
    a.scales = scales;
    fg::run_heads_tails(ctx, a);
    sync_stream(ctx);
  });
}

fg_status fg_tsqr(fg_ctx* c, int32_t n_blocks, const fg_block* blocks,
                  int32_t n, double* R_out) {
  return fg::guard(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    std::vector<fg::Span> spans;
    for (int i = 0; i < n_blocks; ++i) {
      const fg_block& b = blocks[i];
      if (b.col_begin < 0 || b.cols < 0 || b.col_begin + b.cols > n)
        fail(FG_E_ARG, "block exceeds column count");
      spans.push_back({b.data, b.rows, b.ld, b.cols, b.col_begin});
    }
    fg::tsqr(ctx, spans, n, R_out);
    sync_stream(ctx);
  });
}

fg_status fg_join_size(fg_ctx* c, int32_t n_rel, const fg_relation* rels,
                       int32_t root, const int32_t* parent, int32_t memory,
                       uint64_t cap, int64_t* rows) {
  return fg::guard(c, [&] {
    fg::join_rows(*reinterpret_cast<Context*>(c), n_rel, rels, root, parent, memory,
                  cap, nullptr, nullptr, nullptr, rows);
  });
}

fg_status fg_materialize_join(fg_ctx* c, int32_t n_rel, const fg_relation* rels,
                              int32_t root, const int32_t* parent, int32_t memory,
                              uint64_t cap, double* A_out, int64_t* rows) {
  return fg::guard(c, [&] {
    if (!A_out) fail(FG_E_ARG, "A_out is null");
    fg::join_rows(*reinterpret_cast<Context*>(c), n_rel, rels, root, parent, memory,
                  cap, nullptr, A_out, nullptr, rows);
  });
}

fg_status fg_recover_q(fg_ctx* c, int32_t n_rel, const fg_relation* rels,
                       int32_t root, const int32_t* parent, int32_t memory,
                       uint64_t cap, const double* R, double* A_out, double* Q_out,
                       int64_t* rows) {
  return fg::guard(c, [&] {
    if (!R) fail(FG_E_ARG, "recover_q: R is null");
    fg::join_rows(*reinterpret_cast<Context*>(c), n_rel, rels, root, parent, memory,
                  cap, R, A_out, Q_out, rows);
  });
}

fg_status fg_ctx_set_nccl(fg_ctx* c, void* comm) {
  return fg::guard(c, [&] { fg::set_nccl(*reinterpret_cast<Context*>(c), comm); });
}

fg_status fg_gather_r(fg_ctx* c, const double* R_local, int32_t n, int32_t memory,
                      double* R_out) {
  return fg::guard(c, [&] {
    if (!R_local || !R_out) fail(FG_E_ARG, "fg_gather_r: null buffer");
    fg::gather_r(*reinterpret_cast<Context*>(c), R_local, n, memory, R_out);
  });
}

}  // extern "C"
