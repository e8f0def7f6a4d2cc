// Join enumeration and streaming Q = A R^{-1} on the device -- the steps
// after R.
//
// Restates for_each_join_row (join.hpp:47-92), materialize_join
// (join.hpp:96-112) and recover_q (postprocess.hpp:293-321):
//   * the join rows come in the reference's depth-first order: root rows in
//     input order, then for every node in pre-order the rows of that relation
//     whose parent-shared key equals its parent's current row's, in input
//     order (EdgeIndex keeps row ids in insertion order, join.hpp:29-38);
//   * a row is the concatenation of the relations' data rows in the
//     pre-order column layout;
//   * q solves q R = a by forward substitution with the reference's
//     operation order (acc = a_j - q_0 R_0j - q_1 R_1j - ...; q_j = acc/R_jj),
//     unfused multiply / subtract / divide, so equal inputs give equal bits.
//
// Device plan: per edge, a stable radix grouping of the child's rows by the
// parent-shared key and a binary-search lookup from every parent row; per
// row the number of complete join rows below it (saturating u64, bottom-up);
// the cap check on their sum at the root; then level-by-level expansion of
// row-id tuples in pre-order (only rows with completions, so every partial
// tuple extends to at least one join row and memory stays within the cap);
// finally one warp per join row gathers A and solves for Q.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_reduce.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>

#include "host_tree.hpp"

namespace fg {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxNodes = 64;

struct JNode {
  std::string name;
  int n_key = 0, w = 0;
  int64_t rows = 0;
  std::vector<std::string> key_names, data_names, pattr_names;
  std::vector<int> key_attr, pattr;
  int parent = -1;
  std::vector<int> children;
  const int64_t* keys = nullptr;
  const double* data = nullptr;
  DevArray<int64_t> keys_own;
  DevArray<double> data_own;
  GroupOut grp;               // own rows grouped by the parent-shared key
  DevArray<int> lk;           // parent's rows -> group in grp, or -1
  DevArray<uint64_t> nsub;    // per own row: join rows of its subtree
  DevArray<uint64_t> seg_sum; // per group: sum of nsub
  DevArray<int> live, live_begins;  // grp.perm restricted to nsub > 0
};

struct SatAdd {
  uint64_t lim;
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
    const uint64_t s = a + b;
    return (s < a || s > lim) ? lim : s;
  }
};

__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t b, uint64_t lim) {
  if (a == 0 || b == 0) return 0;
  if (__umul64hi(a, b) != 0) return lim;
  const uint64_t p = a * b;
  return p > lim ? lim : p;
}

struct Kids {
  int n;
  const int* lk[kMaxChildren];
  const uint64_t* S[kMaxChildren];
};

__global__ void k_nsub(int64_t rows, Kids k, uint64_t lim, uint64_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = 1;
    for (int c = 0; c < k.n; ++c) {
      const int s = k.lk[c][r];
      v = s < 0 ? 0 : sat_mul(v, k.S[c][s], lim);
    }
    out[r] = v;
  }
}

__global__ void k_gather_u64(const int* __restrict__ perm, int64_t n,
                             const uint64_t* __restrict__ in, uint64_t* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = in[perm[q]];
}

__global__ void k_live_flags(const int* __restrict__ perm, int64_t n,
                             const uint64_t* __restrict__ nsub, int* __restrict__ flag) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    flag[q] = nsub[perm ? perm[q] : q] > 0 ? 1 : 0;
}

// out[s] = live entries before group s (s = 0..G).
__global__ void k_live_begins(const int* __restrict__ begins, int64_t G,
                              const int* __restrict__ incl, int* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= G;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int b = begins[s];
    out[s] = b == 0 ? 0 : incl[b - 1];
  }
}

__global__ void k_tuple_counts(const int* __restrict__ pid, int64_t T,
                               const int* __restrict__ lk, const int* __restrict__ lb,
                               int64_t* __restrict__ cnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = lk[pid[t]];
    cnt[t] = s < 0 ? 0 : (int64_t)(lb[s + 1] - lb[s]);
  }
}

struct Expand {
  int n;
  const int* src[kMaxNodes];
  int* dst[kMaxNodes];
};

// New tuple o = (old tuple t, j-th live match of the node) where t is the
// last tuple with off[t] <= o.
__global__ void k_expand(const int64_t* __restrict__ off, int64_t T, int64_t T2,
                         const int* __restrict__ pid, const int* __restrict__ lk,
                         const int* __restrict__ lb, const int* __restrict__ live,
                         Expand e, int* __restrict__ dst_new) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < T2;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = T;  // first t with off[t] > o, minus one
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= o) lo = mid + 1; else hi = mid;
    }
    const int64_t t = lo - 1;
    const int64_t j = o - off[t];
    for (int i = 0; i < e.n; ++i) e.dst[i][o] = e.src[i][t];
    const int s = lk[pid[t]];
    dst_new[o] = live[lb[s] + j];
  }
}

struct RowArgs {
  const int* ids[kMaxNodes];
  const double* data[kMaxNodes];
  int w[kMaxNodes];
};

// A only: one thread per element.
__global__ void k_rows_a(RowArgs a, const int* __restrict__ col_node,
                         const int* __restrict__ col_j, int n, int64_t T,
                         double* __restrict__ A) {
  const int64_t total = T * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / n;
    const int c = (int)(e - t * n);
    const int nd = col_node[c];
    A[e] = a.data[nd][(int64_t)a.ids[nd][t] * a.w[nd] + col_j[c]];
  }
}

// One warp per join row: lane l holds columns kb*32 + l.  Forward
// substitution in the reference's order (postprocess.hpp:312-316).
template <int KB>
__global__ void __launch_bounds__(kThreads)
    k_rows_q(RowArgs a, const int* __restrict__ col_node, const int* __restrict__ col_j,
             int n, int64_t T, const double* __restrict__ R, double* __restrict__ A,
             double* __restrict__ Q) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < T; t += nw) {
    double x[KB];
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) {
      const int c = kb * 32 + lane;
      x[kb] = 0.0;
      if (c < n) {
        const int nd = col_node[c];
        x[kb] = a.data[nd][(int64_t)a.ids[nd][t] * a.w[nd] + col_j[c]];
        if (A) A[t * n + c] = x[kb];
      }
    }
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) {
      for (int ii = 0; ii < 32; ++ii) {
        const int i = kb * 32 + ii;
        if (i >= n) break;
        double qi = __shfl_sync(0xffffffffu, x[kb], ii);
        qi = __ddiv_rn(qi, R[(int64_t)i * n + i]);
        if (lane == ii) x[kb] = qi;
#pragma unroll
        for (int k2 = kb; k2 < KB; ++k2) {
          const int c = k2 * 32 + lane;
          if (c > i && c < n)
            x[k2] = __dsub_rn(x[k2], __dmul_rn(qi, R[(int64_t)i * n + c]));
        }
      }
    }
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) {
      const int c = kb * 32 + lane;
      if (c < n) Q[t * n + c] = x[kb];
    }
  }
}

int grid_for(const Context& ctx, int64_t n) {
  const int64_t g = ceil_div(n, kThreads);
  const int64_t cap = (int64_t)ctx.sm_count * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

template <class T>
void to_host_sync(Context& ctx, T* dst, const T* src, size_t n) {
  if (n) FG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
  FG_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace

void join_rows(Context& ctx, int32_t n_rel, const fg_relation* rels, int32_t root,
               const int32_t* parent, int32_t memory, uint64_t cap, const double* R,
               double* A_out, double* Q_out, int64_t* rows_out) {
  if (n_rel <= 0 || !rels || !parent) fail(FG_E_ARG, "no relations");
  if (!rows_out) fail(FG_E_ARG, "rows is null");
  if (Q_out && !R) fail(FG_E_ARG, "recover_q: R is null");
  if (n_rel > kMaxNodes) fail(FG_E_UNSUPPORTED, "join enumeration: more than 64 relations");
  cudaStream_t st = ctx.stream;
  std::vector<std::unique_ptr<JNode>> nodes;
  for (int i = 0; i < n_rel; ++i) {
    const fg_relation& r = rels[i];
    auto n = std::make_unique<JNode>();
    n->name = r.name ? r.name : ("R" + std::to_string(i));
    n->n_key = r.n_key;
    n->w = r.n_data;
    n->rows = r.rows;
    if (r.n_key < 0 || r.n_data < 0 || r.rows < 0)
      fail(FG_E_ARG, "relation " + n->name + ": negative size");
    if (r.rows > INT_MAX)
      fail(FG_E_UNSUPPORTED, "relation " + n->name + ": more than 2^31-1 rows");
    if ((r.rows && r.n_key && !r.keys) || (r.rows && r.n_data && !r.data))
      fail(FG_E_ARG, "relation " + n->name + ": null keys/data");
    for (int k = 0; k < r.n_key; ++k)
      n->key_names.push_back(r.key_attrs && r.key_attrs[k] ? r.key_attrs[k] : "");
    for (int k = 0; k < r.n_data; ++k)
      n->data_names.push_back(r.data_attrs && r.data_attrs[k] ? r.data_attrs[k] : "");
    nodes.push_back(std::move(n));
  }
  std::vector<int> preorder;
  build_tree(nodes, root, parent, preorder);
  validate(nodes);
  const Layout lay = make_layout(nodes, preorder, root);
  const int n = (int)lay.total;

  // recover_q's checks (postprocess.hpp:300-307) before any enumeration.
  std::vector<double> hR;
  if (R) {
    hR.resize((size_t)n * n);
    if (memory == FG_MEM_HOST) {
      std::copy(R, R + hR.size(), hR.begin());
    } else if (!hR.empty()) {
      FG_CUDA(cudaMemcpyAsync(hR.data(), R, hR.size() * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
      FG_CUDA(cudaStreamSynchronize(st));
    }
    double s = 0.0;
    for (double x : hR) s += x * x;
    const double tol = 1e-12 * std::sqrt(s);
    for (int i = 0; i < n; ++i)
      if (!(std::abs(hR[(size_t)i * n + i]) > tol))
        fail(FG_E_RANK, "recover_q: triangular factor is singular at column " +
                            std::to_string(i));
  }
  if (Q_out && n > 128)
    fail(FG_E_UNSUPPORTED, "recover_q: more than 128 data columns");

  for (int i = 0; i < n_rel; ++i) {
    JNode& nd = *nodes[i];
    const fg_relation& r = rels[i];
    if (memory == FG_MEM_HOST) {
      nd.keys_own.alloc(r.rows * r.n_key, st);
      nd.data_own.alloc(r.rows * r.n_data, st);
      if (nd.keys_own.size())
        FG_CUDA(cudaMemcpyAsync(nd.keys_own.get(), r.keys, nd.keys_own.bytes(),
                                cudaMemcpyHostToDevice, st));
      if (nd.data_own.size())
        FG_CUDA(cudaMemcpyAsync(nd.data_own.get(), r.data, nd.data_own.bytes(),
                                cudaMemcpyHostToDevice, st));
      nd.keys = nd.keys_own.get();
      nd.data = nd.data_own.get();
    } else {
      nd.keys = r.keys;
      nd.data = r.data;
    }
  }
  for (int i : preorder)
    if (nodes[i]->rows == 0) {  // some relation is empty: so is the join
      *rows_out = 0;
      return;
    }

  const std::vector<AttrCode> code = encode_attributes(ctx, nodes);
  const uint64_t lim = cap == UINT64_MAX ? cap : cap + 1;
  DevArray<unsigned> scratch_status(1, st);

  // Edges: group each child's rows by the parent-shared key; look every
  // parent row up.
  for (int c : preorder) {
    JNode& ch = *nodes[c];
    if (ch.parent < 0) continue;
    JNode& par = *nodes[ch.parent];
    auto col_in = [](const JNode& x) {
      return [&x](int a) {
        return (int)(std::find(x.key_attr.begin(), x.key_attr.end(), a) - x.key_attr.begin());
      };
    };
    int bits = 0;
    PackSpec sc = make_spec(ch.pattr, code, col_in(ch), &bits, "relation " + ch.name);
    PackSpec sp = make_spec(ch.pattr, code, col_in(par), nullptr, "relation " + par.name);
    DevArray<uint64_t> kc(ch.rows, st), kp(par.rows, st);
    DevArray<int> iota(std::max(ch.rows, par.rows), st);
    launch_pack_keys<uint64_t>(ctx, ch.keys, ch.rows, ch.n_key, sc, kc.get(), iota.get());
    group_sorted(ctx, kc.get(), ch.rows, std::max(bits, 1), iota.get(), ch.grp);
    launch_pack_keys<uint64_t>(ctx, par.keys, par.rows, par.n_key, sp, kp.get(), iota.get());
    PackSpec idn = sc;
    for (int f = 0; f < idn.n; ++f) idn.col[f] = idn.shift[f];
    ch.lk.alloc(par.rows, st);
    launch_lookup(ctx, kp.get(), par.rows, idn, ch.grp.uniq.get(), ch.grp.G, ch.lk.get(),
                  scratch_status.get());
  }

  // Join rows below every row (bottom-up), saturating at cap + 1.
  SatAdd op{lim};
  for (auto it = preorder.rbegin(); it != preorder.rend(); ++it) {
    JNode& nd = *nodes[*it];
    Kids k{};
    if (nd.children.size() > (size_t)kMaxChildren)
      fail(FG_E_UNSUPPORTED, "join enumeration: more than 16 children");
    for (int c : nd.children) {
      k.lk[k.n] = nodes[c]->lk.get();
      k.S[k.n] = nodes[c]->seg_sum.get();
      ++k.n;
    }
    nd.nsub.alloc(nd.rows, st);
    k_nsub<<<grid_for(ctx, nd.rows), kThreads, 0, st>>>(nd.rows, k, lim, nd.nsub.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    if (nd.parent < 0) continue;
    DevArray<uint64_t> g(nd.rows, st);
    k_gather_u64<<<grid_for(ctx, nd.rows), kThreads, 0, st>>>(nd.grp.perm.get(), nd.rows,
                                                               nd.nsub.get(), g.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    nd.seg_sum.alloc(nd.grp.G, st);
    size_t temp = 0;
    const int* b = nd.grp.begins.get();
    FG_CUDA(cub::DeviceSegmentedReduce::Reduce(nullptr, temp, g.get(), nd.seg_sum.get(),
                                               (int)nd.grp.G, b, b + 1, op, uint64_t(0), st));
    DevArray<unsigned char> tmp(temp, st);
    FG_CUDA(cub::DeviceSegmentedReduce::Reduce(tmp.get(), temp, g.get(), nd.seg_sum.get(),
                                               (int)nd.grp.G, b, b + 1, op, uint64_t(0), st));
    ++ctx.launches;
  }
  JNode& rt = *nodes[root];
  uint64_t total = 0;
  {
    DevArray<uint64_t> d_total(1, st);
    size_t temp = 0;
    FG_CUDA(cub::DeviceReduce::Reduce(nullptr, temp, rt.nsub.get(), d_total.get(),
                                      rt.rows, op, uint64_t(0), st));
    DevArray<unsigned char> tmp(temp, st);
    FG_CUDA(cub::DeviceReduce::Reduce(tmp.get(), temp, rt.nsub.get(), d_total.get(),
                                      rt.rows, op, uint64_t(0), st));
    ++ctx.launches;
    to_host_sync(ctx, &total, d_total.get(), 1);
  }
  if (total > cap)  // join.hpp:77-79
    fail(FG_E_SIZE, "join row cap exceeded (" + std::to_string(cap) + " rows)");
  *rows_out = (int64_t)total;
  if ((!A_out && !Q_out) || total == 0) return;

  // Live match lists: grouped rows with at least one completion.
  for (int c : preorder) {
    JNode& ch = *nodes[c];
    if (ch.parent < 0) continue;
    DevArray<int> flag(ch.rows, st), incl(ch.rows, st);
    k_live_flags<<<grid_for(ctx, ch.rows), kThreads, 0, st>>>(ch.grp.perm.get(), ch.rows,
                                                               ch.nsub.get(), flag.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    inclusive_sum_int(ctx, flag.get(), incl.get(), ch.rows);
    ch.live.alloc(ch.rows, st);
    DevArray<int64_t> nsel(1, st);
    size_t temp = 0;
    FG_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, ch.grp.perm.get(), flag.get(),
                                       ch.live.get(), nsel.get(), ch.rows, st));
    DevArray<unsigned char> tmp(temp, st);
    FG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), temp, ch.grp.perm.get(), flag.get(),
                                       ch.live.get(), nsel.get(), ch.rows, st));
    ++ctx.launches;
    ch.live_begins.alloc(ch.grp.G + 1, st);
    k_live_begins<<<grid_for(ctx, ch.grp.G + 1), kThreads, 0, st>>>(
        ch.grp.begins.get(), ch.grp.G, incl.get(), ch.live_begins.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
  }
  // Root tuples, then one expansion per pre-order node.
  std::vector<DevArray<int>> ids(n_rel);
  int64_t T = 0;
  {
    DevArray<int> flag(rt.rows, st), iota(rt.rows, st);
    k_live_flags<<<grid_for(ctx, rt.rows), kThreads, 0, st>>>(nullptr, rt.rows,
                                                               rt.nsub.get(), flag.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    launch_iota(ctx, iota.get(), rt.rows);
    ids[root].alloc(rt.rows, st);
    DevArray<int64_t> nsel(1, st);
    size_t temp = 0;
    FG_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, iota.get(), flag.get(),
                                       ids[root].get(), nsel.get(), rt.rows, st));
    DevArray<unsigned char> tmp(temp, st);
    FG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), temp, iota.get(), flag.get(),
                                       ids[root].get(), nsel.get(), rt.rows, st));
    ++ctx.launches;
    to_host_sync(ctx, &T, nsel.get(), 1);
  }
  for (size_t d = 1; d < preorder.size(); ++d) {
    const int c = preorder[d];
    JNode& ch = *nodes[c];
    DevArray<int64_t> cnt(T, st), off(T, st);
    k_tuple_counts<<<grid_for(ctx, T), kThreads, 0, st>>>(ids[ch.parent].get(), T,
                                                           ch.lk.get(), ch.live_begins.get(),
                                                           cnt.get());
    FG_LAUNCHED(ctx);
    FG_KERNEL_CHECK();
    size_t temp = 0;
    FG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, cnt.get(), off.get(), T, st));
    DevArray<unsigned char> tmp(temp, st);
    FG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), temp, cnt.get(), off.get(), T, st));
    ++ctx.launches;
    int64_t last[2] = {0, 0};
    FG_CUDA(cudaMemcpyAsync(&last[0], off.get() + T - 1, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    FG_CUDA(cudaMemcpyAsync(&last[1], cnt.get() + T - 1, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    FG_CUDA(cudaStreamSynchronize(st));
    const int64_t T2 = last[0] + last[1];
    Expand e{};
    std::vector<DevArray<int>> nxt(n_rel);
    for (size_t k = 0; k < d; ++k) {
      const int m = preorder[k];
      nxt[m].alloc(T2, st);
      e.src[e.n] = ids[m].get();
      e.dst[e.n] = nxt[m].get();
      ++e.n;
    }
    nxt[c].alloc(T2, st);
    if (T2 > 0) {
      k_expand<<<grid_for(ctx, T2), kThreads, 0, st>>>(
          off.get(), T, T2, ids[ch.parent].get(), ch.lk.get(), ch.live_begins.get(),
          ch.live.get(), e, nxt[c].get());
      FG_LAUNCHED(ctx);
      FG_KERNEL_CHECK();
    }
    for (size_t k = 0; k <= d; ++k) ids[preorder[k]] = std::move(nxt[preorder[k]]);
    T = T2;
  }
  if (T != (int64_t)total) fail(FG_E_INTEGRITY, "join enumeration: row count mismatch");
  if (n == 0) return;

  // Rows of A (and Q).
  std::vector<int> h_node(n), h_j(n);
  RowArgs ra{};
  for (int i : preorder) {
    ra.ids[i] = ids[i].get();
    ra.data[i] = nodes[i]->data;
    ra.w[i] = nodes[i]->w;
    for (int j = 0; j < nodes[i]->w; ++j) {
      h_node[lay.node_offset[i] + j] = i;
      h_j[lay.node_offset[i] + j] = j;
    }
  }
  DevArray<int> col_node(n, st), col_j(n, st);
  FG_CUDA(cudaMemcpyAsync(col_node.get(), h_node.data(), n * sizeof(int),
                          cudaMemcpyHostToDevice, st));
  FG_CUDA(cudaMemcpyAsync(col_j.get(), h_j.data(), n * sizeof(int),
                          cudaMemcpyHostToDevice, st));
  const bool host = memory == FG_MEM_HOST;
  DevArray<double> dA, dQ, dR;
  double* A = A_out;
  double* Qd = Q_out;
  if (host && A_out) { dA.alloc(T * n, st); A = dA.get(); }
  if (host && Q_out) { dQ.alloc(T * n, st); Qd = dQ.get(); }
  if (Q_out) {
    dR.alloc((size_t)n * n, st);
    FG_CUDA(cudaMemcpyAsync(dR.get(), hR.data(), dR.bytes(), cudaMemcpyHostToDevice, st));
    const int64_t blocks = std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(T, kThreads / 32), (int64_t)ctx.sm_count * 16));
    const int KB = (n + 31) / 32;
    auto go = [&](auto kern) {
      kern<<<(int)blocks, kThreads, 0, st>>>(ra, col_node.get(), col_j.get(), n, T,
                                             dR.get(), A, Qd);
    };
    if (KB == 1) go(k_rows_q<1>);
    else if (KB == 2) go(k_rows_q<2>);
    else if (KB == 3) go(k_rows_q<3>);
    else go(k_rows_q<4>);
  } else {
    k_rows_a<<<grid_for(ctx, T * n), kThreads, 0, st>>>(ra, col_node.get(), col_j.get(), n,
                                                         T, A);
  }
  FG_LAUNCHED(ctx);
  FG_KERNEL_CHECK();
  if (host && A_out) FG_CUDA(cudaMemcpyAsync(A_out, A, T * n * sizeof(double),
                                             cudaMemcpyDeviceToHost, st));
  if (host && Q_out) FG_CUDA(cudaMemcpyAsync(Q_out, Qd, T * n * sizeof(double),
                                             cudaMemcpyDeviceToHost, st));
  FG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace fg
