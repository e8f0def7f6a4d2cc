// figaro_gpu.hpp -- C++ host facade over figaro_cuda.h for code written
// against the reference library (proj/include/figaro/*.hpp).
//
//   #include "figaro/driver.hpp"   // the reference: Relation, JoinTree, ...
//   #include "figaro_gpu.hpp"      // this header
//   figaro::PipelineResult res = figaro::gpu::run_pipeline<figaro::PipelineResult>(
//       figaro::gpu::default_device(), relations, tree, opts, keep_r0);
//
// The call has the shape of figaro::run_pipeline (driver.hpp:47-85) with a
// leading Device and the result type as the first template argument: it
// returns the caller's PipelineResult filled exactly like the reference's
// (driver.hpp:33-43) -- factor {r, column_names, zero_diagonal_rows},
// r0_rows, input_rows, data_columns, seconds_counts / _figaro /
// _postprocess, counts (CountTables with all six maps of every node,
// counts.hpp:24-41) and, with keep_r0, r0 (AlmostTriangular, figaro.hpp:29-76;
// one OutBlock per R0 span = the reference's blocks of one (node, col_begin)
// stacked in its order, so dense(), row_count() and gram_product() agree).
//
// Templated on the relation / tree / options / result types so it binds to
// the reference's own classes without depending on their headers.  String
// keys are dictionary-encoded on the host (order-preserving per attribute)
// and decoded again in the count tables.  Errors come back as the exception
// types the caller supplies through the `Errors` traits (default:
// std::runtime_error, which run()'s catch (const std::exception&) reports
// like the reference's own errors).
//
// Multi-GPU from C++: one process (or thread) per GPU, each with its own
// Device and an NCCL communicator attached with attach_nccl(); gather_r()
// all-gathers the per-rank factors and merges them on the device
// (fg_gather_r).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "figaro_cuda.h"

namespace figaro::gpu {

struct Device {
  fg_ctx* ctx = nullptr;
  explicit Device(int device = 0) {
    if (fg_ctx_create(device, &ctx) != FG_OK)
      throw std::runtime_error("figaro::gpu: no usable sm_100 device");
  }
  ~Device() { fg_ctx_destroy(ctx); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
};

// Process-wide device for call sites that have none in scope (the one-line
// swap inside driver.hpp:run()).  FIGARO_GPU_DEVICE selects
// the ordinal (default 0).
inline Device& default_device() {
  static Device dev([] {
    const char* e = std::getenv("FIGARO_GPU_DEVICE");
    return e ? std::atoi(e) : 0;
  }());
  return dev;
}

// Default error mapping: one std::runtime_error for every status.  Pass the
// reference's classes to get figaro::integrity_error etc.
struct DefaultErrors {
  [[noreturn]] static void raise(fg_status, const std::string& msg) {
    throw std::runtime_error(msg);
  }
};

// Flat C-ABI description of reference relations (keys encoded as int64).
struct Marshalled {
  std::vector<std::vector<int64_t>> keys;
  std::vector<std::vector<const char*>> kn, dn;
  std::vector<fg_relation> desc;
  std::vector<int32_t> parent;
  std::map<std::string, std::vector<std::string>> strings;  // per attribute
  std::size_t n = 0;  // total data columns
};

template <class Rel, class Tree>
void marshal(const std::vector<Rel>& rels, const Tree& tree, Marshalled& m) {
  const std::size_t r = rels.size();
  // Per attribute: integer keys pass through; string keys get ranks.
  auto& strings = m.strings;
  for (const auto& rel : rels)
    for (std::size_t c = 0; c < rel.key_attrs.size(); ++c)
      for (const auto& k : rel.keys)
        if (std::holds_alternative<std::string>(k[c]))
          strings[rel.key_attrs[c]].push_back(std::get<std::string>(k[c]));
  for (auto& [a, v] : strings) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  m.keys.assign(r, {});
  m.kn.assign(r, {});
  m.dn.assign(r, {});
  m.desc.assign(r, fg_relation{});
  m.parent.assign(r, -1);
  for (std::size_t i = 0; i < r; ++i) {
    const auto& rel = rels[i];
    const std::size_t nk = rel.key_attrs.size();
    auto& keys = m.keys[i];
    keys.resize(rel.keys.size() * nk);
    for (std::size_t row = 0; row < rel.keys.size(); ++row)
      for (std::size_t c = 0; c < nk; ++c) {
        const auto& kv = rel.keys[row][c];
        if (std::holds_alternative<std::string>(kv)) {
          const auto& v = strings[rel.key_attrs[c]];
          keys[row * nk + c] =
              std::lower_bound(v.begin(), v.end(), std::get<std::string>(kv)) - v.begin();
        } else {
          keys[row * nk + c] = std::get<int64_t>(kv);
        }
      }
    for (const auto& a : rel.key_attrs) m.kn[i].push_back(a.c_str());
    for (const auto& a : rel.data_attrs) m.dn[i].push_back(a.c_str());
    m.desc[i] = fg_relation{rel.name.c_str(), (int32_t)nk, m.kn[i].data(),
                            (int32_t)rel.data.cols(), m.dn[i].data(),
                            (int64_t)rel.keys.size(), keys.data(), rel.data.data()};
    m.parent[i] = tree.nodes[i].parent;
    m.n += rel.data.cols();
  }
}

namespace detail {

template <class Errors>
void check(Device& dev, fg_status st) {
  if (st != FG_OK) Errors::raise(st, fg_last_error(dev.ctx));
}

// One count table of a node as the caller's CountMap (std::map<KeyTuple,
// u64>), keys decoded back to int64 / string values of `attrs`.
template <class CountMap, class Errors>
void fill_map(Device& dev, const Marshalled& m, int node, const std::vector<std::string>& attrs,
              const std::vector<int64_t>& keys, int kind, std::size_t count, CountMap& out) {
  using KeyTuple = typename CountMap::key_type;
  using KeyValue = typename KeyTuple::value_type;
  std::vector<uint64_t> v(count);
  if (count) check<Errors>(dev, fg_get_counts(dev.ctx, node, kind, v.data()));
  const std::size_t nk = attrs.size();
  out.clear();
  for (std::size_t g = 0; g < count; ++g) {
    KeyTuple k;
    k.reserve(nk);
    for (std::size_t c = 0; c < nk; ++c) {
      const int64_t x = keys[g * nk + c];
      auto it = m.strings.find(attrs[c]);
      if (it != m.strings.end()) k.push_back(KeyValue{it->second[(std::size_t)x]});
      else k.push_back(KeyValue{x});
    }
    out.emplace_hint(out.end(), std::move(k), v[g]);  // ascending key order
  }
}

}  // namespace detail

// figaro::run_pipeline (driver.hpp:47-85) on the GPU.  `opts` is the
// reference's PipelineOptions: assume_reduced and engine are honoured (both
// engines run the device TSQR), threads is ignored (the device decides).
template <class PipelineResult, class Errors = DefaultErrors, class Rel, class Tree, class Opts>
PipelineResult run_pipeline(Device& dev, const std::vector<Rel>& relations, const Tree& tree,
                            const Opts& opts, bool keep_r0 = false) {
  const std::size_t r = relations.size();
  Marshalled m;
  marshal(relations, tree, m);
  fg_options o;
  fg_options_default(&o);
  o.assume_reduced = opts.assume_reduced ? 1 : 0;
  o.engine = static_cast<int32_t>(opts.engine);  // PostprocessEngine{thin, householder}
  o.memory = FG_MEM_HOST;
  o.keep_r0 = keep_r0 ? 1 : 0;
  o.fuse = keep_r0 ? 0 : 1;  // fused tails never reach HBM, so R0 needs fuse off
  const std::size_t n = m.n;
  std::vector<double> rbuf(n * n, 0.0);
  fg_result out{};
  detail::check<Errors>(dev, fg_run_pipeline(dev.ctx, (int32_t)r, m.desc.data(), tree.root,
                                             m.parent.data(), &o, rbuf.data(), &out));
  PipelineResult res;
  using Matrix = std::decay_t<decltype(res.factor.r)>;
  res.factor.r = Matrix(n, n);
  std::copy(rbuf.begin(), rbuf.end(), res.factor.r.data());
  for (int node : tree.preorder)
    for (const auto& a : relations[node].data_attrs)
      res.factor.column_names.push_back(relations[node].name + "." + a);
  for (std::size_t i = 0; i < n; ++i)
    if (rbuf[i * n + i] == 0.0) res.factor.zero_diagonal_rows.push_back(i);
  res.r0_rows = (std::size_t)out.r0_rows;
  res.input_rows = (std::size_t)out.input_rows;
  res.data_columns = (std::size_t)out.data_columns;
  res.seconds_counts = out.seconds_group + out.seconds_counts;  // grouping = counts' scans
  res.seconds_figaro = out.seconds_figaro;
  res.seconds_postprocess = out.seconds_postprocess;

  // CountTables (counts.hpp:33-41): every node's six maps in key order.
  res.counts.node.resize(r);
  res.counts.scans.assign(r, 1u);  // one pass over each relation's rows
  using CountMap = std::decay_t<decltype(res.counts.node[0].rows_per_key)>;
  for (std::size_t i = 0; i < r; ++i) {
    int64_t G = 0, P = 0;
    detail::check<Errors>(dev, fg_get_sizes(dev.ctx, (int32_t)i, &G, &P));
    const auto& ka = relations[i].key_attrs;
    const auto& pa = tree.nodes[i].parent_attrs;
    std::vector<int64_t> ok((std::size_t)G * ka.size()), pk((std::size_t)P * pa.size());
    if (!ok.empty()) detail::check<Errors>(dev, fg_get_keys(dev.ctx, (int32_t)i, 0, ok.data()));
    if (!pk.empty()) detail::check<Errors>(dev, fg_get_keys(dev.ctx, (int32_t)i, 1, pk.data()));
    auto& nc = res.counts.node[i];
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, ka, ok, FG_ROWS_PER_KEY, G, nc.rows_per_key);
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, ka, ok, FG_THETA_DOWN, G, nc.theta_down);
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, ka, ok, FG_FULL_JOIN_SIZE, G,
                                       nc.full_join_size);
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, ka, ok, FG_PHI_CIRC, G, nc.phi_circ);
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, pa, pk, FG_PHI_DOWN, P, nc.phi_down);
    detail::fill_map<CountMap, Errors>(dev, m, (int)i, pa, pk, FG_PHI_UP, P, nc.phi_up);
  }

  if (keep_r0) {
    using AT = typename std::decay_t<decltype(res.r0)>::value_type;
    AT at;
    at.columns = n;
    int32_t spans = 0;
    detail::check<Errors>(dev, fg_get_r0_span_count(dev.ctx, &spans));
    for (int32_t s = 0; s < spans; ++s) {
      int32_t node = 0;
      int64_t cb = 0, rows = 0, cols = 0;
      detail::check<Errors>(dev, fg_get_r0_span(dev.ctx, s, &node, &cb, &rows, &cols, nullptr));
      typename decltype(at.blocks)::value_type b;
      b.node = node;
      b.col_begin = (std::size_t)cb;
      b.rows = Matrix((std::size_t)rows, (std::size_t)cols);
      if (rows > 0 && cols > 0)
        detail::check<Errors>(dev, fg_get_r0_span(dev.ctx, s, nullptr, nullptr, nullptr, nullptr,
                                                  b.rows.data()));
      at.blocks.push_back(std::move(b));
    }
    res.r0 = std::move(at);
  }
  return res;
}

// recover_q (postprocess.hpp:293-321) on the device: streams every join row
// (for_each_join_row order, join.hpp:47-92) and its Q = A R^-1 row to
// sink(a_row, q_row); `r` is the n x n factor, row-major.  Returns the row
// count.  Singular R -> FG_E_RANK, more than `cap` rows -> FG_E_SIZE, both
// before the sink sees a row.
template <class Rel, class Tree, class Errors = DefaultErrors, class Sink>
std::uint64_t recover_q(Device& dev, const std::vector<Rel>& rels, const Tree& tree,
                        const std::vector<double>& r, Sink&& sink,
                        std::uint64_t cap = 1'000'000) {
  Marshalled m;
  marshal(rels, tree, m);
  if (r.size() != m.n * m.n) Errors::raise(FG_E_ARG, "recover_q: factor size does not match column layout");
  int64_t rows = 0;
  fg_status st = fg_recover_q(dev.ctx, (int32_t)rels.size(), m.desc.data(), tree.root,
                              m.parent.data(), FG_MEM_HOST, cap, r.data(), nullptr,
                              nullptr, &rows);
  if (st != FG_OK) Errors::raise(st, fg_last_error(dev.ctx));
  std::vector<double> a((std::size_t)rows * m.n), q((std::size_t)rows * m.n);
  if (rows && m.n) {
    st = fg_recover_q(dev.ctx, (int32_t)rels.size(), m.desc.data(), tree.root,
                      m.parent.data(), FG_MEM_HOST, cap, r.data(), a.data(), q.data(), &rows);
    if (st != FG_OK) Errors::raise(st, fg_last_error(dev.ctx));
  }
  for (int64_t i = 0; i < rows; ++i)
    sink(std::span<const double>(a.data() + i * m.n, m.n),
         std::span<const double>(q.data() + i * m.n, m.n));
  return (std::uint64_t)rows;
}

// Multi-GPU: attach this rank's NCCL communicator (ncclComm_t) to the
// device's context, then merge every rank's factor into the global R.
template <class Errors = DefaultErrors>
void attach_nccl(Device& dev, void* nccl_comm) {
  detail::check<Errors>(dev, fg_ctx_set_nccl(dev.ctx, nccl_comm));
}

// All-gathers the per-rank n x n factors (host, row-major) and returns the
// merged, sign-normalised global R (one final small QR).
template <class Errors = DefaultErrors>
std::vector<double> gather_r(Device& dev, const std::vector<double>& r_local, std::size_t n) {
  std::vector<double> out(n * n, 0.0);
  detail::check<Errors>(dev, fg_gather_r(dev.ctx, r_local.data(), (int32_t)n, FG_MEM_HOST,
                                         out.data()));
  return out;
}

}  // namespace figaro::gpu
