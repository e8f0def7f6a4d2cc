// figaro_gpu.hpp -- C++ host facade over figaro_cuda.h for code written
// against the reference library (proj/include/figaro/*.hpp).
//
//   #include "figaro/driver.hpp"   // the reference: Relation, JoinTree, ...
//   #include "figaro_gpu.hpp"      // this header
//   figaro::gpu::Device dev(0);
//   auto res = figaro::gpu::run_pipeline(dev, relations, tree, opts);
//   // res.factor.r is the sign-normalised N x N R, as from
//   // figaro::run_pipeline (driver.hpp:47-85).
//
// Templated on the relation / tree / options types so it binds to the
// reference's own classes without depending on their headers: a Relation
// needs name, key_attrs, data_attrs, keys (vector of tuples of
// std::variant<int64_t, std::string>) and data (rows(), cols(), data()); a
// JoinTree needs root and nodes[i].parent.  String-valued keys are
// dictionary-encoded on the host (order-preserving per attribute) before the
// call.  Errors come back as the exception types the caller supplies through
// the `Errors` traits (defaults: std::runtime_error), mirroring error.hpp.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
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

struct Result {
  std::vector<double> r;  // N x N row-major, sign-normalised
  std::size_t n = 0;
  std::size_t r0_rows = 0;
  std::size_t input_rows = 0;
  double seconds_counts = 0, seconds_figaro = 0, seconds_postprocess = 0;
  double seconds_total = 0;
};

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
  std::size_t n = 0;  // total data columns
};

template <class Rel, class Tree>
void marshal(const std::vector<Rel>& rels, const Tree& tree, Marshalled& m) {
  const std::size_t r = rels.size();
  // Per attribute: integer keys pass through; string keys get ranks.
  std::map<std::string, std::vector<std::string>> strings;
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

template <class Rel, class Tree, class Errors = DefaultErrors>
Result run_pipeline(Device& dev, const std::vector<Rel>& rels, const Tree& tree,
                    bool assume_reduced = false) {
  const std::size_t r = rels.size();
  Marshalled m;
  marshal(rels, tree, m);
  auto& desc = m.desc;
  auto& parent = m.parent;
  fg_options o;
  fg_options_default(&o);
  o.assume_reduced = assume_reduced ? 1 : 0;
  o.memory = FG_MEM_HOST;
  const std::size_t n = m.n;
  Result res;
  res.n = n;
  res.r.assign(n * n, 0.0);
  fg_result out{};
  const fg_status st = fg_run_pipeline(dev.ctx, (int32_t)r, desc.data(), tree.root,
                                       parent.data(), &o, res.r.data(), &out);
  if (st != FG_OK) Errors::raise(st, fg_last_error(dev.ctx));
  res.r0_rows = out.r0_rows;
  res.input_rows = out.input_rows;
  res.seconds_counts = out.seconds_counts;
  res.seconds_figaro = out.seconds_figaro;
  res.seconds_postprocess = out.seconds_postprocess;
  res.seconds_total = out.seconds_total;
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

}  // namespace figaro::gpu
