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

template <class Rel, class Tree, class Errors = DefaultErrors>
Result run_pipeline(Device& dev, const std::vector<Rel>& rels, const Tree& tree,
                    bool assume_reduced = false) {
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
  std::vector<std::vector<int64_t>> keys(r);
  std::vector<std::vector<const char*>> kn(r), dn(r);
  std::vector<fg_relation> desc(r);
  std::vector<int32_t> parent(r);
  for (std::size_t i = 0; i < r; ++i) {
    const auto& rel = rels[i];
    const std::size_t nk = rel.key_attrs.size();
    keys[i].resize(rel.keys.size() * nk);
    for (std::size_t row = 0; row < rel.keys.size(); ++row)
      for (std::size_t c = 0; c < nk; ++c) {
        const auto& kv = rel.keys[row][c];
        if (std::holds_alternative<std::string>(kv)) {
          const auto& v = strings[rel.key_attrs[c]];
          keys[i][row * nk + c] =
              std::lower_bound(v.begin(), v.end(), std::get<std::string>(kv)) - v.begin();
        } else {
          keys[i][row * nk + c] = std::get<int64_t>(kv);
        }
      }
    for (const auto& a : rel.key_attrs) kn[i].push_back(a.c_str());
    for (const auto& a : rel.data_attrs) dn[i].push_back(a.c_str());
    desc[i] = fg_relation{rel.name.c_str(), (int32_t)nk, kn[i].data(),
                          (int32_t)rel.data.cols(), dn[i].data(),
                          (int64_t)rel.keys.size(), keys[i].data(), rel.data.data()};
    parent[i] = tree.nodes[i].parent;
  }
  fg_options o;
  fg_options_default(&o);
  o.assume_reduced = assume_reduced ? 1 : 0;
  o.memory = FG_MEM_HOST;
  std::size_t n = 0;
  for (const auto& rel : rels) n += rel.data.cols();
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

}  // namespace figaro::gpu
