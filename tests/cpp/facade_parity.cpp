// GPU parity through the C++ facade (include/figaro_gpu.hpp) on the
// reference's own types: random_acyclic_database (testbench.hpp:164) and the
// four-relation fixture shape, reference run_pipeline (driver.hpp:47) vs
// figaro::gpu::run_pipeline.  Test infrastructure: built by oracle/Makefile
// against /root/reference headers; run by tests/test_gpu_parity.py.
#include <cmath>
#include <cstdio>

#include "figaro/driver.hpp"
#include "figaro/join.hpp"
#include "figaro/testbench.hpp"
#include "figaro_gpu.hpp"

namespace {

struct RefErrors {
  [[noreturn]] static void raise(fg_status st, const std::string& m) {
    switch (st) {
      case FG_E_INTEGRITY: throw figaro::integrity_error(m);
      case FG_E_SIZE: throw figaro::size_error(m);
      case FG_E_TREE: throw figaro::tree_error(m);
      case FG_E_SCHEMA: throw figaro::schema_error(m);
      case FG_E_EMPTY_JOIN: throw figaro::empty_join_error(m);
      case FG_E_RANK: throw figaro::rank_error(m);
      default: throw figaro::error(m);
    }
  }
};

double rel_dist(const std::vector<double>& a, const figaro::Matrix& b, bool gram) {
  const std::size_t n = b.rows();
  double diff = 0, ref = 0;
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      double x = 0, y = 0;
      if (gram) {
        for (std::size_t k = 0; k < n; ++k) {
          x += a[k * n + i] * a[k * n + j];
          y += b(k, i) * b(k, j);
        }
      } else {
        x = a[i * n + j];
        y = b(i, j);
      }
      diff += (x - y) * (x - y);
      ref += y * y;
    }
  return ref == 0 ? std::sqrt(diff) : std::sqrt(diff / ref);
}

}  // namespace

int main() {
  figaro::gpu::Device dev(0);
  int bad = 0;
  double worst = 0;
  for (std::uint64_t seed = 1; seed <= 40; ++seed) {
    figaro::bench::RandomDbSpec spec;
    spec.max_rows = 300;
    spec.key_domain = 6;
    auto db = figaro::bench::random_acyclic_database(spec, seed * 31);
    figaro::PipelineOptions opts;
    opts.assume_reduced = true;
    auto ref = figaro::run_pipeline(db.relations, db.tree, opts);
    auto got = figaro::gpu::run_pipeline<figaro::PipelineResult, RefErrors>(
        dev, db.relations, db.tree, opts, /*keep_r0=*/seed % 4 == 0);
    // The whole PipelineResult: counts map by map, column names, sizes.
    bool same_counts = got.counts.node.size() == ref.counts.node.size();
    for (std::size_t i = 0; same_counts && i < ref.counts.node.size(); ++i) {
      const auto& a = got.counts.node[i];
      const auto& b = ref.counts.node[i];
      same_counts = a.rows_per_key == b.rows_per_key && a.theta_down == b.theta_down &&
                    a.full_join_size == b.full_join_size && a.phi_circ == b.phi_circ &&
                    a.phi_down == b.phi_down && a.phi_up == b.phi_up;
    }
    if (!same_counts || got.factor.column_names != ref.factor.column_names ||
        got.data_columns != ref.data_columns ||
        got.counts.total_join_size(db.tree.root) != ref.counts.total_join_size(db.tree.root)) {
      ++bad;
      std::printf("seed %llu: counts / column names differ\n", (unsigned long long)seed);
    }
    if (got.r0) {
      // Same R0 rows in the same order (blocks are spans of the reference's blocks).
      figaro::PipelineResult ref0 = figaro::run_pipeline(db.relations, db.tree, opts, true);
      const figaro::Matrix dg = got.r0->dense(), dr = ref0.r0->dense();
      double diff = 0, nrm = 0;
      bool shape = dg.rows() == dr.rows() && dg.cols() == dr.cols();
      for (std::size_t i = 0; shape && i < dr.rows() * dr.cols(); ++i) {
        diff = std::max(diff, std::abs(dg.data()[i] - dr.data()[i]));
        nrm = std::max(nrm, std::abs(dr.data()[i]));
      }
      if (!shape || diff > 1e-12 * std::max(1.0, nrm)) {
        ++bad;
        std::printf("seed %llu: R0 differs (shape %d, max diff %.3e)\n",
                    (unsigned long long)seed, (int)shape, diff);
      }
    }
    bool full = ref.factor.zero_diagonal_rows.empty();
    for (std::size_t i = 0; i < ref.factor.r.rows() && full; ++i)
      full = std::abs(ref.factor.r(i, i)) > 1e-8 * std::abs(ref.factor.r(0, 0));
    const auto& gr = got.factor.r;
    const double d =
        rel_dist(std::vector<double>(gr.data(), gr.data() + gr.rows() * gr.cols()),
                 ref.factor.r, !full);
    // recover_q with the reference's R: identical (a_row, q_row) streams.
    {
      const figaro::Layout layout = figaro::make_layout(db.relations, db.tree);
      std::vector<double> ra, rq, ga, gq;
      bool ref_rank = false, gpu_rank = false;
      try {
        figaro::recover_q(db.relations, db.tree, layout, ref.factor,
                          [&](std::span<const double> a, std::span<const double> q) {
                            ra.insert(ra.end(), a.begin(), a.end());
                            rq.insert(rq.end(), q.begin(), q.end());
                          });
      } catch (const figaro::rank_error&) {
        ref_rank = true;
      }
      const auto& R = ref.factor.r;
      std::vector<double> rv(R.data(), R.data() + R.rows() * R.cols());
      try {
        figaro::gpu::recover_q<figaro::Relation, figaro::JoinTree, RefErrors>(
            dev, db.relations, db.tree, rv,
            [&](std::span<const double> a, std::span<const double> q) {
              ga.insert(ga.end(), a.begin(), a.end());
              gq.insert(gq.end(), q.begin(), q.end());
            });
      } catch (const figaro::rank_error&) {
        gpu_rank = true;
      }
      if (ref_rank != gpu_rank || ra != ga || rq != gq) {
        ++bad;
        std::printf("seed %llu: recover_q differs (rank %d/%d, rows %zu/%zu)\n",
                    (unsigned long long)seed, (int)ref_rank, (int)gpu_rank, ra.size(),
                    ga.size());
      }
    }
    worst = std::max(worst, d);
    if (d > 1e-10 || got.r0_rows != ref.r0_rows || got.input_rows != ref.input_rows) {
      ++bad;
      std::printf("seed %llu: dist %.3e r0 %zu/%zu\n", (unsigned long long)seed, d,
                  got.r0_rows, ref.r0_rows);
    }
  }
  // Unreduced input: integrity_error through the facade, like the reference.
  figaro::bench::RandomDbSpec spec;
  auto db = figaro::bench::random_acyclic_database(spec, 5);
  db.relations[0].keys.push_back(db.relations[0].keys[0]);
  for (auto& v : db.relations[0].keys.back())
    if (std::holds_alternative<std::int64_t>(v)) v = std::int64_t{987654};
  db.relations[0].data.resize(db.relations[0].keys.size(), db.relations[0].data.cols());
  bool threw = false;
  try {
    figaro::PipelineOptions o;
    o.assume_reduced = true;
    figaro::gpu::run_pipeline<figaro::PipelineResult, RefErrors>(dev, db.relations, db.tree, o);
  } catch (const figaro::integrity_error&) {
    threw = true;
  }
  if (db.relations.size() > 1 && !threw) {
    ++bad;
    std::printf("unreduced input did not raise integrity_error\n");
  }
  std::printf("%s facade parity: 40 databases, worst %.3e\n", bad ? "FAIL" : "PASS", worst);
  return bad ? 1 : 0;
}
