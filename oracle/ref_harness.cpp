// ORACLE / TEST INFRASTRUCTURE ONLY -- never part of the product path.
//
// Harness around the UNMODIFIED reference library (header-only C++20 under
// /root/reference/proj/include).  Compiled by oracle/Makefile into
// oracle/_ref/figaro_ref.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may execute it.
//
// It reads a database in the repo's FGDB binary format (see
// paper_2204_00525_b200/fgdb.py), runs the reference pipeline and writes the
// results in the FGRS binary format, so the GPU path and the reference see the
// same bytes.  Modes:
//
//   run  IN.fgdb OUT.fgrs [--threads T] [--r0] [--reduce] [--householder]
//        [--repeat K] [--budget SECONDS]
//        canonicalize (relation.hpp:127) + build_join_tree (join_tree.hpp:72)
//        + run_pipeline (driver.hpp:47), timing each phase.  With --repeat the
//        pipeline runs K times on the once-canonicalised relations (one
//        "rep=" line per run).
//   materialized IN.fgdb OUT.fgrs
//        householder_oracle (postprocess.hpp:255) of materialize_join
//        (join.hpp:96) -- the quadratic ground truth for small databases.
//   random SEED OUT.fgdb [--max-rows N] [--max-rel R] [--key-domain K]
//          [--max-cols C]
//        random_acyclic_database (testbench.hpp:164), already reduced.
//   ground_truth P Q N1 N2 SEED OUT.fgdb OUT_RFIXED.bin
//        generate_ground_truth (testbench.hpp:51).
//   csv CONFIG OUT.fgrm OUT.txt
//        load_database (join_tree.hpp:432) of a config + CSV files, then
//        run_pipeline with semi-join reduction: R (FGRM) and a text dump of
//        the loaded, canonicalised relations ("name|keys|data" per row, keys
//        as written in the CSV, data as %.17g).
//   q IN.fgdb IN.fgrs OUT.fgrq [--cap N]
//        recover_q (postprocess.hpp:293) with the R stored in IN.fgrs, on the
//        relations as read (not canonicalised): every streamed (a_row, q_row)
//        pair, in for_each_join_row order (join.hpp:47).

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "figaro/driver.hpp"
#include "figaro/join.hpp"
#include "figaro/testbench.hpp"

using namespace figaro;

namespace {

struct Reader {
  std::ifstream in;
  explicit Reader(const std::string& p) : in(p, std::ios::binary) {
    if (!in) throw std::runtime_error("cannot open " + p);
  }
  template <class T>
  T get() {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!in) throw std::runtime_error("truncated input");
    return v;
  }
  std::string str() {
    auto n = get<std::uint32_t>();
    std::string s(n, '\0');
    in.read(s.data(), n);
    return s;
  }
  template <class T>
  void arr(T* p, std::size_t n) {
    in.read(reinterpret_cast<char*>(p), sizeof(T) * n);
    if (!in) throw std::runtime_error("truncated array");
  }
};

struct Writer {
  std::ofstream out;
  explicit Writer(const std::string& p) : out(p, std::ios::binary) {
    if (!out) throw std::runtime_error("cannot write " + p);
  }
  template <class T>
  void put(T v) { out.write(reinterpret_cast<const char*>(&v), sizeof v); }
  void str(const std::string& s) {
    put<std::uint32_t>(static_cast<std::uint32_t>(s.size()));
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
  }
  template <class T>
  void arr(const T* p, std::size_t n) {
    out.write(reinterpret_cast<const char*>(p),
              static_cast<std::streamsize>(sizeof(T) * n));
  }
};

struct Db {
  std::vector<Relation> rels;
  int root = 0;
  std::vector<int> parent;
};

Db read_db(const std::string& path) {
  Reader r(path);
  char magic[8];
  r.arr(magic, 8);
  if (std::memcmp(magic, "FGDB0001", 8) != 0)
    throw std::runtime_error("bad FGDB magic");
  Db db;
  const auto nrel = r.get<std::uint32_t>();
  db.rels.resize(nrel);
  for (auto& rel : db.rels) {
    rel.name = r.str();
    const auto nk = r.get<std::uint32_t>();
    for (std::uint32_t i = 0; i < nk; ++i) rel.key_attrs.push_back(r.str());
    const auto nd = r.get<std::uint32_t>();
    for (std::uint32_t i = 0; i < nd; ++i) rel.data_attrs.push_back(r.str());
    const auto rows = r.get<std::uint64_t>();
    std::vector<std::int64_t> keys(rows * nk);
    r.arr(keys.data(), keys.size());
    rel.keys.resize(rows);
    for (std::uint64_t i = 0; i < rows; ++i) {
      rel.keys[i].resize(nk);
      for (std::uint32_t c = 0; c < nk; ++c) rel.keys[i][c] = keys[i * nk + c];
    }
    rel.data.resize(rows, nd);
    r.arr(rel.data.data(), rows * nd);
  }
  db.root = r.get<std::int32_t>();
  db.parent.resize(nrel);
  r.arr(db.parent.data(), nrel);
  return db;
}

void write_db(const std::string& path, const std::vector<Relation>& rels,
              const JoinTree& tree) {
  Writer w(path);
  w.arr("FGDB0001", 8);
  w.put<std::uint32_t>(static_cast<std::uint32_t>(rels.size()));
  for (const auto& rel : rels) {
    w.str(rel.name);
    w.put<std::uint32_t>(static_cast<std::uint32_t>(rel.key_attrs.size()));
    for (const auto& a : rel.key_attrs) w.str(a);
    w.put<std::uint32_t>(static_cast<std::uint32_t>(rel.data_attrs.size()));
    for (const auto& a : rel.data_attrs) w.str(a);
    w.put<std::uint64_t>(rel.row_count());
    for (const auto& k : rel.keys)
      for (const auto& v : k) w.put<std::int64_t>(std::get<std::int64_t>(v));
    w.arr(rel.data.data(), rel.row_count() * rel.data_attrs.size());
  }
  w.put<std::int32_t>(tree.root);
  for (const auto& n : tree.nodes) w.put<std::int32_t>(n.parent);
}

void put_keys(Writer& w, const KeyTuple& k) {
  for (const auto& v : k) w.put<std::int64_t>(std::get<std::int64_t>(v));
}

// FGRS0001: R, sizes, phase seconds, then per node (index order) the key
// groups and all six count maps in std::map order, then optionally R0.
void write_result(const std::string& path, const std::vector<Relation>& rels,
                  const JoinTree& tree, const PipelineResult& res,
                  double t_canon, double t_total) {
  Writer w(path);
  w.arr("FGRS0001", 8);
  const std::size_t n = res.factor.r.rows();
  w.put<std::uint32_t>(static_cast<std::uint32_t>(rels.size()));
  w.put<std::uint64_t>(n);
  w.arr(res.factor.r.data(), n * n);
  w.put<std::uint64_t>(res.r0_rows);
  w.put<std::uint64_t>(res.input_rows);
  w.put<double>(res.seconds_counts);
  w.put<double>(res.seconds_figaro);
  w.put<double>(res.seconds_postprocess);
  w.put<double>(t_canon);
  w.put<double>(t_total);
  for (std::size_t i = 0; i < rels.size(); ++i) {
    const auto& rel = rels[i];
    const auto& nc = res.counts.node[i];
    const auto groups = rel.key_groups();
    w.put<std::uint64_t>(groups.size());
    for (const auto& g : groups) w.put<std::uint64_t>(g.first);
    w.put<std::uint64_t>(rel.row_count());
    w.put<std::uint32_t>(static_cast<std::uint32_t>(rel.key_attrs.size()));
    for (const auto& [k, v] : nc.rows_per_key) put_keys(w, k);
    for (const auto& [k, v] : nc.rows_per_key) w.put<std::uint64_t>(v);
    for (const auto& [k, v] : nc.theta_down) w.put<std::uint64_t>(v);
    for (const auto& [k, v] : nc.full_join_size) w.put<std::uint64_t>(v);
    for (const auto& [k, v] : nc.phi_circ) w.put<std::uint64_t>(v);
    const auto& pattrs = tree.nodes[i].parent_attrs;
    w.put<std::uint32_t>(static_cast<std::uint32_t>(pattrs.size()));
    for (const auto& a : pattrs) w.str(a);
    w.put<std::uint64_t>(nc.phi_down.size());
    for (const auto& [k, v] : nc.phi_down) put_keys(w, k);
    for (const auto& [k, v] : nc.phi_down) w.put<std::uint64_t>(v);
    for (const auto& [k, v] : nc.phi_up) w.put<std::uint64_t>(v);
  }
  if (res.r0) {
    w.put<std::uint64_t>(res.r0->blocks.size());
    for (const auto& b : res.r0->blocks) {
      w.put<std::int32_t>(b.node);
      w.put<std::uint64_t>(b.col_begin);
      w.put<std::uint64_t>(b.rows.rows());
      w.put<std::uint64_t>(b.rows.cols());
      w.arr(b.rows.data(), b.rows.rows() * b.rows.cols());
    }
  } else {
    w.put<std::uint64_t>(~std::uint64_t{0});
  }
}

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
      .count();
}

int cmd_run(int argc, char** argv) {
  if (argc < 4) throw std::runtime_error("run IN OUT [opts]");
  PipelineOptions opts;
  opts.assume_reduced = true;
  bool keep_r0 = false;
  int repeat = 1;
  double budget = 0.0;
  for (int i = 4; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--threads" && i + 1 < argc)
      opts.threads = static_cast<unsigned>(std::stoul(argv[++i]));
    else if (a == "--repeat" && i + 1 < argc)
      repeat = std::max(1, std::stoi(argv[++i]));
    else if (a == "--budget" && i + 1 < argc)
      budget = std::stod(argv[++i]);
    else if (a == "--r0")
      keep_r0 = true;
    else if (a == "--reduce")
      opts.assume_reduced = false;
    else if (a == "--householder")
      opts.engine = PostprocessEngine::householder;
    else
      throw std::runtime_error("unknown option " + a);
  }
  Db db = read_db(argv[2]);
  auto t0 = std::chrono::steady_clock::now();
  for (auto& rel : db.rels) canonicalize(rel);
  const double t_canon = since(t0);
  JoinTree tree = build_join_tree(db.rels, db.root, db.parent);
  t0 = std::chrono::steady_clock::now();
  // run_pipeline takes the relations by value; the reduced copy is what the
  // counts/segments refer to, so reduce here when asked (driver.hpp:791-794).
  std::vector<Relation> rels = std::move(db.rels);
  if (!opts.assume_reduced) {
    rels = semi_join_reduce(std::move(rels), tree);
    opts.assume_reduced = true;
  }
  double t_total = 0.0;
  PipelineResult res;
  if (repeat <= 1) {
    res = run_pipeline(rels, tree, opts, keep_r0);
    t_total = since(t0);
  } else {
    // --repeat K: the database is loaded and canonicalised once; every
    // repetition copies the relations outside the timer (run_pipeline takes
    // them by value) and times run_pipeline alone.  --budget S stops after
    // the repetition that crosses S seconds of pipeline time.
    double spent = 0.0;
    for (int k = 0; k < repeat; ++k) {
      std::vector<Relation> in = rels;
      const auto tk = std::chrono::steady_clock::now();
      res = run_pipeline(std::move(in), tree, opts, keep_r0);
      const double dt = since(tk);
      std::printf("rep=%d pipeline=%.6f counts=%.6f figaro=%.6f post=%.6f\n", k, dt,
                  res.seconds_counts, res.seconds_figaro, res.seconds_postprocess);
      std::fflush(stdout);
      t_total = dt;
      spent += dt;
      if (budget > 0.0 && spent >= budget) break;
    }
  }
  write_result(argv[3], rels, tree, res, t_canon, t_total);
  std::printf("ok threads=%u M=%zu N=%zu r0_rows=%zu counts=%.6f figaro=%.6f "
              "post=%.6f canon=%.6f pipeline=%.6f\n",
              opts.threads, res.input_rows, res.data_columns, res.r0_rows,
              res.seconds_counts, res.seconds_figaro, res.seconds_postprocess,
              t_canon, t_total);
  return 0;
}

int cmd_materialized(int argc, char** argv) {
  if (argc < 4) throw std::runtime_error("materialized IN OUT");
  Db db = read_db(argv[2]);
  for (auto& rel : db.rels) canonicalize(rel);
  JoinTree tree = build_join_tree(db.rels, db.root, db.parent);
  Layout layout = make_layout(db.rels, tree);
  Matrix a = materialize_join(db.rels, tree, layout, 4'000'000);
  if (a.rows() < a.cols()) {
    Matrix padded(a.cols(), a.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
      for (std::size_t j = 0; j < a.cols(); ++j) padded(i, j) = a(i, j);
    a = std::move(padded);
  }
  Matrix r = householder_oracle(a);
  Writer w(argv[3]);
  w.arr("FGRM0001", 8);
  w.put<std::uint64_t>(r.rows());
  w.arr(r.data(), r.rows() * r.cols());
  std::printf("ok join_rows=%zu N=%zu\n", a.rows(), a.cols());
  return 0;
}

int cmd_random(int argc, char** argv) {
  if (argc < 4) throw std::runtime_error("random SEED OUT [opts]");
  bench::RandomDbSpec spec;
  for (int i = 4; i + 1 < argc; i += 2) {
    std::string a = argv[i];
    const unsigned long v = std::stoul(argv[i + 1]);
    if (a == "--max-rows") spec.max_rows = v;
    else if (a == "--max-rel") spec.max_relations = static_cast<int>(v);
    else if (a == "--min-rel") spec.min_relations = static_cast<int>(v);
    else if (a == "--key-domain") spec.key_domain = static_cast<int>(v);
    else if (a == "--max-cols") spec.max_total_data_cols = v;
    else throw std::runtime_error("unknown option " + a);
  }
  auto db = bench::random_acyclic_database(spec, std::stoull(argv[2]));
  write_db(argv[3], db.relations, db.tree);
  std::printf("ok relations=%zu join_rows=%llu\n", db.relations.size(),
              static_cast<unsigned long long>(db.join_rows));
  return 0;
}

int cmd_ground_truth(int argc, char** argv) {
  if (argc < 9) throw std::runtime_error("ground_truth P Q N1 N2 SEED DB RF");
  auto inst = bench::generate_ground_truth(
      std::stoul(argv[2]), std::stoul(argv[3]), std::stoul(argv[4]),
      std::stoul(argv[5]), std::stoull(argv[6]));
  write_db(argv[7], inst.relations, inst.tree);
  Writer w(argv[8]);
  w.arr("FGRM0001", 8);
  w.put<std::uint64_t>(inst.r_fixed.rows());
  w.arr(inst.r_fixed.data(), inst.r_fixed.rows() * inst.r_fixed.cols());
  std::printf("ok\n");
  return 0;
}

int cmd_csv(int argc, char** argv) {
  if (argc < 5) throw std::runtime_error("csv CONFIG OUT.fgrm OUT.txt");
  std::ifstream cfg_in(argv[2]);
  if (!cfg_in) throw std::runtime_error("cannot open config");
  const std::string cfg_path = argv[2];
  const auto slash = cfg_path.find_last_of('/');
  const std::string base = slash == std::string::npos ? "" : cfg_path.substr(0, slash);
  DatabaseConfig cfg = parse_config(cfg_in);
  Database db = load_database(cfg, base);
  {
    std::ofstream txt(argv[4]);
    for (const auto& rel : db.relations)
      for (std::size_t i = 0; i < rel.row_count(); ++i) {
        txt << rel.name << '|';
        for (std::size_t c = 0; c < rel.keys[i].size(); ++c) {
          if (c) txt << ';';
          const auto& v = rel.keys[i][c];
          if (std::holds_alternative<std::int64_t>(v)) txt << std::get<std::int64_t>(v);
          else txt << std::get<std::string>(v);
        }
        txt << '|';
        for (std::size_t c = 0; c < rel.data.cols(); ++c) {
          if (c) txt << ';';
          char buf[40];
          std::snprintf(buf, sizeof buf, "%.17g", rel.data(i, c));
          txt << buf;
        }
        txt << '\n';
      }
  }
  PipelineOptions opts;
  opts.threads = 1;
  PipelineResult res = run_pipeline(db.relations, db.tree, opts);
  Writer w(argv[3]);
  w.arr("FGRM0001", 8);
  w.put<std::uint64_t>(res.factor.r.rows());
  w.arr(res.factor.r.data(), res.factor.r.rows() * res.factor.r.cols());
  std::printf("ok N=%zu\n", res.factor.r.rows());
  return 0;
}

int cmd_q(int argc, char** argv) {
  if (argc < 5) throw std::runtime_error("q IN.fgdb IN.fgrs OUT.fgrq [--cap N]");
  Db db = read_db(argv[2]);
  std::uint64_t cap = kDefaultJoinCap;
  for (int i = 5; i + 1 < argc; i += 2)
    if (std::string(argv[i]) == "--cap") cap = std::stoull(argv[i + 1]);
  Reader rr(argv[3]);
  char magic[8];
  rr.arr(magic, 8);
  if (std::memcmp(magic, "FGRS0001", 8) != 0) throw std::runtime_error("bad FGRS magic");
  (void)rr.get<std::uint32_t>();
  const auto n = rr.get<std::uint64_t>();
  TriangularFactor f;
  f.r = Matrix(n, n);
  rr.arr(f.r.data(), n * n);
  JoinTree tree = build_join_tree(db.rels, db.root, db.parent);
  Layout layout = make_layout(db.rels, tree);
  std::vector<double> a_rows, q_rows;
  const std::uint64_t rows = recover_q(
      db.rels, tree, layout, f,
      [&](std::span<const double> a, std::span<const double> q) {
        a_rows.insert(a_rows.end(), a.begin(), a.end());
        q_rows.insert(q_rows.end(), q.begin(), q.end());
      },
      cap);
  Writer w(argv[4]);
  w.arr("FGRQ0001", 8);
  w.put<std::uint64_t>(rows);
  w.put<std::uint64_t>(n);
  w.arr(a_rows.data(), a_rows.size());
  w.arr(q_rows.data(), q_rows.size());
  std::printf("ok rows=%llu n=%llu\n", static_cast<unsigned long long>(rows),
              static_cast<unsigned long long>(n));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::runtime_error("usage: figaro_ref MODE ...");
    std::string mode = argv[1];
    if (mode == "run") return cmd_run(argc, argv);
    if (mode == "materialized") return cmd_materialized(argc, argv);
    if (mode == "random") return cmd_random(argc, argv);
    if (mode == "ground_truth") return cmd_ground_truth(argc, argv);
    if (mode == "q") return cmd_q(argc, argv);
    if (mode == "csv") return cmd_csv(argc, argv);
    throw std::runtime_error("unknown mode " + mode);
  } catch (const integrity_error& e) {
    std::fprintf(stderr, "figaro_ref: integrity_error: %s\n", e.what());
    return 3;
  } catch (const size_error& e) {
    std::fprintf(stderr, "figaro_ref: size_error: %s\n", e.what());
    return 4;
  } catch (const parse_error& e) {
    std::fprintf(stderr, "figaro_ref: parse_error: %s\n", e.what());
    return 6;
  } catch (const schema_error& e) {
    std::fprintf(stderr, "figaro_ref: schema_error: %s\n", e.what());
    return 7;
  } catch (const rank_error& e) {
    std::fprintf(stderr, "figaro_ref: rank_error: %s\n", e.what());
    return 5;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "figaro_ref: error: %s\n", e.what());
    return 2;
  }
}
