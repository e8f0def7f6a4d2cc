// Host-side join-tree helpers shared by the pipeline (pipeline.cu) and the
// join enumeration (join.cu): tree construction and validation
// (join_tree.hpp:72-180), the pre-order column layout (join_tree.hpp:186-219)
// and the per-attribute key encodings behind the packed u64 keys.
#pragma once

#include <algorithm>
#include <climits>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "launchers.cuh"

namespace fg {

// ---------------------------------------------------------------- host tree

template <class Node>
void build_tree(std::vector<std::unique_ptr<Node>>& nodes, int root,
                const int32_t* parent, std::vector<int>& preorder) {
  const int r = (int)nodes.size();
  if (r == 0) fail(FG_E_TREE, "join tree: no relations");
  if (root < 0 || root >= r) fail(FG_E_TREE, "join tree: bad root index");
  for (int i = 0; i < r; ++i) {
    const int p = parent[i];
    nodes[i]->parent = p;
    if (i == root) {
      if (p != -1) fail(FG_E_TREE, "join tree: root cannot have a parent");
      continue;
    }
    if (p < 0 || p >= r)
      fail(FG_E_TREE, "join tree: bad parent index for node " + nodes[i]->name);
    nodes[p]->children.push_back(i);
    // parent_attrs: shared key attributes sorted by name (join_tree.hpp:37-45)
    std::set<std::string> pk(nodes[p]->key_names.begin(),
                             nodes[p]->key_names.end());
    std::vector<std::string> shared;
    for (const auto& k : nodes[i]->key_names)
      if (pk.count(k)) shared.push_back(k);
    std::sort(shared.begin(), shared.end());
    nodes[i]->pattr_names = shared;
  }
  std::vector<int> stack{root};
  std::vector<char> seen(r, 0);
  // Pre-order, children in index order (join_tree.hpp:47-51).
  std::function<void(int)> walk = [&](int n) {
    if (seen[n]) fail(FG_E_TREE, "join tree: not a connected tree");
    seen[n] = 1;
    preorder.push_back(n);
    for (int c : nodes[n]->children) walk(c);
  };
  walk(root);
  if ((int)preorder.size() != r)
    fail(FG_E_TREE, "join tree: not a connected tree");
}

// The checks of join_tree.hpp:104-180 (path property, every key attribute
// shared, data attribute names disjoint from everything else), restated as
// a connectivity count with a depth-based path walk for the error report,
// plus canonicalize's schema checks (relation.hpp:128-146).
template <class Node>
void validate(const std::vector<std::unique_ptr<Node>>& nodes) {
  for (const auto& n : nodes) {
    std::vector<std::string> names = n->key_names;
    names.insert(names.end(), n->data_names.begin(), n->data_names.end());
    std::sort(names.begin(), names.end());
    auto dup = std::adjacent_find(names.begin(), names.end());
    if (dup != names.end())
      fail(FG_E_SCHEMA, "relation " + n->name + ": duplicate attribute '" +
                            *dup + "'");
    for (const auto& s : names)
      if (s.empty())
        fail(FG_E_SCHEMA, "relation " + n->name + ": empty attribute name");
  }
  const int r = (int)nodes.size();
  if (r <= 1) return;
  // Depth of every node; the tree path a -> b is a's ancestor chain up to
  // their lowest common ancestor followed by b's chain back down.
  std::vector<int> depth(r, 0);
  for (int i = 0; i < r; ++i)
    for (int x = nodes[i]->parent; x != -1; x = nodes[x]->parent) ++depth[i];
  std::vector<std::set<std::string>> has(r);
  for (int i = 0; i < r; ++i) has[i].insert(nodes[i]->key_names.begin(), nodes[i]->key_names.end());
  // First node on the path a -> b (in path order) lacking `attr`, or -1.
  auto first_gap = [&](int a, int b, const std::string& attr) {
    std::vector<int> down;  // b's side, collected bottom-up
    int x = a, y = b;
    std::vector<int> up;
    while (depth[x] > depth[y]) { up.push_back(x); x = nodes[x]->parent; }
    while (depth[y] > depth[x]) { down.push_back(y); y = nodes[y]->parent; }
    while (x != y) {
      up.push_back(x);
      down.push_back(y);
      x = nodes[x]->parent;
      y = nodes[y]->parent;
    }
    up.push_back(x);  // the common ancestor
    up.insert(up.end(), down.rbegin(), down.rend());
    for (int n : up)
      if (!has[n].count(attr)) return n;
    return -1;
  };
  // Holders of each key attribute, in relation order.
  std::map<std::string, std::vector<int>> holders;
  for (int i = 0; i < r; ++i)
    for (const auto& k : nodes[i]->key_names) holders[k].push_back(i);
  for (const auto& entry : holders) {
    const std::string& attr = entry.first;
    const std::vector<int>& hs = entry.second;
    if (hs.size() == 1)
      fail(FG_E_TREE, "key attribute '" + attr + "' of relation " + nodes[hs[0]]->name +
                          " is not shared with any other relation");
    // Connected holders <=> (#holders - 1) tree edges between holders; only
    // a disconnected set needs the pairwise search for the reported relation.
    int edges = 0;
    for (int h : hs)
      if (nodes[h]->parent != -1 && has[nodes[h]->parent].count(attr)) ++edges;
    if (edges == (int)hs.size() - 1) continue;
    for (size_t i = 0; i < hs.size(); ++i)
      for (size_t j = i + 1; j < hs.size(); ++j) {
        const int gap = first_gap(hs[i], hs[j], attr);
        if (gap >= 0)
          fail(FG_E_TREE, "path property violated for attribute '" + attr + "': relation " +
                              nodes[gap]->name + " does not contain it");
      }
  }
  // Data attribute names: one owner each, never a key attribute anywhere.
  std::map<std::string, int> owner;
  for (int i = 0; i < r; ++i)
    for (const auto& d : nodes[i]->data_names) {
      const auto ins = owner.insert({d, i});
      if (!ins.second)
        fail(FG_E_SCHEMA, "data attribute '" + d + "' appears in both " +
                              nodes[ins.first->second]->name + " and " + nodes[i]->name);
      if (holders.count(d))
        fail(FG_E_SCHEMA, "attribute '" + d + "' is a data column of " + nodes[i]->name +
                              " but a key column elsewhere");
    }
}

struct Layout {
  int64_t total = 0;
  std::vector<int64_t> node_offset, node_width, sub_begin, sub_end;
};

template <class Node>
Layout make_layout(const std::vector<std::unique_ptr<Node>>& nodes,
                   const std::vector<int>& preorder, int root) {
  Layout l;
  const size_t r = nodes.size();
  l.node_offset.resize(r);
  l.node_width.resize(r);
  l.sub_begin.resize(r);
  l.sub_end.resize(r);
  for (int n : preorder) {
    l.node_offset[n] = l.total;
    l.node_width[n] = nodes[n]->w;
    l.total += nodes[n]->w;
  }
  std::function<int64_t(int)> fill = [&](int n) -> int64_t {
    l.sub_begin[n] = l.node_offset[n];
    int64_t end = l.node_offset[n] + l.node_width[n];
    for (int c : nodes[n]->children) end = fill(c);
    l.sub_end[n] = end;
    return end;
  };
  fill(root);
  return l;
}

// ---------------------------------------------------------------- encoding

struct AttrCode {
  long long min = 0;
  int bits = 0;
};

inline int bitlen(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// Fields of `attrs` (attribute ids, in this order) packed MSB first, taking
// values from source positions given by `src(attr)`.
inline PackSpec make_spec(const std::vector<int>& attrs,
                   const std::vector<AttrCode>& code,
                   const std::function<int(int)>& src, int* total_bits,
                   const std::string& what) {
  PackSpec s{};
  if (attrs.size() > (size_t)kMaxKeyCols)
    fail(FG_E_UNSUPPORTED, what + ": more than 16 key attributes");
  s.n = (int)attrs.size();
  int total = 0;
  for (int a : attrs) total += code[a].bits;
  if (total > 64)
    fail(FG_E_UNSUPPORTED, what + ": key tuple needs " + std::to_string(total) +
                               " bits after range packing (> 64)");
  int pos = total;
  for (int f = 0; f < s.n; ++f) {
    const int a = attrs[f];
    pos -= code[a].bits;
    s.shift[f] = pos;
    s.bits[f] = code[a].bits;
    s.min[f] = code[a].min;
    s.col[f] = src(a);
  }
  if (total_bits) *total_bits = total;
  return s;
}

// Global attribute ids (first appearance order), each node's key_attr
// (declaration order) and pattr (parent-shared, name order), and the
// per-attribute offset encodings from a device min/max pass (one sync).
template <class Node>
std::vector<AttrCode> encode_attributes(Context& ctx,
                                        std::vector<std::unique_ptr<Node>>& nodes) {
  cudaStream_t st = ctx.stream;
  std::map<std::string, int> attr_id;
  for (auto& n : nodes)
    for (const auto& k : n->key_names) {
      auto it = attr_id.emplace(k, (int)attr_id.size()).first;
      n->key_attr.push_back(it->second);
    }
  for (auto& n : nodes)
    for (const auto& k : n->pattr_names) n->pattr.push_back(attr_id.at(k));
  const int n_attr = (int)attr_id.size();
  std::vector<AttrCode> code(n_attr);
  if (n_attr) {
    std::vector<long long> init_min(n_attr, LLONG_MAX), init_max(n_attr, LLONG_MIN);
    DevArray<long long> dmin(n_attr, st), dmax(n_attr, st);
    FG_CUDA(cudaMemcpyAsync(dmin.get(), init_min.data(), dmin.bytes(),
                            cudaMemcpyHostToDevice, st));
    FG_CUDA(cudaMemcpyAsync(dmax.get(), init_max.data(), dmax.bytes(),
                            cudaMemcpyHostToDevice, st));
    std::vector<DevArray<int>> col_attr;
    for (auto& n : nodes) {
      DevArray<int> ca(n->n_key, st);
      if (n->n_key)
        FG_CUDA(cudaMemcpyAsync(ca.get(), n->key_attr.data(), ca.bytes(),
                                cudaMemcpyHostToDevice, st));
      launch_key_minmax(ctx, n->keys, n->rows, n->n_key, ca.get(), dmin.get(),
                        dmax.get());
      col_attr.push_back(std::move(ca));
    }
    std::vector<long long> hmin(n_attr), hmax(n_attr);
    FG_CUDA(cudaMemcpyAsync(hmin.data(), dmin.get(), dmin.bytes(),
                            cudaMemcpyDeviceToHost, st));
    FG_CUDA(cudaMemcpyAsync(hmax.data(), dmax.get(), dmax.bytes(),
                            cudaMemcpyDeviceToHost, st));
    sync_stream(ctx);
    for (int a = 0; a < n_attr; ++a) {
      if (hmin[a] > hmax[a]) { code[a] = {0, 0}; continue; }  // no rows
      code[a].min = hmin[a];
      code[a].bits = bitlen((uint64_t)hmax[a] - (uint64_t)hmin[a]);
    }
  }

  return code;
}

}  // namespace fg
