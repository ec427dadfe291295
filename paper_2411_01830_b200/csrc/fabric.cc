// Topology, bandwidth matrix and Alg. 1 NVLink path selection.
// Restates tubesim topology.py:65-443 and nvlink_sched.py:42-302.
#include <mutex>
#include <tuple>
#include <algorithm>

#include "decisions.h"

namespace ft {

namespace {
bool jint(const JVal& v) { return v.t == JVal::NUM && v.is_int; }
double jnum(const JVal* v, const char* what) {
  if (!v) fail(FT_E_TOPOLOGY, std::string("malformed topology document: '") + what + "'");
  if (v->t == JVal::NUM) return v->n;
  if (v->t == JVal::STR) {
    char* end = nullptr;
    double x = strtod(v->s.c_str(), &end);
    if (end && *end == 0 && !v->s.empty()) return x;
  }
  fail(FT_E_TOPOLOGY, std::string("malformed topology document: bad number for '") + what + "'");
}
const JVal& need(const JVal& o, const char* k) {
  const JVal* v = o.t == JVal::OBJ ? o.get(k) : nullptr;
  if (!v) fail(FT_E_TOPOLOGY, std::string("malformed topology document: '") + k + "'");
  return *v;
}
std::string path_str(const Path& p) {
  std::string s = "[";
  for (size_t i = 0; i < p.size(); ++i) s += (i ? ", " : "") + std::to_string(p[i]);
  return s + "]";
}
void path_json(JsonOut& o, const Path& p) {
  o.raw("[");
  for (size_t i = 0; i < p.size(); ++i) {
    if (i) o.raw(",");
    o.inum(p[i]);
  }
  o.raw("]");
}
}  // namespace

// ------------------------------------------------------------ Topo
struct Topo::CandCache {
  std::mutex mu;
  std::map<std::tuple<int, int, int>, std::vector<Path>> paths;  // node-based: references stay valid
};

std::unique_ptr<Topo> Topo::from_json(const std::string& text) {
  auto t = std::make_unique<Topo>();
  t->cand_cache = std::make_shared<Topo::CandCache>();
  JVal doc = json_parse(text);
  if (doc.t != JVal::OBJ) fail(FT_E_TOPOLOGY, "malformed topology document: not an object");
  const JVal* name = doc.get("name");
  t->name = name && name->t == JVal::STR ? name->s : "custom";
  for (auto& e : need(doc, "links").a) {
    Link l;
    const JVal& k = need(e, "kind");
    l.kind = k.t == JVal::STR ? k.s : "";
    const JVal& ends = need(e, "endpoints");
    if (ends.t != JVal::ARR) fail(FT_E_TOPOLOGY, "malformed topology document: endpoints");
    l.bw = jnum(e.get("bandwidth_gbps"), "bandwidth_gbps");
    const JVal* mult = e.get("multiplicity");
    l.mult = mult ? (int)jnum(mult, "multiplicity") : 1;
    if (l.bw <= 0) fail(FT_E_TOPOLOGY, "link: bandwidth must be > 0");  // topology.py:54-58
    if (l.mult < 1) fail(FT_E_TOPOLOGY, "link: multiplicity must be >= 1");
    if (ends.a.size() != 2 && (l.kind == "nvlink" || l.kind == "nvswitch"))
      fail(FT_E_TOPOLOGY, "malformed topology document: endpoints");
    if (ends.a.size() >= 1) l.a = ends.a[0];
    if (ends.a.size() >= 2) l.b = ends.a[1];
    for (size_t i = 2; i < ends.a.size(); ++i) (void)0;
    t->links.push_back(l);
  }
  t->gpu_count = (int)jnum(&need(doc, "gpu_count"), "gpu_count");
  const JVal& nodes = need(doc, "nodes");
  if (nodes.t != JVal::ARR) fail(FT_E_TOPOLOGY, "malformed topology document: nodes");
  for (auto& n : nodes.a) {
    Node nd;
    nd.id = (int64_t)jnum(&need(n, "id"), "id");
    for (auto& g : need(n, "gpus").a) nd.gpus.push_back((int64_t)jnum(&g, "gpus"));
    t->nodes.push_back(nd);
  }
  const JVal& groups = need(doc, "pcie_groups");
  if (groups.t != JVal::OBJ) fail(FT_E_TOPOLOGY, "malformed topology document: pcie_groups");
  for (auto& kv : groups.o) {
    char* end = nullptr;
    long r = strtol(kv.first.c_str(), &end, 10);
    if (!end || *end) fail(FT_E_TOPOLOGY, "malformed topology document: pcie group key");
    std::vector<int64_t> gs;
    for (auto& g : kv.second.a) gs.push_back((int64_t)jnum(&g, "pcie_groups"));
    bool dup = false;
    for (auto& gr : t->groups)
      if (gr.first == (int)r) { gr.second = gs; dup = true; }
    if (!dup) t->groups.emplace_back((int)r, gs);
  }
  if (const JVal* rates = doc.get("rates")) {
    if (const JVal* x = rates->get("pcie_gbps")) t->pcie = jnum(x, "pcie_gbps");
    if (const JVal* x = rates->get("pcie_pageable_gbps")) t->pageable = jnum(x, "pcie_pageable_gbps");
    if (const JVal* x = rates->get("pcie_peer_gbps")) t->peer = jnum(x, "pcie_peer_gbps");
    if (const JVal* x = rates->get("network_gbps")) t->net = jnum(x, "network_gbps");
  }
  // Topology.__post_init__ (topology.py:79-95)
  for (auto& l : t->links) {
    if (l.kind != "nvlink" && l.kind != "nvswitch") continue;
    if (!jint(l.a) || !jint(l.b)) fail(FT_E_TOPOLOGY, "malformed topology document: nvlink endpoints");
    int a = (int)l.a.n, b = (int)l.b.n;
    auto key = std::make_pair(std::min(a, b), std::max(a, b));
    auto it = t->nv_pos.find(key);
    if (it == t->nv_pos.end()) {
      t->nv_pos[key] = t->nv.size();
      t->nv.push_back({key, 0.0 + l.bw * l.mult});
    } else {
      t->nv[it->second].second += l.bw * l.mult;
    }
    t->nv_kind[key] = l.kind;
  }
  for (auto& n : t->nodes)
    for (auto g : n.gpus) t->gpu_node[g] = n.id;
  for (auto& gr : t->groups)
    for (auto g : gr.second) t->gpu_root[g] = gr.first;
  auto bad = t->validate();
  if (!bad.empty()) {
    std::string m = "invalid topology: ";
    for (auto& b : bad) m += b + "; ";
    fail(FT_E_TOPOLOGY, m);
  }
  return t;
}

std::vector<std::string> Topo::validate() const {
  std::vector<std::string> out;
  std::map<int64_t, int64_t> seen;
  for (auto& n : nodes)
    for (auto g : n.gpus) {
      if (seen.count(g)) out.push_back("gpu " + std::to_string(g) + " assigned to two nodes");
      seen[g] = n.id;
    }
  for (int g = 0; g < gpu_count; ++g)
    if (!seen.count(g)) out.push_back("gpu " + std::to_string(g) + " belongs to no node");
  std::map<int64_t, int> seen_r;
  for (auto& gr : groups)
    for (auto g : gr.second) {
      if (seen_r.count(g)) out.push_back("gpu " + std::to_string(g) + " in two PCIe groups");
      seen_r[g] = gr.first;
    }
  for (int g = 0; g < gpu_count; ++g)
    if (!seen_r.count(g)) out.push_back("gpu " + std::to_string(g) + " has no PCIe group");
  for (auto& l : links)
    for (const JVal* e : {&l.a, &l.b})
      if (jint(*e) && !seen.count((int64_t)e->n))
        out.push_back("link references unknown gpu " + std::to_string((int64_t)e->n));
  return out;
}

void Topo::check(int g) const {
  if (!gpu_node.count(g)) fail(FT_E_TOPOLOGY, "unknown GPU id " + std::to_string(g));
}
int Topo::node_of(int g) const { check(g); return (int)gpu_node.at(g); }
int Topo::root_of(int g) const {
  check(g);
  auto it = gpu_root.find(g);
  if (it == gpu_root.end()) fail(FT_E_KEY, "gpu has no PCIe root");
  return (int)it->second;
}
double Topo::nvlink_gbps(int u, int v) const {
  check(u);
  check(v);
  auto it = nv_pos.find({std::min(u, v), std::max(u, v)});
  return it == nv_pos.end() ? 0.0 : nv[it->second].second;
}
std::vector<int> Topo::neighbors(int g) const {
  check(g);
  std::vector<int> out;
  for (auto& kv : nv) {
    auto [a, b] = kv.first;
    if (a == g) out.push_back(b);
    else if (b == g) out.push_back(a);
  }
  std::sort(out.begin(), out.end());
  return out;
}
int Topo::kind(int u, int v) const {
  auto it = nv_kind.find({std::min(u, v), std::max(u, v)});
  if (it == nv_kind.end()) return 0;
  return it->second == "nvswitch" ? 2 : 1;
}
double Topo::switch_port_gbps(int g) const {
  bool any = false;
  double best = 0.0;
  for (auto& kv : nv) {
    auto [a, b] = kv.first;
    if ((a == g || b == g) && nv_kind.at(kv.first) == "nvswitch") {
      if (!any || kv.second > best) best = kv.second;  // max(): first wins ties
      any = true;
    }
  }
  return any ? best : 0.0;
}
double Topo::degree_gbps(int g) const {
  double p = switch_port_gbps(g);
  if (p > 0) return p;
  PySum s;
  for (auto& kv : nv)
    if (kv.first.first == g || kv.first.second == g) s.add(kv.second);
  return s.value();
}
double Topo::pair_bandwidth(int u, int v) const {
  if (u == v) fail(FT_E_TOPOLOGY, "pair_bandwidth needs two distinct GPUs");
  double c = nvlink_gbps(u, v);
  if (c > 0) return c;
  if (node_of(u) != node_of(v)) return net;
  return peer;
}
std::vector<int> Topo::sorted_roots() const {
  std::vector<int> r;
  for (auto& g : groups) r.push_back(g.first);
  std::sort(r.begin(), r.end());
  return r;
}
const std::vector<int64_t>& Topo::group(int root) const {
  for (auto& g : groups)
    if (g.first == root) return g.second;
  fail(FT_E_KEY, "unknown PCIe root " + std::to_string(root));
}

// ------------------------------------------------------------ Matrix
Matrix::Matrix(const Topo* t) : topo(t) {
  n = t->gpu_count;
  for (auto& kv : t->nv) n = std::max(n, std::max(kv.first.first, kv.first.second) + 1);
  dcap.assign((size_t)n * n, NAN);
  dres.assign((size_t)n * n, NAN);
  for (auto& kv : t->nv) {
    auto [u, v] = kv.first;
    for (auto e : {std::make_pair(u, v), std::make_pair(v, u)}) {
      capacity[e] = kv.second;
      residual[e] = kv.second;
      owners[e];
      dcap[(size_t)e.first * n + e.second] = kv.second;
      dres[(size_t)e.first * n + e.second] = kv.second;
    }
  }
  for (int g = 0; g < t->gpu_count; ++g) {
    double b = t->degree_gbps(g);
    egress[g] = b;
    ingress[g] = b;
  }
}
double Matrix::res(int u, int v) const {
  if (u < 0 || v < 0 || u >= n || v >= n) return 0.0;
  double r = dres[(size_t)u * n + v];
  return std::isnan(r) ? 0.0 : r;
}
bool Matrix::idle(int u, int v) const {
  if (u < 0 || v < 0 || u >= n || v >= n) return false;
  double r = dres[(size_t)u * n + v];
  return !std::isnan(r) && r == dcap[(size_t)u * n + v];
}
void Matrix::hold(const std::string& f, const Path& p, double rate) {
  for (size_t i = 0; i + 1 < p.size(); ++i)
    if (res(p[i], p[i + 1]) + 1e-12 < rate)
      fail(FT_E_TOPOLOGY, "hold over capacity on edge (" + std::to_string(p[i]) + ", " + std::to_string(p[i + 1]) + ")");
  for (size_t i = 0; i + 1 < p.size(); ++i) {
    auto it = residual.find({p[i], p[i + 1]});
    if (it == residual.end()) fail(FT_E_KEY, "hold on a missing edge");
    it->second -= rate;
    dres[(size_t)p[i] * n + p[i + 1]] = it->second;
    owners[{p[i], p[i + 1]}].push_back(f);
  }
  if (!egress.count(p.front()) || !ingress.count(p.back())) fail(FT_E_KEY, "hold endpoint is not a GPU");
  egress[p.front()] -= rate;
  ingress[p.back()] -= rate;
  auto* lst = held.find(f);
  if (!lst) lst = &held.set(f, {});
  lst->push_back({p, rate});
}
void Matrix::give_back(const std::string& f, const Path& p, double rate) {
  for (size_t i = 0; i + 1 < p.size(); ++i) {
    double& r = residual[{p[i], p[i + 1]}];
    r += rate;
    if (p[i] >= 0 && p[i + 1] >= 0 && p[i] < n && p[i + 1] < n) dres[(size_t)p[i] * n + p[i + 1]] = r;
    auto& ow = owners[{p[i], p[i + 1]}];
    auto it = std::find(ow.begin(), ow.end(), f);
    if (it != ow.end()) ow.erase(it);
  }
  egress[p.front()] += rate;
  ingress[p.back()] += rate;
}
void Matrix::release(const std::string& f) {
  auto* lst = held.find(f);
  if (!lst) fail(FT_E_TOPOLOGY, "release without claim for '" + f + "'");
  auto copy = *lst;
  held.erase(f);
  for (auto& pr : copy) give_back(f, pr.first, pr.second);
}
void Matrix::release_path(const std::string& f, const Path& p) {
  auto* lst = held.find(f);
  if (lst) {
    for (size_t i = 0; i < lst->size(); ++i) {
      if ((*lst)[i].first == p) {
        double rate = (*lst)[i].second;
        lst->erase(lst->begin() + i);
        give_back(f, p, rate);
        if (lst->empty()) held.erase(f);
        return;
      }
    }
  }
  fail(FT_E_TOPOLOGY, "'" + f + "' does not hold path " + path_str(p));
}
std::vector<std::string> Matrix::holders(int u, int v) const {
  auto it = owners.find({u, v});
  return it == owners.end() ? std::vector<std::string>{} : it->second;
}
double Matrix::aggregate(const std::string& f) const {
  const auto* lst = held.find(f);
  PySum s;
  if (lst)
    for (auto& pr : *lst) s.add(pr.second);
  return s.value();
}
std::string Matrix::state_json() const {
  JsonOut o;
  o.raw("{\"residual\":[");
  bool first = true;
  for (auto& kv : residual) {
    if (!first) o.raw(",");
    first = false;
    o.raw("[");
    o.inum(kv.first.first);
    o.raw(",");
    o.inum(kv.first.second);
    o.raw(",");
    o.num(kv.second);
    o.raw("]");
  }
  o.raw("],\"egress\":[");
  first = true;
  for (auto& kv : egress) {
    if (!first) o.raw(",");
    first = false;
    o.num(kv.second);
  }
  o.raw("],\"ingress\":[");
  first = true;
  for (auto& kv : ingress) {
    if (!first) o.raw(",");
    first = false;
    o.num(kv.second);
  }
  o.raw("],\"held\":{");
  first = true;
  for (auto& kv : held.items) {
    if (!first) o.raw(",");
    first = false;
    o.str(kv.first);
    o.raw(":[");
    for (size_t i = 0; i < kv.second.size(); ++i) {
      if (i) o.raw(",");
      o.raw("[");
      path_json(o, kv.second[i].first);
      o.raw(",");
      o.num(kv.second[i].second);
      o.raw("]");
    }
    o.raw("]");
  }
  o.raw("}}");
  return o.s;
}

// ------------------------------------------------------------ Alg. 1
static std::vector<Path> enumerate_paths(const Topo& t, int s, int d, int max_hops);

const std::vector<Path>& candidate_paths(const Topo& t, int s, int d, int max_hops) {
  Topo::CandCache* cc = t.cand_cache.get();  // created with the topology (Topo::from_json)
  std::lock_guard<std::mutex> lk(cc->mu);
  auto key = std::make_tuple(s, d, max_hops);
  auto it = cc->paths.find(key);
  if (it == cc->paths.end()) it = cc->paths.emplace(key, enumerate_paths(t, s, d, max_hops)).first;
  return it->second;
}

static std::vector<Path> enumerate_paths(const Topo& t, int s, int d, int max_hops) {
  std::vector<Path> out;
  std::vector<std::pair<int, Path>> stack{{s, Path{s}}};
  while (!stack.empty()) {
    auto [node, path] = stack.back();
    stack.pop_back();
    auto nb = t.neighbors(node);
    for (auto it = nb.rbegin(); it != nb.rend(); ++it) {
      int nxt = *it;
      if (std::find(path.begin(), path.end(), nxt) != path.end()) continue;
      if (nxt == d) {
        Path p = path;
        p.push_back(nxt);
        out.push_back(p);
      } else if ((int)path.size() <= max_hops - 1) {
        Path p = path;
        p.push_back(nxt);
        stack.push_back({nxt, p});
      }
    }
  }
  std::stable_sort(out.begin(), out.end(), [](const Path& a, const Path& b) {
    if (a.size() != b.size()) return a.size() < b.size();
    return a < b;
  });
  return out;
}

namespace {
double bottleneck(const Matrix& m, const Path& p) {
  double b = m.res(p[0], p[1]);
  for (size_t i = 1; i + 1 < p.size(); ++i) b = std::min(b, m.res(p[i], p[i + 1]));
  return b;
}
bool all_idle(const Matrix& m, const Path& p) {
  for (size_t i = 0; i + 1 < p.size(); ++i)
    if (!m.idle(p[i], p[i + 1])) return false;
  return true;
}
bool has_edge(const Path& p, std::pair<int, int> e) {
  for (size_t i = 0; i + 1 < p.size(); ++i)
    if (p[i] == e.first && p[i + 1] == e.second) return true;
  return false;
}
double claimable(const Matrix& m, int s, int d, double b) {
  return std::min(std::min(b, m.egress.at(s)), m.ingress.at(d));
}

bool replan_holder(Matrix& m, const std::string& holder, const std::vector<std::pair<Path, double>>& held,
                   const std::vector<std::pair<int, int>>& forbidden) {  // nvlink_sched.py:173-201
  PySum old;
  for (auto& h : held) old.add(h.second);
  double old_aggregate = old.value();
  for (auto& h : held) m.release_path(holder, h.first);
  std::vector<std::pair<Path, double>> repl;
  double total = 0.0;
  int src = held[0].first.front(), dst = held[0].first.back();
  for (auto& c : candidate_paths(*m.topo, src, dst)) {
    bool bad = false;
    for (size_t i = 0; i + 1 < c.size() && !bad; ++i)
      for (auto& f : forbidden)
        if ((f.first == c[i] && f.second == c[i + 1]) || (f.first == c[i + 1] && f.second == c[i])) bad = true;
    if (bad || !all_idle(m, c)) continue;
    double rate = bottleneck(m, c);
    if (rate <= 1e-9) continue;
    m.hold(holder, c, rate);
    repl.push_back({c, rate});
    total += rate;
    if (total >= old_aggregate - 1e-9) break;
  }
  if (total >= old_aggregate - 1e-9) return true;
  for (auto& r : repl) m.release_path(holder, r.first);
  for (auto& h : held) m.hold(holder, h.first, h.second);
  return false;
}

bool try_split(Matrix& m, const std::string& func, int s, int d, const Path& path, const std::string& holder,
               const std::vector<std::pair<Path, double>>& held, NvPath* out) {  // nvlink_sched.py:204-225
  double direct_q = m.topo->nvlink_gbps(s, d);
  double direct_h = m.topo->nvlink_gbps(held[0].first.front(), held[0].first.back());
  PySum halves;
  for (auto& h : held) halves.add(h.second / 2);
  double new_holder_total = m.aggregate(holder) - halves.value();
  if (new_holder_total + 1e-9 < direct_h) return false;
  double freed = held[0].second / 2;
  for (auto& h : held) freed = std::min(freed, h.second / 2);
  double gained = claimable(m, s, d, freed);
  double current = m.aggregate(func);
  if (current + gained + 1e-9 < direct_q) return false;
  if (gained <= 1e-9) return false;
  for (auto& h : held) {
    m.release_path(holder, h.first);
    m.hold(holder, h.first, h.second / 2);
  }
  m.hold(func, path, gained);
  *out = {path, gained, true};
  return true;
}

bool try_adopt(Matrix& m, const std::string& func, int s, int d, const Path& path, NvPath* out) {  // :142-170
  std::vector<std::pair<int, int>> busy;
  for (size_t i = 0; i + 1 < path.size(); ++i)
    if (!m.idle(path[i], path[i + 1])) busy.push_back({path[i], path[i + 1]});
  if (busy.empty()) return false;
  std::set<std::string> hs;
  for (auto& e : busy)
    for (auto& f : m.holders(e.first, e.second)) hs.insert(f);
  if (hs.empty() || hs.count(func) || hs.size() > 1) return false;
  std::string holder = *hs.begin();
  std::vector<std::pair<Path, double>> held;
  if (auto* lst = m.held.find(holder))
    for (auto& pr : *lst) {
      bool hit = false;
      for (auto& e : busy) hit = hit || has_edge(pr.first, e);
      if (hit) held.push_back(pr);
    }
  if (held.empty()) return false;
  if (replan_holder(m, holder, held, busy)) {
    double rate = claimable(m, s, d, bottleneck(m, path));
    if (rate > 1e-9) {
      m.hold(func, path, rate);
      *out = {path, rate, true};
      return true;
    }
    return false;
  }
  return try_split(m, func, s, d, path, holder, held, out);
}
}  // namespace

std::string SelectTrace::json() const {
  JsonOut o;
  o.raw("{\"candidates_examined\":");
  o.inum(candidates);
  for (auto* ph : {&phase1, &phase2}) {
    o.raw(ph == &phase1 ? ",\"phase1\":[" : ",\"phase2\":[");
    for (size_t i = 0; i < ph->size(); ++i) {
      if (i) o.raw(",");
      o.raw("[");
      path_json(o, (*ph)[i].first);
      o.raw(",");
      o.num((*ph)[i].second);
      o.raw("]");
    }
    o.raw("]");
  }
  if (fallback) {
    o.raw(",\"shared_fallback\":");
    path_json(o, shared);
  }
  o.raw("}");
  return o.s;
}

std::vector<NvPath> select_paths(Matrix& m, const std::string& func, int s, int d, bool allow_busy,
                                 SelectTrace* tr) {  // nvlink_sched.py:64-133
  const Topo& t = *m.topo;
  if (s == d) fail(FT_E_TOPOLOGY, "select_paths needs two distinct GPUs");
  t.check(s);
  t.check(d);
  const auto& cands = candidate_paths(t, s, d);
  SelectTrace local;
  SelectTrace& T = tr ? *tr : local;
  T = SelectTrace{};
  T.candidates = (int)cands.size();
  if (cands.size() > 1000) fail(FT_E_TOPOLOGY, "path search exceeded its candidate bound");
  std::vector<NvPath> chosen;
  if (cands.empty()) return chosen;
  auto open = [&] { return m.egress.at(s) > 1e-9 && m.ingress.at(d) > 1e-9; };
  while (open()) {
    std::vector<std::pair<double, const Path*>> idle;
    for (auto& p : cands)
      if (all_idle(m, p)) idle.push_back({bottleneck(m, p), &p});
    if (idle.empty()) break;
    std::stable_sort(idle.begin(), idle.end(), [](const auto& a, const auto& b) {
      if (a.second->size() != b.second->size()) return a.second->size() < b.second->size();
      if (-a.first != -b.first) return -a.first < -b.first;
      return *a.second < *b.second;
    });
    const Path& p = *idle[0].second;
    double rate = claimable(m, s, d, bottleneck(m, p));
    if (rate <= 1e-9) break;
    m.hold(func, p, rate);
    chosen.push_back({p, rate, true});
    T.phase1.push_back({p, rate});
  }
  if (open() && allow_busy) {
    for (auto& p : cands) {
      if (!open()) break;
      bool dup = false;
      for (auto& c : chosen) dup = dup || c.gpus == p;
      if (dup) continue;
      NvPath got;
      if (try_adopt(m, func, s, d, p, &got)) {
        chosen.push_back(got);
        T.phase2.push_back({got.gpus, got.b_min});
      }
    }
  }
  if (chosen.empty()) {
    auto key = [&](const Path& p) {
      double b = t.nvlink_gbps(p[0], p[1]);
      for (size_t i = 1; i + 1 < p.size(); ++i) b = std::min(b, t.nvlink_gbps(p[i], p[i + 1]));
      return b;
    };
    const Path* best = &cands[0];
    double bk = key(*best);
    for (auto& p : cands) {  // max(): first maximal element wins
      double k = key(p);
      if (k > bk || (k == bk && -(double)p.size() > -(double)best->size())) {
        best = &p;
        bk = k;
      }
    }
    chosen.push_back({*best, bk, false});
    T.fallback = true;
    T.shared = *best;
  }
  return chosen;
}

namespace {
double evict_and_replan(Matrix& m, const std::string& func, std::pair<int, int> edge) {  // :262-285
  std::vector<std::pair<Path, double>> victims;
  if (auto* lst = m.held.find(func))
    for (auto& pr : *lst)
      if (has_edge(pr.first, edge)) victims.push_back(pr);
  double lost = 0.0;
  for (auto& v : victims) {
    m.release_path(func, v.first);
    double regained = 0.0;
    for (auto& c : candidate_paths(*m.topo, v.first.front(), v.first.back())) {
      if (has_edge(c, edge) || !all_idle(m, c)) continue;
      double rate = std::min(bottleneck(m, c), v.second - regained);
      if (rate <= 1e-9) continue;
      m.hold(func, c, rate);
      regained += rate;
      if (regained >= v.second - 1e-9) break;
    }
    lost += std::max(0.0, v.second - regained);
  }
  return lost;
}
}  // namespace

std::string claim_direct(Matrix& m, const std::vector<std::pair<int, int>>& pairs, const std::string& wf) {
  std::vector<std::pair<std::pair<int, int>, double>> resv;
  ODict<double> degraded;
  for (auto [a, b] : pairs) {
    if (m.topo->nvlink_gbps(a, b) <= 0) continue;
    for (auto e : {std::make_pair(a, b), std::make_pair(b, a)}) {
      for (auto& f : m.holders(e.first, e.second)) {
        if (f == wf) continue;
        if (!degraded.find(f)) degraded.set(f, 0.0);
        *degraded.find(f) += evict_and_replan(m, f, e);
      }
    }
    double rate = std::min(m.res(a, b), m.res(b, a));
    if (rate > 1e-9) {
      m.hold(wf, {a, b}, rate);
      m.hold(wf, {b, a}, rate);
      resv.push_back({{a, b}, rate});
    }
  }
  JsonOut o;
  o.raw("{\"reservations\":[");
  for (size_t i = 0; i < resv.size(); ++i) {
    if (i) o.raw(",");
    o.raw("[[");
    o.inum(resv[i].first.first);
    o.raw(",");
    o.inum(resv[i].first.second);
    o.raw("],");
    o.num(resv[i].second);
    o.raw("]");
  }
  o.raw("],\"degraded\":{");
  bool first = true;
  for (auto& kv : degraded.items) {
    if (kv.second <= 1e-9) continue;
    if (!first) o.raw(",");
    first = false;
    o.str(kv.first);
    o.raw(":");
    o.num(kv.second);
  }
  o.raw("}}");
  return o.s;
}

std::vector<int64_t> distribute_chunks(int64_t n, const std::vector<double>& w) {  // :288-302
  if (w.empty()) fail(FT_E_VALUE, "distribute_chunks needs at least one path");
  PySum s;
  for (double x : w) s.add(x);
  double total = s.value();
  if (total <= 0) fail(FT_E_VALUE, "paths carry no bandwidth");
  std::vector<double> raw;
  std::vector<int64_t> cnt;
  for (double x : w) {
    double r = (double)n * x / total;
    raw.push_back(r);
    cnt.push_back((int64_t)r);
  }
  int64_t sum = 0;
  for (auto c : cnt) sum += c;
  int64_t shortfall = n - sum;
  std::vector<size_t> order(w.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    double ka = -(raw[a] - (double)cnt[a]), kb = -(raw[b] - (double)cnt[b]);
    if (ka != kb) return ka < kb;
    return a < b;
  });
  int64_t len = (int64_t)order.size();
  int64_t stop = shortfall >= 0 ? std::min(shortfall, len) : std::max<int64_t>(0, len + shortfall);
  for (int64_t i = 0; i < stop; ++i) cnt[order[i]] += 1;
  return cnt;
}

}  // namespace ft
