// Data index, transfer-plan dispatch and the managed-stage arbiter.
// Restates tubesim dataplane.py:55-369 and engine.py:116-142, 537-646.
#include <algorithm>
#include <cmath>

#include "decisions.h"

namespace ft {

// ------------------------------------------------------------ DataIndex
double Index::store(int64_t id, int node, int gpu, double size, double now, const std::string& producer,
                    bool resp) {  // dataplane.py:72-83
  std::lock_guard<std::mutex> lk(mu);
  auto& t = local[node];
  if (t.count(id) || table.count(id)) fail(FT_E_DUPLICATE, "data id " + std::to_string(id) + " already stored");
  double vis = sync > 0 ? (double)((int64_t)py_floordiv(now, sync) + 1) * sync : now;
  auto e = std::make_shared<Entry>(Entry{id, size, node, gpu, now, producer, resp, vis});
  t[id] = e;
  table[id] = e;
  return vis;
}
std::shared_ptr<Index::Entry> Index::resolve(int64_t id, int node, double now, double* cost,
                                             double* ready) {  // dataplane.py:85-96
  std::lock_guard<std::mutex> lk(mu);
  auto lt = local.find(node);
  if (lt != local.end()) {
    auto it = lt->second.find(id);
    if (it != lt->second.end()) {
      *cost = local_ms;
      *ready = now;
      return it->second;
    }
  }
  auto it = table.find(id);
  if (it == table.end()) fail(FT_E_MISSING, "data id " + std::to_string(id) + " not found in local or global table");
  *cost = local_ms + global_ms;
  *ready = std::max(now, it->second->visible);
  return it->second;
}
void Index::drop(int64_t id) {  // dataplane.py:98-101
  std::lock_guard<std::mutex> lk(mu);
  auto it = table.find(id);
  if (it == table.end()) return;
  auto e = it->second;
  table.erase(it);
  auto lt = local.find(e->node);
  if (lt != local.end()) lt->second.erase(id);
}
void Index::relocate(int64_t id, int node, int gpu) {  // dataplane.py:103-107
  std::lock_guard<std::mutex> lk(mu);
  auto it = table.find(id);
  if (it == table.end()) fail(FT_E_KEY, "data id " + std::to_string(id) + " not in the global table");
  auto e = it->second;
  auto lt = local.find(e->node);
  if (lt != local.end()) lt->second.erase(id);
  e->node = node;
  e->gpu = gpu;
  local[node][id] = e;
}

// ------------------------------------------------------------ plans
namespace {
const char* kMethod[] = {"intra_gpu", "inter_gpu", "host_gpu", "inter_node"};
const char* kLink[] = {"h2d", "d2h", "nv", "nvp_out", "nvp_in", "net"};
std::vector<LinkId> hop_links(const Topo& t, int u, int v) {  // dataplane.py:128-133
  if (t.kind(u, v) == 2) return {{FT_LINK_NVP_OUT, u, -1}, {FT_LINK_NVP_IN, v, -1}};
  return {{FT_LINK_NV, u, v}};
}
Branch make_branch(std::vector<LinkId> links, double share, std::vector<double> caps, double fill) {
  Branch b;
  b.links = std::move(links);
  b.share = share;
  b.hop_caps = std::move(caps);
  b.fill = fill;
  return b;
}
}  // namespace

double Plan::latency() const {  // dataplane.py:351-369
  double total = fixed;
  for (auto& st : stages) {
    double worst = 0.0;
    for (auto& br : st.branches) {
      double rate;
      if (!is_none(br.reserved)) rate = br.reserved;
      else if (!is_none(br.cap)) rate = br.cap;
      else rate = *std::min_element(br.hop_caps.begin(), br.hop_caps.end());
      double x = ms_for(br.share, rate) + br.fill;
      if (x > worst) worst = x;
    }
    total += worst;
  }
  return total;
}

std::string Plan::json() const {
  JsonOut o;
  o.raw("{\"method\":");
  o.str(kMethod[method]);
  o.raw(",\"size_bytes\":");
  o.num(size);
  o.raw(",\"fixed_ms\":");
  o.num(fixed);
  o.raw(",\"claimed_func\":");
  if (claimed.empty()) o.raw("null");
  else o.str(claimed);
  o.raw(",\"note\":");
  o.str(note);
  o.raw(",\"stages\":[");
  for (size_t s = 0; s < stages.size(); ++s) {
    if (s) o.raw(",");
    o.raw(stages[s].managed ? "{\"managed\":true" : "{\"managed\":false");
    o.raw(",\"pinned_bytes\":");
    o.num(stages[s].pinned);
    o.raw(",\"branches\":[");
    for (size_t b = 0; b < stages[s].branches.size(); ++b) {
      const Branch& br = stages[s].branches[b];
      if (b) o.raw(",");
      o.raw("{\"links\":[");
      for (size_t l = 0; l < br.links.size(); ++l) {
        if (l) o.raw(",");
        o.raw("[");
        o.str(kLink[br.links[l].kind]);
        o.raw(",");
        o.inum(br.links[l].a);
        if (br.links[l].kind != FT_LINK_NVP_OUT && br.links[l].kind != FT_LINK_NVP_IN) {
          o.raw(",");
          o.inum(br.links[l].b);
        }
        o.raw("]");
      }
      o.raw("],\"bytes_share\":");
      o.num(br.share);
      o.raw(",\"cap_gbps\":");
      o.num(br.cap);
      o.raw(",\"reserved_gbps\":");
      o.num(br.reserved);
      o.raw(",\"fill_ms\":");
      o.num(br.fill);
      o.raw(",\"hop_caps\":[");
      for (size_t c = 0; c < br.hop_caps.size(); ++c) {
        if (c) o.raw(",");
        o.num(br.hop_caps[c]);
      }
      o.raw("]}");
    }
    o.raw("]}");
  }
  o.raw("],\"latency\":");
  o.num(latency());
  o.raw("}");
  return o.s;
}

Plan Plane::fetch_plan(int sn, int sg, int dn, int dg, double size) {  // dataplane.py:176-186
  if (sn != dn) return inter_node(sn, sg, dn, dg, size);
  if (sg < 0 && dg < 0) {
    Plan p{FT_INTRA_GPU, size, 0.0};
    p.note = "host-to-host shared memory";
    return p;
  }
  if ((sg < 0) != (dg < 0)) return host_gpu(sn, sg, dn, dg, size);
  if (sg == dg) return Plan{FT_INTRA_GPU, size, map_ms};
  return inter_gpu(sn, sg, dn, dg, size);
}

Plan Plane::host_gpu(int sn, int sg, int dn, int dg, double size) {  // dataplane.py:190-201
  bool into = sg < 0;
  int gpu = into ? dg : sg;
  Stage st;
  st.branches = pcie_branches(dn, gpu, size, into);
  st.managed = s.pcie_sched != 0;
  st.pinned = std::min(size, 2 * chunk);
  Plan p{FT_HOST_GPU, size, 0.0};
  p.stages.push_back(st);
  return p;
}

std::vector<Branch> Plane::pcie_branches(int node, int gpu, double size, bool into) {  // :203-222
  int own = topo->root_of(gpu);
  int kind = into ? FT_LINK_H2D : FT_LINK_D2H;
  std::vector<std::vector<LinkId>> routes{{{kind, node, own}}};
  if (s.parallel_pcie) {
    for (int r : topo->sorted_roots()) {
      if (r == own) continue;
      bool here = false;
      for (auto g : topo->group(r)) here = here || topo->node_of((int)g) == node;
      if (!here) continue;
      std::vector<LinkId> detour;
      if (staging_route(node, r, gpu, into, &detour)) routes.push_back(detour);
    }
  }
  double share = size / (double)routes.size();
  std::vector<Branch> out;
  for (auto& links : routes) {
    std::vector<double> caps;
    for (auto& l : links) caps.push_back(link_cap(l));
    double fill = pipeline_fill_ms(caps, std::min(chunk, share));
    out.push_back(make_branch(links, share, caps, fill));
  }
  return out;
}

bool Plane::staging_route(int node, int root, int gpu, bool into, std::vector<LinkId>* out) {  // :224-241
  std::vector<int64_t> gs = topo->group(root);
  std::sort(gs.begin(), gs.end());
  bool found = false;
  Path best;
  for (auto g : gs) {
    if (topo->node_of((int)g) != node) continue;
    Path p;
    if (nv_route((int)g, gpu, into, &p) && (!found || p.size() < best.size())) {
      best = p;
      found = true;
    }
  }
  if (!found) return false;
  LinkId pcie{into ? FT_LINK_H2D : FT_LINK_D2H, node, root};
  std::vector<LinkId> nvl;
  for (size_t i = 0; i + 1 < best.size(); ++i)
    for (auto& l : hop_links(*topo, best[i], best[i + 1])) nvl.push_back(l);
  out->clear();
  if (into) {
    out->push_back(pcie);
    out->insert(out->end(), nvl.begin(), nvl.end());
  } else {
    *out = nvl;
    out->push_back(pcie);
  }
  return true;
}

bool Plane::nv_route(int a, int b, bool into, Path* out) {  // dataplane.py:243-250
  int src = into ? a : b, dst = into ? b : a;
  for (auto& p : candidate_paths(*topo, src, dst, 2)) {
    bool ok = true;
    for (size_t i = 0; i + 1 < p.size(); ++i) ok = ok && m->res(p[i], p[i + 1]) > 0;
    if (ok) {
      *out = p;
      return true;
    }
  }
  return false;
}

double Plane::link_cap(const LinkId& l) const {  // dataplane.py:252-260
  if (l.kind == FT_LINK_H2D || l.kind == FT_LINK_D2H) return topo->pcie;
  if (l.kind == FT_LINK_NV) return topo->nvlink_gbps(l.a, l.b);
  if (l.kind == FT_LINK_NVP_OUT || l.kind == FT_LINK_NVP_IN) return topo->switch_port_gbps(l.a);
  return topo->net;
}

Plan Plane::inter_gpu(int sn, int sg, int dn, int dg, double size) {  // dataplane.py:264-295
  if (s.host_oriented) {
    double pin = std::min(size, 2 * chunk);
    Stage down, up;
    down.branches = pcie_branches(sn, sg, size, false);
    down.pinned = pin;
    up.branches = pcie_branches(dn, dg, size, true);
    up.pinned = pin;
    Plan p{FT_INTER_GPU, size, 0.0};
    p.stages = {down, up};
    p.note = "staged through host memory";
    return p;
  }
  std::string func = "xfer" + std::to_string(claims++);
  std::vector<NvPath> paths;
  if (s.nvlink_sched) {
    paths = select_paths(*m, func, sg, dg, false, nullptr);
  } else {
    double cap = topo->nvlink_gbps(sg, dg);
    if (cap > 0) paths.push_back({{sg, dg}, cap, false});
  }
  if (paths.empty()) return pcie_peer(sn, sg, dn, dg, size);
  PySum tot;
  bool claimed = false;
  for (auto& p : paths) {
    tot.add(p.b_min);
    claimed = claimed || p.held;
  }
  double total = tot.value();
  Stage st;
  for (auto& p : paths) {
    std::vector<LinkId> links;
    std::vector<double> caps;
    for (size_t i = 0; i + 1 < p.gpus.size(); ++i) {
      for (auto& l : hop_links(*topo, p.gpus[i], p.gpus[i + 1])) links.push_back(l);
      caps.push_back(topo->nvlink_gbps(p.gpus[i], p.gpus[i + 1]));
    }
    double share = size * p.b_min / total;
    Branch b = make_branch(links, share, caps, pipeline_fill_ms(caps, std::min(chunk, share)));
    if (p.held) b.reserved = p.b_min;
    st.branches.push_back(b);
  }
  Plan pl{FT_INTER_GPU, size, 0.0};
  pl.stages.push_back(st);
  if (claimed) pl.claimed = func;
  return pl;
}

Plan Plane::pcie_peer(int sn, int sg, int dn, int dg, double size) {
  // dataplane.py:304-324 as intended (the reference raises NameError here:
  // pipeline_latency is not imported — SURVEY Appendix A1).
  std::vector<LinkId> links{{FT_LINK_D2H, sn, topo->root_of(sg)}, {FT_LINK_H2D, dn, topo->root_of(dg)}};
  double peer = topo->peer, pcie = topo->pcie;
  double ch = std::min(chunk, size);
  Branch b;
  Plan p{FT_INTER_GPU, size, 0.0};
  if (pipeline_latency(size, {peer}, ch) <= pipeline_latency(size, {pcie, pcie}, ch)) {
    b = make_branch(links, size, {peer, peer}, pipeline_fill_ms({peer, peer}, ch));
    b.cap = peer;
    p.note = "pcie peer fallback";
  } else {
    b = make_branch(links, size, {pcie, pcie}, pipeline_fill_ms({pcie, pcie}, ch));
    p.note = "pipelined host staging fallback";
  }
  Stage st;
  st.branches.push_back(b);
  p.stages.push_back(st);
  return p;
}

Plan Plane::inter_node(int sn, int sg, int dn, int dg, double size) {  // dataplane.py:328-344
  std::vector<LinkId> hops;
  if (sg >= 0) hops.push_back({FT_LINK_D2H, sn, topo->root_of(sg)});
  hops.push_back({FT_LINK_NET, sn, dn});
  if (dg >= 0) hops.push_back({FT_LINK_H2D, dn, topo->root_of(dg)});
  std::vector<double> caps;
  for (auto& l : hops) caps.push_back(link_cap(l));
  Plan p{FT_INTER_NODE, size, 0.0};
  if (s.host_oriented) {
    for (size_t i = 0; i < hops.size(); ++i) {
      Stage st;
      st.branches.push_back(make_branch({hops[i]}, size, {caps[i]}, 0.0));
      p.stages.push_back(st);
    }
    p.note = "sequential copies through both hosts";
    return p;
  }
  Stage st;
  st.branches.push_back(make_branch(hops, size, caps, pipeline_fill_ms(caps, std::min(chunk, size))));
  p.stages.push_back(st);
  p.note = "pipelined across nodes";
  return p;
}

void Plane::release_claim(const Plan& p) {  // dataplane.py:346-348
  if (!p.claimed.empty() && m->held.find(p.claimed)) m->release(p.claimed);
}

// ------------------------------------------------------------ Arbiter
double Arbiter::StageSt::next_boundary(double after, double bb) const {  // engine.py:135-142
  if (!started || rate <= 1e-9) return none();
  double dur = ms_for(bb, rate);
  int64_t k = std::max<int64_t>(1, (int64_t)std::floor((after - anchor) / dur + 1e-9) + 1);
  return anchor + (double)k * dur;
}
void Arbiter::begin() {
  if (quiet) return;
  out_ = JsonOut{};
  out_.raw("[");
  first_ = true;
}
void Arbiter::end() {
  if (quiet) return;
  out_.raw("]");
  last_json = out_.s;
}
void Arbiter::emit(const std::string& item) {
  if (quiet) return;
  if (!first_) out_.raw(",");
  first_ = false;
  out_.s += item;
}
void Arbiter::start(double now, const std::string& key, double total, double slo, double infer, double arrival,
                    double per_branch_cap, int n_branches) {  // engine.py:537-575
  begin();
  Demand d;
  try {
    d = make_demand(key, total, slo, infer, arrival);
  } catch (const Error& e) {
    if (e.code != FT_E_INFEASIBLE) throw;
    d = make_demand(key, total, 1e12, 0.0, arrival);
    d.at_risk = true;
    ++risk_flags;
  }
  StageSt st{key, d, n_branches, per_branch_cap * n_branches};
  stages.set(key, st);
  share.demands.set(key, d);
  resync(now);
  end();
}
void Arbiter::finish(double now, const std::string& key) {  // engine.py:558-564
  begin();
  share.demands.erase(key);
  stages.erase(key);
  resync(now);
  end();
}
void Arbiter::set_bw(double now, double bw_all, double link_gbps) {
  begin();
  share.bw_all = bw_all;
  for (auto& kv : stages.items) kv.second.cap = std::max(kv.second.cap, link_gbps * kv.second.n_flows);
  resync(now);
  end();
}
void Arbiter::boundary(double now, const std::string& key) {  // engine.py:637-646
  begin();
  StageSt* m = stages.find(key);
  if (m) {
    m->armed = none();
    if (!is_none(m->pending)) {
      PySum others;
      for (auto& kv : stages.items)
        if (kv.second.started && kv.second.key != key) others.add(kv.second.rate);
      set_rate(now, *m, std::min(m->pending, std::max(0.0, share.bw_all - others.value())));
    }
    resync(now);
  }
  end();
}
void Arbiter::resync(double now) {  // engine.py:581-612
  ODict<double> targets = partition(share, now);
  if (!quiet) {
    JsonOut o;
    o.raw("[\"partition\",{");
    for (size_t i = 0; i < targets.items.size(); ++i) {
      if (i) o.raw(",");
      o.str(targets.items[i].first);
      o.raw(":");
      o.num(targets.items[i].second);
    }
    o.raw("}]");
    emit(o.s);
  }
  PySum cs;
  for (auto& kv : stages.items)
    if (kv.second.started) cs.add(kv.second.rate);
  double committed = cs.value();
  std::vector<StageSt*> order;
  std::vector<double> slack;
  for (auto& kv : stages.items) order.push_back(&kv.second);
  std::vector<size_t> idx(order.size());
  for (size_t i = 0; i < idx.size(); ++i) {
    idx[i] = i;
    slack.push_back(order[i]->demand.slack(now));
  }
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    if (slack[a] != slack[b]) return slack[a] < slack[b];
    if (order[a]->demand.arrival != order[b]->demand.arrival) return order[a]->demand.arrival < order[b]->demand.arrival;
    return order[a]->demand.func < order[b]->demand.func;
  });
  double leftover = 0.0;
  for (size_t j : idx) {
    StageSt& m = *order[j];
    const double* tg = targets.find(m.demand.func);
    double target = (tg ? *tg : 0.0) + leftover;
    double want = std::min(target, m.cap);
    leftover = std::max(0.0, target - want);
    if (!m.started) {
      double headroom = share.bw_all - committed;
      double rate = std::min(want, headroom);
      if (rate > 1e-9 && (rate >= want - 1e-9 || committed <= 1e-9)) {
        set_rate(now, m, rate);
        committed += rate;
      } else {
        double b = none();
        for (auto* x : order) {
          double nb = x->next_boundary(now, batch_bytes);
          if (!is_none(nb) && (is_none(b) || nb < b)) b = nb;
        }
        if (!is_none(b)) arm(now, m, b);
      }
    } else if (std::fabs(want - m.rate) > 1e-6) {
      m.pending = want;
      if (!quiet) {
        JsonOut o;
        o.raw("[\"pending\",");
        o.str(m.key);
        o.raw(",");
        o.num(want);
        o.raw("]");
        emit(o.s);
      }
      arm(now, m, m.next_boundary(now, batch_bytes));
    }
  }
}
void Arbiter::set_rate(double now, StageSt& m, double rate) {  // engine.py:614-622
  m.rate = rate;
  m.started = true;
  m.pending = none();
  m.anchor = now;
  if (quiet) return;
  JsonOut o;
  o.raw("[\"set_rate\",");
  o.str(m.key);
  o.raw(",");
  o.num(rate);
  o.raw(",");
  o.num(rate / m.n_flows);
  o.raw("]");
  emit(o.s);
}
void Arbiter::arm(double now, StageSt& m, double t) {  // engine.py:628-635
  if (is_none(t) || t <= now + 1e-9) return;
  if (!is_none(m.armed) && m.armed <= t + 1e-9) return;
  m.armed = t;
  if (quiet) return;
  JsonOut o;
  o.raw("[\"arm\",");
  o.str(m.key);
  o.raw(",");
  o.num(t);
  o.raw("]");
  emit(o.s);
}
std::string Arbiter::state_json() const {
  JsonOut o;
  o.raw("{");
  for (size_t i = 0; i < stages.items.size(); ++i) {
    const StageSt& m = stages.items[i].second;
    if (i) o.raw(",");
    o.str(m.key);
    o.raw(":[");
    o.num(m.rate);
    o.raw(m.started ? ",true," : ",false,");
    o.num(m.pending);
    o.raw(",");
    o.num(m.anchor);
    o.raw(",");
    o.num(m.armed);
    o.raw("]");
  }
  o.raw("}");
  return o.s;
}

}  // namespace ft
