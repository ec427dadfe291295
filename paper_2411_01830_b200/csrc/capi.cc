// extern "C" boundary for the decision side (include/faastube.h).
#include <cmath>
#include <cstring>
#include <map>

#include "decisions.h"

using namespace ft;

struct ft_topo { std::unique_ptr<Topo> t; };
struct ft_matrix { Matrix m; };
struct ft_pcie_state { PcieState s; };
struct ft_ring { Ring r; };
struct ft_hist { Hist h; };
struct ft_pool_policy { PoolPolicy p; };
struct ft_index { Index x; };
struct ft_plane {
  Plane p;
  // route stream pairs per GPU (the tube's per-transfer CE pairs), for ft_h2g_routes
  std::map<int, std::vector<std::pair<void*, void*>>> pairs;
};
struct ft_plan { Plan p; };
struct ft_arbiter { Arbiter a; };

#define FT_TRY try {
#define FT_CATCH                                   \
  }                                                \
  catch (const ft::Error& e) {                     \
    ft::set_last_error(e.what());                  \
    return e.code;                                 \
  }                                                \
  catch (const std::bad_alloc&) {                  \
    ft::set_last_error("out of host memory");      \
    return FT_E_OOM;                               \
  }                                                \
  catch (const std::exception& e) {                \
    ft::set_last_error(e.what());                  \
    return FT_E_VALUE;                             \
  }                                                \
  return FT_OK;

#define NEED(p)                                            \
  if (!(p)) {                                              \
    ft::set_last_error("null argument: " #p);              \
    return FT_E_VALUE;                                     \
  }

static int put_count(int want, int cap, int* n) {
  if (n) *n = want;
  if (want > cap) {
    ft::set_last_error("output array too small");
    return FT_E_TRUNCATED;
  }
  return FT_OK;
}
static std::string sfunc(const char* f) { return f ? std::string(f) : std::string(); }
static Path to_path(const int32_t* p, int n) { return Path(p, p + n); }

extern "C" {

const char* ft_version(void) { return "faastube-b200 0.1 (sm_100a)"; }

// ---------------------------------------------------------------- topology
int ft_topo_create(const char* json_doc, ft_topo** out) {
  NEED(json_doc);
  NEED(out);
  FT_TRY
  auto* t = new ft_topo{Topo::from_json(json_doc)};
  *out = t;
  FT_CATCH
}
void ft_topo_destroy(ft_topo* t) { delete t; }
int ft_topo_gpu_count(const ft_topo* t, int* out) {
  NEED(t);
  *out = t->t->gpu_count;
  return FT_OK;
}
int ft_topo_node_of(const ft_topo* t, int gpu, int* out) { NEED(t); FT_TRY *out = t->t->node_of(gpu); FT_CATCH }
int ft_topo_root_of(const ft_topo* t, int gpu, int* out) { NEED(t); FT_TRY *out = t->t->root_of(gpu); FT_CATCH }
int ft_topo_nvlink_gbps(const ft_topo* t, int u, int v, double* out) { NEED(t); FT_TRY *out = t->t->nvlink_gbps(u, v); FT_CATCH }
int ft_topo_neighbors(const ft_topo* t, int gpu, int32_t* out, int cap, int* n) {
  NEED(t);
  FT_TRY
  auto nb = t->t->neighbors(gpu);
  int rc = put_count((int)nb.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < nb.size(); ++i) out[i] = nb[i];
  FT_CATCH
}
int ft_topo_pair_kind(const ft_topo* t, int u, int v, int* out) { NEED(t); FT_TRY *out = t->t->kind(u, v); FT_CATCH }
int ft_topo_switch_port_gbps(const ft_topo* t, int gpu, double* out) { NEED(t); FT_TRY *out = t->t->switch_port_gbps(gpu); FT_CATCH }
int ft_topo_degree_gbps(const ft_topo* t, int gpu, double* out) { NEED(t); FT_TRY *out = t->t->degree_gbps(gpu); FT_CATCH }
int ft_topo_pair_bandwidth(const ft_topo* t, int u, int v, double* out) { NEED(t); FT_TRY *out = t->t->pair_bandwidth(u, v); FT_CATCH }
int ft_topo_rate(const ft_topo* t, int which, double* out) {
  NEED(t);
  switch (which) {
    case 0: *out = t->t->pcie; return FT_OK;
    case 1: *out = t->t->pageable; return FT_OK;
    case 2: *out = t->t->peer; return FT_OK;
    case 3: *out = t->t->net; return FT_OK;
  }
  ft::set_last_error("unknown rate selector");
  return FT_E_VALUE;
}
int ft_topo_roots(const ft_topo* t, int32_t* roots, int cap, int* n) {
  NEED(t);
  auto r = t->t->sorted_roots();
  int rc = put_count((int)r.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < r.size(); ++i) roots[i] = r[i];
  return FT_OK;
}

// ---------------------------------------------------------------- matrix
int ft_matrix_create(const ft_topo* t, ft_matrix** out) { NEED(t); FT_TRY *out = new ft_matrix{Matrix(t->t.get())}; FT_CATCH }
void ft_matrix_destroy(ft_matrix* m) { delete m; }
int ft_matrix_hold(ft_matrix* m, const char* func, const int32_t* path, int n, double rate) {
  NEED(m);
  FT_TRY
  if (n < 2) fail(FT_E_VALUE, "path needs at least two GPUs");
  m->m.hold(sfunc(func), to_path(path, n), rate);
  FT_CATCH
}
int ft_matrix_release(ft_matrix* m, const char* func) { NEED(m); FT_TRY m->m.release(sfunc(func)); FT_CATCH }
int ft_release_paths(ft_matrix* m, const char* func) { return ft_matrix_release(m, func); }
int ft_matrix_release_path(ft_matrix* m, const char* func, const int32_t* path, int n) {
  NEED(m);
  FT_TRY m->m.release_path(sfunc(func), to_path(path, n)); FT_CATCH
}
int ft_matrix_residual(const ft_matrix* m, int u, int v, double* out) { NEED(m); *out = m->m.res(u, v); return FT_OK; }
int ft_matrix_budgets(const ft_matrix* m, int gpu, double* eg, double* in) {
  NEED(m);
  auto e = m->m.egress.find(gpu);
  if (e == m->m.egress.end()) {
    ft::set_last_error("unknown GPU id");
    return FT_E_TOPOLOGY;
  }
  if (eg) *eg = e->second;
  if (in) *in = m->m.ingress.at(gpu);
  return FT_OK;
}
int ft_matrix_aggregate_of(const ft_matrix* m, const char* func, double* out) {
  NEED(m);
  *out = m->m.aggregate(sfunc(func));
  return FT_OK;
}
int ft_matrix_state_json(const ft_matrix* m, char* buf, size_t cap, size_t* need) {
  NEED(m);
  FT_TRY return emit_json(m->m.state_json(), buf, cap, need); FT_CATCH
}

// ---------------------------------------------------------------- nvlink
static void fill_nvpath(ft_nvpath* o, const Path& p, double b, bool held) {
  memset(o, 0, sizeof *o);
  o->n = (int32_t)p.size();
  for (size_t i = 0; i < p.size() && i < FT_MAX_PATH; ++i) o->gpus[i] = p[i];
  o->held = held;
  o->b_min_gbps = b;
}
int ft_candidate_paths(const ft_topo* t, int src, int dst, int max_hops, ft_nvpath* out, int cap, int* n) {
  NEED(t);
  FT_TRY
  auto c = candidate_paths(*t->t, src, dst, max_hops);
  int rc = put_count((int)c.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < c.size(); ++i) fill_nvpath(&out[i], c[i], 0.0, false);
  FT_CATCH
}
int ft_select_paths(ft_matrix* m, const char* func, int src, int dst, int allow_busy, ft_nvpath* out, int cap,
                    int* n, char* trace_json, size_t trace_cap) {
  NEED(m);
  FT_TRY
  SelectTrace tr;
  auto ps = select_paths(m->m, sfunc(func), src, dst, allow_busy != 0, &tr);
  if (trace_json) {
    int rc = emit_json(tr.json(), trace_json, trace_cap, nullptr);
    if (rc) return rc;
  }
  int rc = put_count((int)ps.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < ps.size(); ++i) fill_nvpath(&out[i], ps[i].gpus, ps[i].b_min, ps[i].held);
  FT_CATCH
}
int ft_claim_direct(ft_matrix* m, const int32_t* pairs, int npairs, const char* func, char* buf, size_t cap,
                    size_t* need) {
  NEED(m);
  FT_TRY
  std::vector<std::pair<int, int>> ps;
  for (int i = 0; i < npairs; ++i) ps.push_back({pairs[2 * i], pairs[2 * i + 1]});
  return emit_json(claim_direct(m->m, ps, sfunc(func)), buf, cap, need);
  FT_CATCH
}
int ft_distribute_chunks(int64_t chunk_count, const double* b, int npaths, int64_t* counts) {
  FT_TRY
  auto c = distribute_chunks(chunk_count, std::vector<double>(b, b + npaths));
  for (size_t i = 0; i < c.size(); ++i) counts[i] = c[i];
  FT_CATCH
}

// ---------------------------------------------------------------- pcie
int ft_min_rate(double b, double slo, double infer, double* out) { FT_TRY *out = min_rate(b, slo, infer); FT_CATCH }
int ft_pcie_state_create(double bw, int bc, int64_t chunk, ft_pcie_state** out) {
  FT_TRY *out = new ft_pcie_state{PcieState{bw, bc, chunk, {}}}; FT_CATCH
}
void ft_pcie_state_destroy(ft_pcie_state* s) { delete s; }
int ft_pcie_state_add(ft_pcie_state* s, const char* func, double bytes, double slo, double infer, double arrival) {
  NEED(s);
  FT_TRY s->s.demands.set(sfunc(func), make_demand(sfunc(func), bytes, slo, infer, arrival)); FT_CATCH
}
int ft_pcie_state_remove(ft_pcie_state* s, const char* func) { NEED(s); s->s.demands.erase(sfunc(func)); return FT_OK; }
int ft_pcie_rate_idle(const ft_pcie_state* s, double* out) { NEED(s); *out = s->s.rate_idle(); return FT_OK; }
int ft_demand_slack(const ft_pcie_state* s, const char* func, double now, double* out) {
  NEED(s);
  const Demand* d = s->s.demands.find(sfunc(func));
  if (!d) {
    ft::set_last_error("unknown demand");
    return FT_E_KEY;
  }
  *out = d->slack(now);
  return FT_OK;
}
int ft_rate_demand(double bytes, double slo, double infer, double arrival, double now, double* least,
                   double* slack) {
  FT_TRY
  Demand d = make_demand("", bytes, slo, infer, arrival);
  if (least) *least = d.least;
  if (slack) *slack = d.slack(now);
  FT_CATCH
}
int ft_partition(ft_pcie_state* s, double now, double* rates, int32_t* at_risk, int cap, int* n) {
  NEED(s);
  FT_TRY
  auto r = partition(s->s, now);
  int rc = put_count((int)s->s.demands.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < s->s.demands.items.size(); ++i) {
    const auto& kv = s->s.demands.items[i];
    rates[i] = *r.find(kv.first);
    if (at_risk) at_risk[i] = kv.second.at_risk;
  }
  FT_CATCH
}
int ft_trigger_batches(double total, int64_t chunk, int bc, double* out, int cap, int* n) {
  FT_TRY
  auto b = trigger_batches(total, chunk, bc);
  int rc = put_count((int)b.size(), cap, n);
  if (rc) return rc;
  for (size_t i = 0; i < b.size(); ++i) out[i] = b[i];
  FT_CATCH
}
int ft_ring_create(double capacity, double cost, int prewarmed, ft_ring** out) {
  FT_TRY *out = new ft_ring{Ring{capacity, cost, prewarmed ? capacity : 0.0}}; FT_CATCH
}
void ft_ring_destroy(ft_ring* r) { delete r; }
int ft_ring_acquire(ft_ring* r, double need, double* ms) { NEED(r); FT_TRY *ms = r->r.acquire(need); FT_CATCH }
int ft_ring_state(const ft_ring* r, double* warm, double* cold) {
  NEED(r);
  if (warm) *warm = r->r.warm;
  if (cold) *cold = r->r.cold;
  return FT_OK;
}
int64_t ft_default_ring_capacity(int links, int64_t batch_bytes) { return 2 * batch_bytes * links; }

// ---------------------------------------------------------------- simcore
int ft_pipeline_latency(double size, const double* hops, int n, double chunk, double* out) {
  FT_TRY *out = pipeline_latency(size, std::vector<double>(hops, hops + n), chunk); FT_CATCH
}
int ft_pipeline_fill_ms(const double* hops, int n, double chunk, double* out) {
  FT_TRY *out = pipeline_fill_ms(std::vector<double>(hops, hops + n), chunk); FT_CATCH
}
int ft_nearest_rank(const double* v, int n, double pct, double* out) {
  FT_TRY *out = nearest_rank(std::vector<double>(v, v + n), pct); FT_CATCH
}

// ---------------------------------------------------------------- datastore
int ft_size_class(double b, int64_t* out) { FT_TRY *out = size_class(b); FT_CATCH }
int ft_p99(const double* s, int n, double* out) {
  FT_TRY
  if (n <= 0) fail(FT_E_VALUE, "empty sample");
  *out = p99(std::vector<double>(s, s + n));
  FT_CATCH
}
int ft_hist_create(const char* func, int window, ft_hist** out) {
  FT_TRY
  auto* h = new ft_hist{};
  h->h.func = sfunc(func);
  h->h.window = window > 0 ? (size_t)window : 1000;
  *out = h;
  FT_CATCH
}
void ft_hist_destroy(ft_hist* h) { delete h; }
int ft_hist_record(ft_hist* h, double now, double size, double con) { NEED(h); FT_TRY h->h.record(now, size, con); FT_CATCH }
int ft_hist_get(const ft_hist* h, double* rw, double* rs, double* rc, double* last) {
  NEED(h);
  if (rw) *rw = h->h.r_window;
  if (rs) *rs = h->h.r_size;
  if (rc) *rc = h->h.r_con;
  if (last) *last = h->h.has_last ? h->h.last : none();
  return FT_OK;
}
int ft_hist_reservation(const ft_hist* h, double* out) { NEED(h); *out = h->h.reservation(); return FT_OK; }
int ft_hist_window_active(const ft_hist* h, double now, int* out) { NEED(h); *out = h->h.active(now); return FT_OK; }
int ft_pool_target(const ft_hist* const* hs, int n, double now, double floor, double* out) {
  std::vector<const Hist*> v;
  for (int i = 0; i < n; ++i) v.push_back(&hs[i]->h);
  *out = pool_target(v, now, floor);
  return FT_OK;
}
int ft_pool_policy_create(int gpu, int mode, double floor, double alloc_ms, double physical, ft_pool_policy** out) {
  FT_TRY
  if (mode < 0 || mode > 2) fail(FT_E_VALUE, "unknown pool mode");
  auto* p = new ft_pool_policy{};
  p->p.gpu = gpu;
  p->p.mode = mode;
  p->p.floor = floor;
  p->p.alloc_ms = alloc_ms;
  p->p.physical = physical;
  *out = p;
  FT_CATCH
}
void ft_pool_policy_destroy(ft_pool_policy* p) { delete p; }
int ft_pool_policy_allocate(ft_pool_policy* p, double size, int64_t* id, int64_t* cls, double* cost) {
  NEED(p);
  FT_TRY
  double c = 0;
  auto b = p->p.allocate(size, &c);
  if (id) *id = b.id;
  if (cls) *cls = b.cls;
  if (cost) *cost = c;
  FT_CATCH
}
int ft_pool_policy_free(ft_pool_policy* p, int64_t id) { NEED(p); FT_TRY p->p.free_block(id); FT_CATCH }
int ft_pool_policy_record(ft_pool_policy* p, const char* func, double now, double size, double con) {
  NEED(p);
  FT_TRY p->p.hist(sfunc(func)).record(now, size, con); FT_CATCH
}
int ft_pool_policy_shrink(ft_pool_policy* p, double now, int64_t* dropped, int cap, int* n) {
  NEED(p);
  FT_TRY
  auto d = p->p.shrink(now);
  if (n) *n = (int)d.size();
  for (size_t i = 0; i < d.size() && (int)i < cap; ++i) dropped[i] = d[i];
  if ((int)d.size() > cap) {
    ft::set_last_error("dropped-id array too small (blocks were still dropped)");
    return FT_E_TRUNCATED;
  }
  FT_CATCH
}
// The request path's bookkeeping of one store in one call: the index entry
// (dataplane.py:72-83), the producer's histogram sample (datastore.py:51-62) and
// its reservation window for the shrink timer (engine.py:656-659).
int ft_store_commit(ft_index* x, ft_pool_policy* p, int64_t id, int node, int gpu, double size, double now,
                    const char* producer, int response, double concurrency, double* r_window, double* last) {
  NEED(x);
  NEED(p);
  FT_TRY
  x->x.store(id, node, gpu, size, now, sfunc(producer), response != 0);
  Hist& h = p->p.hist(sfunc(producer));
  h.record(now, size, concurrency);
  if (r_window) *r_window = h.r_window;
  if (last) *last = h.has_last ? h.last : none();
  FT_CATCH
}
// ... and of one retire: drop the index entry (dataplane.py:98-101), return the
// block to the policy when it is free (datastore.py:146-149; block_id < 0: still
// pinned by a view), and the producer's window.
int ft_retire_commit(ft_index* x, ft_pool_policy* p, int64_t id, int64_t block_id, const char* producer,
                     double* r_window, double* last) {
  NEED(x);
  NEED(p);
  FT_TRY
  x->x.drop(id);
  if (block_id >= 0) p->p.free_block(block_id);
  const Hist* h = p->p.hists.find(sfunc(producer));
  if (r_window) *r_window = h ? h->r_window : 0.0;
  if (last) *last = h && h->has_last ? h->last : none();
  FT_CATCH
}
// the same-GPU put in one call: wait the block's previous users, TMA copy of the
// producer's output into the block, record `ready`, then the store commit above
int ft_store_local(ft_index* x, ft_pool_policy* p, int64_t id, int node, int gpu, double size, double now,
                   const char* producer, int response, double concurrency, void* block_ptr, const void* src,
                   void* stream, uint32_t hints, void* const* waits, int nwaits, void* ready, double* r_window,
                   double* last) {
  NEED(x);
  NEED(p);
  int rc = ft_copy_ordered(block_ptr, src, (uint64_t)size, gpu, stream, hints, waits, nwaits, ready);
  if (rc != FT_OK) return rc;
  return ft_store_commit(x, p, id, node, gpu, size, now, producer, response, concurrency, r_window, last);
}
// the same-GPU get into the caller's input in one call: wait `waits` (the stored
// bytes), copy block -> dst, record `done`; the last consumer also retires
// (block_id < 0: a view still pins the block)
int ft_fetch_local(ft_index* x, ft_pool_policy* p, int64_t id, int64_t block_id, const char* producer, int retire,
                   void* dst, const void* block_ptr, uint64_t bytes, int device, void* stream, uint32_t hints,
                   void* const* waits, int nwaits, void* done, double* r_window, double* last) {
  NEED(x);
  NEED(p);
  int rc = ft_copy_ordered(dst, block_ptr, bytes, device, stream, hints, waits, nwaits, done);
  if (rc != FT_OK || !retire) return rc;
  return ft_retire_commit(x, p, id, block_id, producer, r_window, last);
}
// n retires in one call (batched fetch)
int ft_retire_many(ft_index* x, ft_pool_policy* p, int n, const int64_t* ids, const int64_t* block_ids,
                   const char* const* producers, double* r_windows, double* lasts) {
  NEED(x);
  NEED(p);
  for (int i = 0; i < n; ++i) {
    int rc = ft_retire_commit(x, p, ids[i], block_ids[i], producers[i], r_windows ? r_windows + i : nullptr,
                              lasts ? lasts + i : nullptr);
    if (rc != FT_OK) return rc;
  }
  return FT_OK;
}
int ft_pool_policy_target(ft_pool_policy* p, double now, double* out) { NEED(p); *out = p->p.target(now); return FT_OK; }
int ft_pool_policy_hist(const ft_pool_policy* p, const char* func, double* rw, double* last) {
  NEED(p);
  const Hist* h = p->p.hists.find(sfunc(func));
  if (rw) *rw = h ? h->r_window : 0.0;
  if (last) *last = h && h->has_last ? h->last : none();
  return FT_OK;
}
int ft_pool_policy_state_json(const ft_pool_policy* p, char* buf, size_t cap, size_t* need) {
  NEED(p);
  return emit_json(p->p.state_json(), buf, cap, need);
}
int ft_migration_plan(const ft_stored_object* objs, int n, double pressure, int policy, int32_t* actions,
                      int32_t* indices, int cap, int* nout) {
  FT_TRY
  auto pl = migration_plan(objs, n, pressure, policy);
  int rc = put_count((int)pl.size(), cap, nout);
  if (rc) return rc;
  for (size_t i = 0; i < pl.size(); ++i) {
    actions[i] = pl[i].first;
    indices[i] = pl[i].second;
  }
  FT_CATCH
}
int ft_prefetch_back(const ft_stored_object* objs, int n, double free_bytes, int32_t* indices, int cap, int* nout) {
  FT_TRY
  auto s = prefetch_back(objs, n, free_bytes);
  int rc = put_count((int)s.size(), cap, nout);
  if (rc) return rc;
  for (size_t i = 0; i < s.size(); ++i) indices[i] = s[i];
  FT_CATCH
}

// ---------------------------------------------------------------- strategies
int ft_strategy_preset(const char* name, ft_strategy* out) {
  NEED(name);
  std::string n(name);
  // strategies.py:33-55
  if (n == "infless_plus") *out = {1, 0, 1, 0, 0, 2, 2};
  else if (n == "deepplan_plus") *out = {1, 1, 1, 0, 0, 2, 2};
  else if (n == "faastube_star") *out = {0, 1, 1, 0, 0, 2, 2};
  else if (n == "faastube") *out = {0, 1, 1, 1, 1, 0, 0};
  else {
    ft::set_last_error("unknown strategy '" + n + "'");
    return FT_E_VALUE;
  }
  return FT_OK;
}

// ---------------------------------------------------------------- index
int ft_index_create(double sync, double lo, double gl, ft_index** out) {
  FT_TRY
  auto* x = new ft_index{};
  x->x.sync = sync;
  x->x.local_ms = lo;
  x->x.global_ms = gl;
  *out = x;
  FT_CATCH
}
void ft_index_destroy(ft_index* x) { delete x; }
int ft_index_unique_id(ft_index* x, int64_t* out) { NEED(x); *out = x->x.unique_id(); return FT_OK; }
int ft_index_store(ft_index* x, int64_t id, int node, int gpu, double size, double now, const char* producer, int resp,
                   double* vis) {
  NEED(x);
  FT_TRY
  double v = x->x.store(id, node, gpu, size, now, sfunc(producer), resp != 0);
  if (vis) *vis = v;
  FT_CATCH
}
int ft_index_resolve(ft_index* x, int64_t id, int node, double now, int* en, int* eg, double* cost, double* ready,
                     double* size) {
  NEED(x);
  FT_TRY
  double c, r;
  auto e = x->x.resolve(id, node, now, &c, &r);
  if (en) *en = e->node;
  if (eg) *eg = e->gpu;
  if (cost) *cost = c;
  if (ready) *ready = r;
  if (size) *size = e->size;
  FT_CATCH
}
int ft_index_drop(ft_index* x, int64_t id) { NEED(x); x->x.drop(id); return FT_OK; }
int ft_index_relocate(ft_index* x, int64_t id, int node, int gpu) { NEED(x); FT_TRY x->x.relocate(id, node, gpu); FT_CATCH }

// ---------------------------------------------------------------- plane
int ft_plane_create(const ft_topo* t, const ft_strategy* s, ft_matrix* m, double chunk, double map_ms,
                    ft_plane** out) {
  NEED(t);
  NEED(s);
  NEED(m);
  FT_TRY
  auto* p = new ft_plane{};
  p->p.topo = t->t.get();
  p->p.s = *s;
  p->p.m = &m->m;
  p->p.chunk = chunk;
  p->p.map_ms = map_ms;
  *out = p;
  FT_CATCH
}
void ft_plane_destroy(ft_plane* p) { delete p; }
int ft_fetch_plan(ft_plane* p, int sn, int sg, int dn, int dg, double size, ft_plan** out) {
  NEED(p);
  FT_TRY *out = new ft_plan{p->p.fetch_plan(sn, sg, dn, dg, size)}; FT_CATCH
}
void ft_plan_destroy(ft_plan* plan) { delete plan; }
int ft_plan_method(const ft_plan* plan, int* method, double* fixed, int* n_stages) {
  NEED(plan);
  if (method) *method = plan->p.method;
  if (fixed) *fixed = plan->p.fixed;
  if (n_stages) *n_stages = (int)plan->p.stages.size();
  return FT_OK;
}
int ft_plan_add_fixed_ms(ft_plan* plan, double ms) { NEED(plan); plan->p.fixed += ms; return FT_OK; }
int ft_plan_stage(const ft_plan* plan, int s, int* managed, double* pinned, int* nb) {
  NEED(plan);
  if (s < 0 || s >= (int)plan->p.stages.size()) {
    ft::set_last_error("stage index out of range");
    return FT_E_VALUE;
  }
  const Stage& st = plan->p.stages[s];
  if (managed) *managed = st.managed;
  if (pinned) *pinned = st.pinned;
  if (nb) *nb = (int)st.branches.size();
  return FT_OK;
}
int ft_plan_branch(const ft_plan* plan, int s, int b, ft_branch* out) {
  NEED(plan);
  NEED(out);
  if (s < 0 || s >= (int)plan->p.stages.size() || b < 0 || b >= (int)plan->p.stages[s].branches.size()) {
    ft::set_last_error("branch index out of range");
    return FT_E_VALUE;
  }
  const Branch& br = plan->p.stages[s].branches[b];
  memset(out, 0, sizeof *out);
  out->n_links = (int32_t)br.links.size();
  for (size_t i = 0; i < br.links.size() && i < FT_MAX_LINKS; ++i)
    out->links[i] = {br.links[i].kind, br.links[i].a, br.links[i].b};
  out->n_caps = (int32_t)br.hop_caps.size();
  for (size_t i = 0; i < br.hop_caps.size() && i < FT_MAX_LINKS; ++i) out->hop_caps[i] = br.hop_caps[i];
  out->bytes_share = br.share;
  out->cap_gbps = br.cap;
  out->reserved_gbps = br.reserved;
  out->fill_ms = br.fill;
  return FT_OK;
}
int ft_plan_pack(const ft_plan* plan, double* buf, size_t cap, size_t* need) {
  NEED(plan);
  std::vector<double> v;
  v.push_back((double)plan->p.stages.size());
  for (auto& st : plan->p.stages) {
    v.push_back(st.managed ? 1.0 : 0.0);
    v.push_back(st.pinned);
    v.push_back((double)st.branches.size());
    for (auto& br : st.branches) {
      v.push_back((double)br.links.size());
      for (auto& l : br.links) {
        v.push_back(l.kind);
        v.push_back(l.a);
        v.push_back(l.b);
      }
      v.push_back((double)br.hop_caps.size());
      for (double c : br.hop_caps) v.push_back(c);
      v.push_back(br.share);
      v.push_back(br.cap);
      v.push_back(br.reserved);
      v.push_back(br.fill);
    }
  }
  if (need) *need = v.size();
  if (v.size() > cap || !buf) {
    ft::set_last_error("ft_plan_pack: buffer too small");
    return FT_E_TRUNCATED;
  }
  std::memcpy(buf, v.data(), v.size() * sizeof(double));
  return FT_OK;
}
int ft_plan_json(const ft_plan* plan, char* buf, size_t cap, size_t* need) {
  NEED(plan);
  return emit_json(plan->p.json(), buf, cap, need);
}
int ft_plan_latency(const ft_plan* plan, double* out) { NEED(plan); *out = plan->p.latency(); return FT_OK; }
int ft_release_claim(ft_plane* p, const ft_plan* plan) { NEED(p); NEED(plan); FT_TRY p->p.release_claim(plan->p); FT_CATCH }

// ---------------------------------------------------------------- arbiter
int ft_arbiter_create(double bw, int bc, int64_t chunk, ft_arbiter** out) {
  FT_TRY
  auto* a = new ft_arbiter{};
  a->a.share = PcieState{bw, bc, chunk, {}};
  a->a.batch_bytes = (double)(chunk * bc);
  *out = a;
  FT_CATCH
}
void ft_arbiter_destroy(ft_arbiter* a) { delete a; }
int ft_arbiter_start(ft_arbiter* a, double now, const char* key, double total, double slo, double infer,
                     double arrival, double pbc, int nb) {
  NEED(a);
  FT_TRY
  if (nb <= 0) fail(FT_E_VALUE, "a stage needs at least one branch");
  a->a.start(now, sfunc(key), total, slo, infer, arrival, pbc, nb);
  FT_CATCH
}
int ft_arbiter_boundary(ft_arbiter* a, double now, const char* key) { NEED(a); FT_TRY a->a.boundary(now, sfunc(key)); FT_CATCH }
int ft_arbiter_finish(ft_arbiter* a, double now, const char* key) { NEED(a); FT_TRY a->a.finish(now, sfunc(key)); FT_CATCH }
int ft_arbiter_decisions_json(const ft_arbiter* a, char* buf, size_t cap, size_t* need) {
  NEED(a);
  return emit_json(a->a.last_json.empty() ? "[]" : a->a.last_json, buf, cap, need);
}
int ft_arbiter_state_json(const ft_arbiter* a, char* buf, size_t cap, size_t* need) {
  NEED(a);
  return emit_json(a->a.state_json(), buf, cap, need);
}
int ft_arbiter_stage(const ft_arbiter* a, const char* key, double* rate, int* started, double* pending,
                     double* armed) {
  NEED(a);
  const auto* m = a->a.stages.find(sfunc(key));
  if (!m) {
    ft::set_last_error("unknown stage");
    return FT_E_KEY;
  }
  if (rate) *rate = m->rate;
  if (started) *started = m->started;
  if (pending) *pending = m->pending;
  if (armed) *armed = m->armed;
  return FT_OK;
}
int ft_arbiter_next_event(const ft_arbiter* a, double* t, char* key, size_t key_cap) {
  NEED(a);
  double best = none();
  const std::string* bk = nullptr;
  for (auto& kv : a->a.stages.items)
    if (!is_none(kv.second.armed) && (is_none(best) || kv.second.armed < best)) {
      best = kv.second.armed;
      bk = &kv.first;
    }
  *t = best;
  if (key && key_cap) {
    std::string k = bk ? *bk : "";
    snprintf(key, key_cap, "%s", k.c_str());
  }
  return FT_OK;
}

}  // extern "C"

// ---------------------------------------------- host->GPU fetch, one call
extern "C" {

int ft_plane_set_pairs(ft_plane* p, int gpu, int n, void* const* ce, void* const* fw) {
  NEED(p);
  if (n <= 0 || !ce || !fw) {
    ft::set_last_error("ft_plane_set_pairs: bad arguments");
    return FT_E_VALUE;
  }
  auto& v = p->pairs[gpu];
  v.clear();
  for (int i = 0; i < n; ++i) v.emplace_back(ce[i], fw[i]);
  return FT_OK;
}

// tube._host_to_gpu's plan -> routes step in one call: plan a host->GPU transfer
// (dataplane.py:190-250), cut the object into each branch's contiguous byte range
// (tube._stripes: shares accumulate in float64, boundaries floored to 256 B), pick
// each route's stream pair on the GPU whose PCIe root carries it (slot keyed by the
// consumer stream, as tube._pair), and return what ft_pacer_submit takes.
int ft_h2g_routes(ft_plane* p, int node, int dst_gpu, uint64_t bytes, void* consumer_stream, ft_route* routes,
                  int cap, int* k, int* managed, double* per_branch_cap, uint64_t* nvlink_bytes) {
  NEED(p);
  NEED(routes);
  NEED(k);
  FT_TRY
  Plan plan = p->p.fetch_plan(node, -1, node, dst_gpu, (double)bytes);
  if (plan.method != FT_HOST_GPU || plan.stages.size() != 1) throw Error(FT_E_VALUE, "not a host->GPU plan");
  const Stage& st = plan.stages[0];
  const int nb = (int)st.branches.size();
  if (nb > cap) throw Error(FT_E_TRUNCATED, "ft_h2g_routes: more branches than route slots");
  // byte ranges (tube._stripes)
  const double total = py_sum(st.branches.begin(), st.branches.end(), [](const Branch& b) { return b.share; });
  std::vector<uint64_t> bounds{0};
  if (total <= 0 || bytes == 0) {
    for (int i = 0; i < nb; ++i) bounds.push_back(bytes);
  } else {
    double acc = 0.0;
    for (int i = 0; i + 1 < nb; ++i) {
      acc += st.branches[i].share;
      const uint64_t b = (uint64_t)std::floor((double)bytes * (acc / total)) / 256 * 256;
      bounds.push_back(std::max(bounds.back(), std::min(bytes, b)));
    }
    bounds.push_back(bytes);
  }
  const uint64_t sp = (uint64_t)(uintptr_t)consumer_stream;
  const unsigned __int128 slot = ((unsigned __int128)(sp >> 4) * 0x9E3779B1ull) >> 16;
  double capmin = INFINITY;
  uint64_t nv = 0;
  for (int i = 0; i < nb; ++i) {
    const Branch& b = st.branches[i];
    int sg = dst_gpu;  // tube._staging_gpu: the first GPU the branch lands on
    for (auto& l : b.links)
      if (l.kind == FT_LINK_NVP_OUT || l.kind == FT_LINK_NV) {
        sg = l.a;
        break;
      }
    auto it = p->pairs.find(sg);
    if (it == p->pairs.end() || it->second.empty())
      throw Error(FT_E_NOT_SUPPORTED, "the plan routes through GPU " + std::to_string(sg) +
                                          ", which this tube does not drive");
    const auto& pr = it->second[(size_t)(slot % it->second.size())];
    const uint64_t off = bounds[i], len = bounds[i + 1] - bounds[i];
    routes[i] = ft_route{sg, 0, off, len, pr.first, pr.second};
    if (sg != dst_gpu) nv += len;
    for (double c : b.hop_caps) capmin = std::min(capmin, c);
  }
  *k = nb;
  if (managed) *managed = p->p.s.pcie_sched && st.managed;
  if (per_branch_cap) *per_branch_cap = capmin;
  if (nvlink_bytes) *nvlink_bytes = nv;
  FT_CATCH
}

}  // extern "C"
