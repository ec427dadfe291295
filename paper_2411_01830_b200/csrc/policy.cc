// PCIe rate policy, latency model and elastic-store policy.
// Restates tubesim pcie_sched.py:23-162, simcore.py:21-50,247-252 and
// datastore.py:24-238 with CPython float semantics.
#include <algorithm>
#include <numeric>

#include "decisions.h"

namespace ft {

// ------------------------------------------------------------ pcie_sched
double min_rate(double bytes, double slo, double infer) {  // pcie_sched.py:23-33
  if (bytes < 0) fail(FT_E_VALUE, "data size must be >= 0");
  if (bytes == 0) return 0.0;
  double w = slo - infer;
  if (w <= 0) fail(FT_E_INFEASIBLE, "slo <= inference with bytes pending");
  return bytes / (w * 1e6);
}
Demand make_demand(const std::string& f, double bytes, double slo, double infer, double arrival) {
  Demand d{f, bytes, slo, infer, arrival, min_rate(bytes, slo, infer)};
  return d;
}
double Demand::slack(double now) const {  // pcie_sched.py:49-55
  double deadline = arrival + slo - infer;
  if (least <= 0) return deadline - now;
  return (deadline - now) - bytes / (least * 1e6);
}
double PcieState::rate_idle() const {  // pcie_sched.py:69-71
  PySum s;
  for (auto& kv : demands.items) s.add(kv.second.least);
  return std::max(0.0, bw_all - s.value());
}
ODict<double> partition(PcieState& st, double now) {  // pcie_sched.py:80-104
  ODict<double> rates;
  if (st.demands.empty()) return rates;
  PySum s;
  for (auto& kv : st.demands.items) s.add(kv.second.least);
  double total = s.value();
  if (total > st.bw_all) {
    double scale = st.bw_all / total;
    for (auto& kv : st.demands.items) {
      kv.second.at_risk = true;
      rates.set(kv.first, kv.second.least * scale);
    }
    return rates;
  }
  for (auto& kv : st.demands.items) {
    kv.second.at_risk = false;
    rates.set(kv.first, kv.second.least);
  }
  double idle = st.bw_all - total;
  if (idle > 0) {
    const Demand* t = nullptr;
    double ts = 0;
    for (auto& kv : st.demands.items) {
      const Demand& d = kv.second;
      double sl = d.slack(now);
      bool better = !t || sl < ts || (sl == ts && (d.arrival < t->arrival || (d.arrival == t->arrival && d.func < t->func)));
      if (better) {
        t = &d;
        ts = sl;
      }
    }
    *rates.find(t->func) += idle;
  }
  return rates;
}
std::vector<double> trigger_batches(double total, int64_t chunk, int batch_chunks) {  // :107-119
  std::vector<double> out;
  if (total <= 0) return out;
  int64_t chunks = std::max<int64_t>(1, py_ceil(total / (double)chunk));
  double bb = (double)(batch_chunks * chunk);
  int64_t nb = py_ceil((double)chunks / (double)batch_chunks);
  double rem = total;
  for (int64_t i = 0; i < nb; ++i) {
    double size = bb < rem ? bb : rem;  // min(remaining, batch): first wins ties
    out.push_back(size);
    rem -= size;
  }
  return out;
}
double Ring::acquire(double need) {  // pcie_sched.py:138-150
  if (need < 0) fail(FT_E_VALUE, "bytes must be >= 0");
  double usable = std::min(need, capacity);
  double shortfall = std::max(0.0, usable - warm) + std::max(0.0, need - capacity);
  if (usable > warm) warm = usable;
  if (shortfall > 0) {
    cold += shortfall;
    return cost * shortfall / 1e6;
  }
  return 0.0;
}

// ------------------------------------------------------------ simcore
double ms_for(double bytes, double gbps) { return bytes / (gbps * 1e6); }
static size_t slowest(const std::vector<double>& h) {
  size_t s = 0;
  for (size_t i = 1; i < h.size(); ++i)
    if (h[i] < h[s]) s = i;
  return s;
}
double pipeline_latency(double size, const std::vector<double>& hops, double chunk) {  // simcore.py:25-42
  if (hops.empty()) fail(FT_E_VALUE, "pipeline_latency needs at least one hop");
  for (double b : hops)
    if (b <= 0) fail(FT_E_VALUE, "hop bandwidths must be > 0");
  if (chunk <= 0 || chunk > size) chunk = size;
  size_t s = slowest(hops);
  double total = ms_for(size, hops[s]);
  for (size_t i = 0; i < hops.size(); ++i)
    if (i != s) total += ms_for(chunk, hops[i]);
  return total;
}
double pipeline_fill_ms(const std::vector<double>& hops, double chunk) {  // simcore.py:45-50
  if (hops.size() <= 1) return 0.0;
  size_t s = slowest(hops);
  PySum sum;
  for (size_t i = 0; i < hops.size(); ++i)
    if (i != s) sum.add(ms_for(chunk, hops[i]));
  return sum.value();
}
double nearest_rank(const std::vector<double>& v, double pct) {  // simcore.py:247-252
  if (v.empty()) fail(FT_E_VALUE, "empty sample");
  int64_t rank = std::max<int64_t>(1, py_ceil(pct / 100.0 * (double)v.size()));
  return v[rank - 1];
}

// ------------------------------------------------------------ datastore
int64_t size_class(double bytes) {  // datastore.py:24-29
  const int64_t CLS = 2000000;
  if (bytes <= 0) fail(FT_E_VALUE, "allocation size must be > 0");
  return CLS * std::max<int64_t>(1, py_ceil(bytes / (double)CLS));
}
double p99(std::vector<double> xs) {  // datastore.py:32-35
  std::stable_sort(xs.begin(), xs.end());
  int64_t rank = std::max<int64_t>(1, py_ceil(0.99 * (double)xs.size()));
  return xs[rank - 1];
}
namespace {
// nearest-rank p99 (datastore.py:32-35) of an already sorted window
double p99_sorted(const std::vector<double>& v) {
  int64_t rank = std::max<int64_t>(1, py_ceil(0.99 * (double)v.size()));
  return v[rank - 1];
}
}  // namespace
void Hist::record(double now, double size, double con) {  // datastore.py:51-62
  if (size < 0 || con < 0) fail(FT_E_VALUE, "histogram samples must be >= 0");
  auto push = [this](std::deque<double>& q, std::vector<double>& s, double x) {
    q.push_back(x);
    s.insert(std::upper_bound(s.begin(), s.end(), x), x);  // after its equals: arrival order
    if (q.size() > window) {
      double old = q.front();  // the oldest sample: first of its equal range
      q.pop_front();
      s.erase(std::lower_bound(s.begin(), s.end(), old));
    }
  };
  if (has_last) push(gaps, gaps_s, now - last);
  last = now;
  has_last = true;
  push(sizes, sizes_s, size);
  push(conc, conc_s, con);
  if (!gaps_s.empty()) r_window = p99_sorted(gaps_s);
  r_size = p99_sorted(sizes_s);
  r_con = p99_sorted(conc_s);
}
double Hist::reservation() const {  // datastore.py:64-67
  if (sizes.empty()) return 0.0;
  return r_size * std::max(1.0, r_con);
}
bool Hist::active(double now) const {  // datastore.py:69-72
  if (!has_last) return false;
  return now - last <= std::max(r_window, 0.0);
}
double pool_target(const std::vector<const Hist*>& hs, double now, double floor) {  // :79-82
  PySum s;
  for (auto* h : hs)
    if (h->active(now)) s.add(h->reservation());
  return std::max(s.value(), floor);
}
double PoolPolicy::pool_bytes() const {
  int64_t s = 0;
  for (auto& b : blocks) s += b.cls;
  return (double)s;
}
double PoolPolicy::in_use_bytes() const {
  int64_t s = 0;
  for (auto& b : blocks)
    if (b.in_use) s += b.cls;
  return (double)s;
}
Hist& PoolPolicy::hist(const std::string& f) {
  if (auto* h = hists.find(f)) return *h;
  Hist h;
  h.func = f;
  h.window = 1000;
  return hists.set(f, h);
}
double PoolPolicy::target(double now) const {
  std::vector<const Hist*> hs;
  for (auto& kv : hists.items) hs.push_back(&kv.second);
  return pool_target(hs, now, floor);
}
PoolPolicy::Block PoolPolicy::allocate(double size, double* cost) {  // datastore.py:130-144
  int64_t cls = size_class(size);
  bool cached = false;
  for (auto& b : blocks) cached = cached || (b.cls == cls && !b.in_use);
  if (pool_bytes() + (double)cls > physical && !cached)
    fail(FT_E_OOM, "gpu " + std::to_string(gpu) + ": pool would exceed physical memory");
  if (mode != 2) {
    for (auto& b : blocks)
      if (!b.in_use && b.cls == cls) {
        b.in_use = true;
        *cost = 0.0;
        return b;
      }
  }
  Block b{cls, true, next_id++};
  blocks.push_back(b);
  *cost = alloc_ms;
  return b;
}
void PoolPolicy::free_block(int64_t id) {  // datastore.py:146-149
  for (size_t i = 0; i < blocks.size(); ++i)
    if (blocks[i].id == id) {
      blocks[i].in_use = false;
      if (mode == 2) blocks.erase(blocks.begin() + i);
      return;
    }
  fail(FT_E_KEY, "unknown pool block " + std::to_string(id));
}
std::vector<int64_t> PoolPolicy::shrink(double now) {  // datastore.py:151-166
  std::vector<int64_t> dropped;
  if (mode != 0) return dropped;
  double limit = target(now);
  bool any = false;
  for (auto& kv : hists.items) any = any || kv.second.active(now);
  if (!any) limit = std::min(limit, floor);
  std::vector<Block> idle;
  for (auto& b : blocks)
    if (!b.in_use) idle.push_back(b);
  std::stable_sort(idle.begin(), idle.end(), [](const Block& a, const Block& b) { return -a.cls < -b.cls; });
  for (auto& b : idle) {
    if (pool_bytes() - (double)b.cls < std::min(limit, floor)) break;
    if (pool_bytes() <= limit) break;
    for (size_t i = 0; i < blocks.size(); ++i)
      if (blocks[i].id == b.id) {
        blocks.erase(blocks.begin() + i);
        break;
      }
    dropped.push_back(b.id);
  }
  return dropped;
}
std::string PoolPolicy::state_json() const {
  JsonOut o;
  o.raw("{\"blocks\":[");
  for (size_t i = 0; i < blocks.size(); ++i) {
    if (i) o.raw(",");
    o.raw("[");
    o.inum(blocks[i].cls);
    o.raw(blocks[i].in_use ? ",true," : ",false,");
    o.inum(blocks[i].id);
    o.raw("]");
  }
  o.raw("],\"pool_bytes\":");
  o.num(pool_bytes());
  o.raw(",\"in_use_bytes\":");
  o.num(in_use_bytes());
  o.raw("}");
  return o.s;
}

static int nearest_pos(const ft_stored_object& o) {
  int m = o.consumer_pos[0];
  for (int i = 1; i < o.n_consumers; ++i) m = std::min(m, (int)o.consumer_pos[i]);
  return m;
}

std::vector<std::pair<int, int>> migration_plan(const ft_stored_object* objs, int n, double pressure,
                                                int policy) {  // datastore.py:192-222
  if (pressure <= 0) fail(FT_E_VALUE, "pressure must be > 0");
  if (policy != 0 && policy != 1) fail(FT_E_VALUE, "unknown migration policy");
  std::vector<std::pair<int, int>> plan;
  double freed = 0.0;
  std::vector<int> on_gpu;
  for (int i = 0; i < n; ++i)
    if (objs[i].location == 0) on_gpu.push_back(i);
  std::vector<int> dead;
  for (int i : on_gpu)
    if (!objs[i].live) dead.push_back(i);
  std::stable_sort(dead.begin(), dead.end(), [&](int a, int b) { return objs[a].data_id < objs[b].data_id; });
  for (int i : dead) {
    plan.push_back({0, i});
    freed += objs[i].size_bytes;
    if (freed >= pressure) return plan;
  }
  std::vector<int> cand;
  for (int i : on_gpu)
    if (objs[i].live && objs[i].n_consumers > 0) cand.push_back(i);
  if (policy == 0) {
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
      int ka = -nearest_pos(objs[a]), kb = -nearest_pos(objs[b]);
      if (ka != kb) return ka < kb;
      return objs[a].data_id < objs[b].data_id;
    });
  } else {
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
      if (objs[a].stored_at_ms != objs[b].stored_at_ms) return objs[a].stored_at_ms < objs[b].stored_at_ms;
      return objs[a].data_id < objs[b].data_id;
    });
  }
  for (int i : cand) {
    plan.push_back({1, i});
    freed += objs[i].size_bytes;
    if (freed >= pressure) return plan;
  }
  fail(FT_E_HARD_PRESSURE, "pressure cannot be relieved by reclaim/migration");
}

std::vector<int> prefetch_back(const ft_stored_object* objs, int n, double free_bytes) {  // :225-238
  if (free_bytes <= 0) fail(FT_E_VALUE, "free_bytes must be > 0");
  std::vector<int> mig;
  for (int i = 0; i < n; ++i)
    if (objs[i].location == 1 && objs[i].live && objs[i].n_consumers > 0) mig.push_back(i);
  std::stable_sort(mig.begin(), mig.end(), [&](int a, int b) {
    int ka = nearest_pos(objs[a]), kb = nearest_pos(objs[b]);
    if (ka != kb) return ka < kb;
    return objs[a].data_id < objs[b].data_id;
  });
  std::vector<int> out;
  double room = free_bytes;
  for (int i : mig)
    if (objs[i].size_bytes <= room) {
      out.push_back(i);
      room -= objs[i].size_bytes;
    }
  return out;
}

}  // namespace ft
