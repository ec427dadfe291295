// Decision side of the data-passing layer: the reference's control-plane
// policies restated in C++ with bit-identical float64 arithmetic. Each class
// cites the tubesim module it replaces (paths under pkg/src/tubesim/).
#pragma once

#include <deque>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "common.h"

namespace ft {

using Path = std::vector<int>;

// ------------------------------------------------------------ topology.py
struct Topo {
  std::string name;
  int gpu_count = 0;
  struct Node { int64_t id; std::vector<int64_t> gpus; };
  std::vector<Node> nodes;
  struct Link { std::string kind; JVal a, b; double bw; int mult; };
  std::vector<Link> links;
  std::vector<std::pair<int, std::vector<int64_t>>> groups;  // pcie_groups, insertion order
  double pcie = 12.0, pageable = 3.0, peer = 7.9, net = 10.0;
  // _nv / _nv_kind keyed (min, max) in first-seen order
  std::vector<std::pair<std::pair<int, int>, double>> nv;
  std::map<std::pair<int, int>, size_t> nv_pos;
  std::map<std::pair<int, int>, std::string> nv_kind;
  std::map<int64_t, int64_t> gpu_node, gpu_root;

  static std::unique_ptr<Topo> from_json(const std::string& doc);  // topology.py:327-355
  std::vector<std::string> validate() const;                       // topology.py:160-185
  void check(int g) const;                                         // topology.py:154-156
  int node_of(int g) const;
  int root_of(int g) const;
  double nvlink_gbps(int u, int v) const;
  std::vector<int> neighbors(int g) const;
  int kind(int u, int v) const;  // 0 none 1 nvlink 2 nvswitch
  double switch_port_gbps(int g) const;
  double degree_gbps(int g) const;
  double pair_bandwidth(int u, int v) const;
  std::vector<int> sorted_roots() const;
  const std::vector<int64_t>& group(int root) const;
  // candidate_paths results per (src, dst, max_hops): the topology is immutable,
  // and the enumeration (157 paths on an 8-GPU mesh) dominated every select
  struct CandCache;
  std::shared_ptr<CandCache> cand_cache;
};

// --------------------------------------------------- BandwidthMatrix
struct Matrix {
  const Topo* topo;
  std::map<std::pair<int, int>, double> capacity, residual;
  // dense mirrors of capacity/residual (NaN = no edge): res()/idle() are called
  // for every hop of every candidate on each select
  int n = 0;
  std::vector<double> dcap, dres;
  std::map<int, double> egress, ingress;
  std::map<std::pair<int, int>, std::vector<std::string>> owners;
  ODict<std::vector<std::pair<Path, double>>> held;

  explicit Matrix(const Topo* t);
  double res(int u, int v) const;
  bool idle(int u, int v) const;
  void hold(const std::string& f, const Path& p, double rate);
  void release(const std::string& f);
  void release_path(const std::string& f, const Path& p);
  std::vector<std::string> holders(int u, int v) const;
  double aggregate(const std::string& f) const;
  std::string state_json() const;

 private:
  void give_back(const std::string& f, const Path& p, double rate);
};

// ------------------------------------------------------- nvlink_sched.py
struct NvPath { Path gpus; double b_min; bool held; };
struct SelectTrace {
  int candidates = 0;
  std::vector<std::pair<Path, double>> phase1, phase2;
  bool fallback = false;
  Path shared;
  std::string json() const;
};
const std::vector<Path>& candidate_paths(const Topo& t, int s, int d, int max_hops = 4);
std::vector<NvPath> select_paths(Matrix& m, const std::string& func, int s, int d, bool allow_busy,
                                 SelectTrace* tr);
std::string claim_direct(Matrix& m, const std::vector<std::pair<int, int>>& pairs, const std::string& wf);
std::vector<int64_t> distribute_chunks(int64_t n, const std::vector<double>& w);

// --------------------------------------------------------- pcie_sched.py
double min_rate(double bytes, double slo, double infer);
struct Demand {
  std::string func;
  double bytes, slo, infer, arrival, least;
  bool at_risk = false;
  double slack(double now) const;
};
Demand make_demand(const std::string& f, double bytes, double slo, double infer, double arrival);
struct PcieState {
  double bw_all;
  int batch_chunks;
  int64_t chunk;
  ODict<Demand> demands;
  double batch_bytes() const { return (double)(batch_chunks * chunk); }
  double rate_idle() const;
};
ODict<double> partition(PcieState& st, double now);
std::vector<double> trigger_batches(double total, int64_t chunk, int batch_chunks);
struct Ring {
  double capacity, cost, warm, cold = 0.0;
  double acquire(double need);
};

// ------------------------------------------------------------ simcore.py
double ms_for(double bytes, double gbps);
double pipeline_latency(double size, const std::vector<double>& hops, double chunk);
double pipeline_fill_ms(const std::vector<double>& hops, double chunk);
double nearest_rank(const std::vector<double>& sorted, double pct);

// ---------------------------------------------------------- datastore.py
int64_t size_class(double bytes);
double p99(std::vector<double> xs);
struct Hist {
  std::string func;
  size_t window;
  std::deque<double> gaps, sizes, conc;  // arrival order (window eviction)
  // the same windows kept sorted, equal values in arrival order == sorted() of
  // the deque (Python's sort is stable): p99 is one index, not a sort per record
  std::vector<double> gaps_s, sizes_s, conc_s;
  bool has_last = false;
  double last = 0.0, r_window = 0.0, r_size = 0.0, r_con = 0.0;
  void record(double now, double size, double con);
  double reservation() const;
  bool active(double now) const;
};
double pool_target(const std::vector<const Hist*>& hs, double now, double floor);
struct PoolPolicy {
  int gpu, mode;  // 0 autoscale 1 cache_all 2 none
  double floor, alloc_ms, physical;
  struct Block { int64_t cls; bool in_use; int64_t id; };
  std::vector<Block> blocks;
  ODict<Hist> hists;
  int64_t next_id = 1;
  double pool_bytes() const;
  double in_use_bytes() const;
  double target(double now) const;
  Hist& hist(const std::string& f);
  Block allocate(double size, double* cost);
  void free_block(int64_t id);
  std::vector<int64_t> shrink(double now);
  std::string state_json() const;
};
std::vector<std::pair<int, int>> migration_plan(const ft_stored_object* o, int n, double pressure, int policy);
std::vector<int> prefetch_back(const ft_stored_object* o, int n, double free_bytes);

// ---------------------------------------------------------- dataplane.py
struct Index {
  double sync, local_ms, global_ms;
  int64_t counter = 1;
  struct Entry { int64_t id; double size; int node, gpu; double created; std::string producer; bool response; double visible; };
  std::map<int, std::map<int64_t, std::shared_ptr<Entry>>> local;
  std::map<int64_t, std::shared_ptr<Entry>> table;
  // the daemon's native lane (lane.cc) stores, drops and mints ids from its worker
  // threads while the tube calls in from Python: every method takes the lock
  std::mutex mu;
  int64_t unique_id() {
    std::lock_guard<std::mutex> lk(mu);
    return counter++;
  }
  double store(int64_t id, int node, int gpu, double size, double now, const std::string& producer, bool resp);
  std::shared_ptr<Entry> resolve(int64_t id, int node, double now, double* cost, double* ready);
  void drop(int64_t id);
  void relocate(int64_t id, int node, int gpu);
};

struct LinkId { int kind, a, b; };
struct Branch {
  std::vector<LinkId> links;
  double share;
  double cap = none(), reserved = none(), fill = 0.0;
  std::vector<double> hop_caps;
};
struct Stage { std::vector<Branch> branches; bool managed = false; double pinned = 0.0; };
struct Plan {
  int method;  // ft_method
  double size, fixed = 0.0;
  std::vector<Stage> stages;
  std::string claimed;  // empty = None
  std::string note;
  double latency() const;
  std::string json() const;
};
struct Plane {
  const Topo* topo;
  ft_strategy s;
  Matrix* m;
  double chunk, map_ms;
  int64_t claims = 1;
  Plan fetch_plan(int sn, int sg, int dn, int dg, double size);
  void release_claim(const Plan& p);

 private:
  Plan host_gpu(int sn, int sg, int dn, int dg, double size);
  std::vector<Branch> pcie_branches(int node, int gpu, double size, bool into);
  bool staging_route(int node, int root, int gpu, bool into, std::vector<LinkId>* out);
  bool nv_route(int a, int b, bool into, Path* out);
  double link_cap(const LinkId& l) const;
  Plan inter_gpu(int sn, int sg, int dn, int dg, double size);
  Plan pcie_peer(int sn, int sg, int dn, int dg, double size);
  Plan inter_node(int sn, int sg, int dn, int dg, double size);
};

// ------------------------------------------------- engine.py managed stages
struct Arbiter {
  PcieState share;
  double batch_bytes;
  struct StageSt {
    std::string key;
    Demand demand;
    int n_flows;
    double cap, rate = 0.0, pending = none(), anchor = 0.0, armed = none();
    bool started = false;
    double next_boundary(double after, double batch_bytes) const;
  };
  ODict<StageSt> stages;
  int risk_flags = 0;
  std::string last_json;  // decisions of the last call
  bool quiet = false;     // no decision record (the live pacer when it does not log)
  void start(double now, const std::string& key, double total, double slo, double infer, double arrival,
             double per_branch_cap, int n_branches);
  void boundary(double now, const std::string& key);
  void finish(double now, const std::string& key);
  // live only (no reference counterpart): the link capacity the partition hands out
  // changed (measured by the pacer); re-partition at `now` as any other event does
  // (each stage's cap is raised to at least link_gbps per flow: caps come from the
  // same planned link rate the measurement replaces)
  void set_bw(double now, double bw_all, double link_gbps);
  std::string state_json() const;

 private:
  JsonOut out_;
  bool first_ = true;
  void begin();
  void end();
  void emit(const std::string& item);
  void resync(double now);
  void set_rate(double now, StageSt& m, double rate);
  void arm(double now, StageSt& m, double t);
};

}  // namespace ft
