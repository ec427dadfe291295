/*
 * faastube.h — C ABI of the B200-native FaaSTube data-passing layer
 * (libfaastube.so, built from paper_2411_01830_b200/csrc).
 *
 * The reference (arxiv 2411.01830, /root/reference) ships a Python simulator
 * (`tubesim`); its data-passing surface is Python classes, not an FFI. Each
 * entry point below replaces the reference function cited beside it
 * (paths relative to pkg/src/tubesim/), with the same argument meaning and
 * error behaviour (Python exceptions become FT_E_* status codes, message in
 * ft_last_error()). INTEGRATION.md shows the ctypes binding a maintainer of
 * the reference would add.
 *
 * Conventions: every function returns an int status (FT_OK = 0) unless noted;
 * outputs go through pointers. GB/s = 1e9 B/s, sizes in bytes (double where
 * the reference uses float byte counts), times in ms. "None" in the reference
 * is NaN for doubles and -1 for GPU ids (host location). Arrays sized by the
 * caller: `cap` is the capacity, `*n` the count written (FT_E_TRUNCATED when
 * cap is too small; *n then holds the required count). JSON outputs use
 * ("buf", "cap", "need") with need including the NUL.
 * Decision objects are NOT thread-safe (the reference is single-threaded,
 * SPEC.md:232-233); the device movers are stream-ordered and thread-safe.
 */
#ifndef FAASTUBE_H
#define FAASTUBE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum ft_status {
  FT_OK = 0,
  FT_E_TOPOLOGY = 1,      /* topology.TopologyError            topology.py:40  */
  FT_E_INFEASIBLE = 2,    /* pcie_sched.InfeasibleDemand       pcie_sched.py:19 */
  FT_E_MISSING = 3,       /* dataplane.MissingData             dataplane.py:26 */
  FT_E_DUPLICATE = 4,     /* dataplane.DuplicateStore          dataplane.py:30 */
  FT_E_HARD_PRESSURE = 5, /* datastore.HardPressure            datastore.py:188 */
  FT_E_OOM = 6,           /* MemoryError from MemoryPool       datastore.py:134-136 */
  FT_E_CUDA = 7,          /* CUDA driver/runtime failure (device movers, pool) */
  FT_E_VALUE = 8,         /* ValueError (bad argument)         e.g. datastore.py:27 */
  FT_E_TRUNCATED = 9,     /* caller buffer too small */
  FT_E_KEY = 10,          /* KeyError (unknown id / func) */
  FT_E_NOT_SUPPORTED = 11, /* feature unavailable on this device/driver */
  FT_E_TIMEOUT = 12,       /* a host wait ran out of time */
  FT_E_CLOSED = 13         /* the peer closed the function<->daemon channel */
};

#define FT_MAX_PATH 8   /* GPUs per NVLink path (MAX_HOPS 4 => 5)  nvlink_sched.py:17 */
#define FT_MAX_LINKS 8  /* link ids per branch                      dataplane.py:136-143 */

const char* ft_last_error(void); /* thread-local message of the last failure */
const char* ft_version(void);

/* ------------------------------------------------- topology (topology.py) */
typedef struct ft_topo ft_topo;
/* from_dict(doc)                                          topology.py:327-355 */
int ft_topo_create(const char* json_doc, ft_topo** out);
void ft_topo_destroy(ft_topo* t);
int ft_topo_gpu_count(const ft_topo* t, int* out);
/* Topology.node_of / pcie_root_of                         topology.py:102-108 */
int ft_topo_node_of(const ft_topo* t, int gpu, int* out);
int ft_topo_root_of(const ft_topo* t, int gpu, int* out);
/* Topology.nvlink_gbps                                    topology.py:110-114 */
int ft_topo_nvlink_gbps(const ft_topo* t, int u, int v, double* out);
/* Topology.nvlink_neighbors                               topology.py:116-119 */
int ft_topo_neighbors(const ft_topo* t, int gpu, int32_t* out, int cap, int* n);
/* Topology.pair_kind: 0 none, 1 nvlink, 2 nvswitch        topology.py:124-125 */
int ft_topo_pair_kind(const ft_topo* t, int u, int v, int* out);
/* Topology.switch_port_gbps / nvlink_degree_gbps          topology.py:127-140 */
int ft_topo_switch_port_gbps(const ft_topo* t, int gpu, double* out);
int ft_topo_degree_gbps(const ft_topo* t, int gpu, double* out);
/* Topology.pair_bandwidth                                 topology.py:142-152 */
int ft_topo_pair_bandwidth(const ft_topo* t, int u, int v, double* out);
/* rates: 0 pcie_gbps, 1 pcie_pageable_gbps, 2 pcie_peer_gbps, 3 network_gbps */
int ft_topo_rate(const ft_topo* t, int which, double* out);
/* number of PCIe root groups and their members (sorted root order) */
int ft_topo_roots(const ft_topo* t, int32_t* roots, int cap, int* n);

/* ------------------------------------ bandwidth matrix (topology.py:358-443) */
typedef struct ft_matrix ft_matrix;
int ft_matrix_create(const ft_topo* t, ft_matrix** out); /* snapshot_matrix :446-449 */
void ft_matrix_destroy(ft_matrix* m);
int ft_matrix_hold(ft_matrix* m, const char* func, const int32_t* path, int n, double rate); /* :390-401 */
int ft_matrix_release(ft_matrix* m, const char* func);                                      /* :403-412 */
int ft_matrix_release_path(ft_matrix* m, const char* func, const int32_t* path, int n);     /* :414-428 */
int ft_matrix_residual(const ft_matrix* m, int u, int v, double* out);                      /* :383-384 */
int ft_matrix_budgets(const ft_matrix* m, int gpu, double* egress, double* ingress);
int ft_matrix_aggregate_of(const ft_matrix* m, const char* func, double* out);              /* :433-434 */
/* {"residual": [[u,v,r]...sorted], "egress": [...], "ingress": [...], "held": {func: [[path, rate]...]}} */
int ft_matrix_state_json(const ft_matrix* m, char* buf, size_t cap, size_t* need);

/* ----------------------------------------- NVLink policy (nvlink_sched.py) */
typedef struct {
  int32_t gpus[FT_MAX_PATH];
  int32_t n;          /* GPUs on the path (hops + 1) */
  int32_t held;       /* 1 when held_by == the querying func, 0 for None (shared) */
  double b_min_gbps;
} ft_nvpath;
/* _candidate_paths                                  nvlink_sched.py:42-57 */
int ft_candidate_paths(const ft_topo* t, int src, int dst, int max_hops, ft_nvpath* out, int cap, int* n);
/* select_paths (phase 1, phase 2 busy adoption, shared fallback)  :64-133.
 * trace_json (optional): {"candidates_examined":..,"phase1":[[path,rate]..],"phase2":[..],"shared_fallback":path?} */
int ft_select_paths(ft_matrix* m, const char* func, int src, int dst, int allow_busy, ft_nvpath* out,
                    int cap, int* n, char* trace_json, size_t trace_cap);
/* release_paths                                     nvlink_sched.py:228-230 */
int ft_release_paths(ft_matrix* m, const char* func);
/* claim_direct_for_workflow (+ _evict_and_replan)    nvlink_sched.py:233-285
 * pairs: npairs x (a, b). Result JSON: {"reservations": [[[a,b], rate]..], "degraded": {func: loss}} */
int ft_claim_direct(ft_matrix* m, const int32_t* pairs, int npairs, const char* func, char* buf, size_t cap,
                    size_t* need);
/* distribute_chunks (largest remainder)             nvlink_sched.py:288-302 */
int ft_distribute_chunks(int64_t chunk_count, const double* b_min_gbps, int npaths, int64_t* counts);

/* -------------------------------------------- PCIe policy (pcie_sched.py) */
/* min_rate                                          pcie_sched.py:23-33 */
int ft_min_rate(double data_size_bytes, double slo_ms, double infer_ms, double* out_gbps);
typedef struct ft_pcie_state ft_pcie_state;
/* PcieSchedulerState                                pcie_sched.py:58-77 */
int ft_pcie_state_create(double bw_all_gbps, int batch_chunks, int64_t chunk_bytes, ft_pcie_state** out);
void ft_pcie_state_destroy(ft_pcie_state* s);
/* RateDemand(...) + add (FT_E_INFEASIBLE like the dataclass ctor)  :36-55, :73-74 */
int ft_pcie_state_add(ft_pcie_state* s, const char* func, double bytes, double slo_ms, double infer_ms,
                      double arrival_ms);
int ft_pcie_state_remove(ft_pcie_state* s, const char* func);
int ft_pcie_rate_idle(const ft_pcie_state* s, double* out);                 /* :69-71 */
int ft_demand_slack(const ft_pcie_state* s, const char* func, double now_ms, double* out); /* :49-55 */
/* standalone RateDemand: rate_least and slack_ms(now) (FT_E_INFEASIBLE like the ctor)  :36-55 */
int ft_rate_demand(double bytes, double slo_ms, double infer_ms, double arrival_ms, double now_ms, double* least,
                   double* slack);
/* partition: rates and slo_at_risk in demand insertion order      :80-104 */
int ft_partition(ft_pcie_state* s, double now_ms, double* rates, int32_t* at_risk, int cap, int* n);
/* trigger_batches                                   pcie_sched.py:107-119 */
int ft_trigger_batches(double total_bytes, int64_t chunk_bytes, int batch_chunks, double* out, int cap, int* n);
typedef struct ft_ring ft_ring;
/* PinnedRing                                        pcie_sched.py:122-150 */
int ft_ring_create(double capacity_bytes, double cost_ms_per_mb, int prewarmed, ft_ring** out);
void ft_ring_destroy(ft_ring* r);
int ft_ring_acquire(ft_ring* r, double bytes_needed, double* added_ms);
int ft_ring_state(const ft_ring* r, double* warm_bytes, double* cold_allocated_bytes);
/* default_ring_capacity                             pcie_sched.py:159-162 */
int64_t ft_default_ring_capacity(int pcie_link_count, int64_t batch_bytes);

/* ----------------------------------------------- latency model (simcore.py) */
int ft_pipeline_latency(double size_bytes, const double* hop_gbps, int n, double chunk_bytes, double* out); /* :25-42 */
int ft_pipeline_fill_ms(const double* hop_gbps, int n, double chunk_bytes, double* out);                   /* :45-50 */
int ft_nearest_rank(const double* sorted_values, int n, double pct, double* out);                         /* :247-252 */

/* ----------------------------------------- elastic store (datastore.py) */
int ft_size_class(double size_bytes, int64_t* out);                 /* :24-29 */
int ft_p99(const double* samples, int n, double* out);              /* :32-35 */
typedef struct ft_hist ft_hist;
/* FuncHistogram                                     datastore.py:38-72 */
int ft_hist_create(const char* func, int window, ft_hist** out);
void ft_hist_destroy(ft_hist* h);
int ft_hist_record(ft_hist* h, double now_ms, double size_bytes, double concurrency);
/* r_window_ms, r_size_bytes, r_con, last_request_ms (NaN if none) */
int ft_hist_get(const ft_hist* h, double* r_window, double* r_size, double* r_con, double* last);
int ft_hist_reservation(const ft_hist* h, double* out);
int ft_hist_window_active(const ft_hist* h, double now_ms, int* out);
/* pool_target over histograms                        datastore.py:79-82 */
int ft_pool_target(const ft_hist* const* hists, int n, double now_ms, double floor_bytes, double* out);
typedef struct ft_pool_policy ft_pool_policy;
/* MemoryPool policy: mode 0 autoscale, 1 cache_all, 2 none     datastore.py:91-166 */
int ft_pool_policy_create(int gpu, int mode, double floor_bytes, double native_alloc_ms, double physical_bytes,
                          ft_pool_policy** out);
void ft_pool_policy_destroy(ft_pool_policy* p);
/* allocate -> stable block id (index-free), cost ms    :130-144 */
int ft_pool_policy_allocate(ft_pool_policy* p, double size_bytes, int64_t* block_id, int64_t* class_bytes,
                            double* cost_ms);
int ft_pool_policy_free(ft_pool_policy* p, int64_t block_id);                              /* :146-149 */
int ft_pool_policy_record(ft_pool_policy* p, const char* func, double now_ms, double size, double con);
/* shrink: ids of dropped blocks (the physical memory to release)  :151-166 */
int ft_pool_policy_shrink(ft_pool_policy* p, double now_ms, int64_t* dropped, int cap, int* n);
int ft_pool_policy_target(ft_pool_policy* p, double now_ms, double* out);                  /* :127-128 */
/* R_window and last_request of func's histogram (NaN last if none) — the shrink timer engine.py:656-659 */
int ft_pool_policy_hist(const ft_pool_policy* p, const char* func, double* r_window, double* last);
/* {"blocks": [[class_bytes, in_use, id]..], "pool_bytes":.., "in_use_bytes":..} */
int ft_pool_policy_state_json(const ft_pool_policy* p, char* buf, size_t cap, size_t* need);
#define FT_MAX_CONSUMERS 16
typedef struct {
  int64_t data_id;
  double size_bytes;
  double stored_at_ms;
  int32_t location; /* 0 gpu, 1 host, 2 both              datastore.py:176 */
  int32_t live;
  int32_t n_consumers;
  int32_t consumer_pos[FT_MAX_CONSUMERS];
} ft_stored_object;
/* migration_plan: policy 0 queue_aware, 1 lru; actions 0 reclaim, 1 migrate    :192-222 */
int ft_migration_plan(const ft_stored_object* objs, int n, double pressure_bytes, int policy, int32_t* actions,
                      int32_t* indices, int cap, int* nout);
/* prefetch_back                                     datastore.py:225-238 */
int ft_prefetch_back(const ft_stored_object* objs, int n, double free_bytes, int32_t* indices, int cap, int* nout);

/* ------------------------------------ strategies + data plane (dataplane.py) */
typedef struct {
  int32_t host_oriented, parallel_pcie, unified_interface, pcie_sched, nvlink_sched;
  int32_t pool;      /* 0 autoscale, 1 cache_all, 2 none */
  int32_t migration; /* 0 queue_aware, 1 lru, 2 none */
} ft_strategy;
/* strategy_preset                                   strategies.py:33-62 */
int ft_strategy_preset(const char* name, ft_strategy* out);

typedef struct ft_index ft_index;
/* request-path bookkeeping in one call each (the tube's hot path):
 * store  = ft_index_store + ft_pool_policy_record + ft_pool_policy_hist
 * retire = ft_index_drop + ft_pool_policy_free (block_id >= 0) + ft_pool_policy_hist */
int ft_store_commit(ft_index* x, ft_pool_policy* p, int64_t data_id, int node, int gpu, double size_bytes,
                    double now_ms, const char* producer, int response, double concurrency, double* r_window,
                    double* last);
int ft_retire_commit(ft_index* x, ft_pool_policy* p, int64_t data_id, int64_t block_id, const char* producer,
                     double* r_window, double* last);
/* the same-GPU put in one call (engine.py:383-409, dataplane.py:72-83, datastore.py:51-62):
 * `stream` waits on `waits` (the block's previous users), TMA copy src -> block_ptr
 * (size_bytes, L2 `hints`), records `ready`, then ft_store_commit */
int ft_store_local(ft_index* x, ft_pool_policy* p, int64_t data_id, int node, int gpu, double size_bytes,
                   double now_ms, const char* producer, int response, double concurrency, void* block_ptr,
                   const void* src, void* stream, uint32_t hints, void* const* waits, int nwaits, void* ready,
                   double* r_window, double* last);
/* the same-GPU get into the consumer's input in one call (dataplane.py:184-185,
 * engine.py:667-679): wait `waits`, copy block_ptr -> dst, record `done`; when
 * `retire` (last consumer) also ft_retire_commit */
int ft_fetch_local(ft_index* x, ft_pool_policy* p, int64_t data_id, int64_t block_id, const char* producer,
                   int retire, void* dst, const void* block_ptr, uint64_t bytes, int device, void* stream,
                   uint32_t hints, void* const* waits, int nwaits, void* done, double* r_window, double* last);
/* n x ft_retire_commit (batched fetch) */
int ft_retire_many(ft_index* x, ft_pool_policy* p, int n, const int64_t* data_ids, const int64_t* block_ids,
                   const char* const* producers, double* r_windows, double* lasts);
/* DataIndex                                         dataplane.py:55-107 */
int ft_index_create(double sync_period_ms, double local_lookup_ms, double global_lookup_ms, ft_index** out);
void ft_index_destroy(ft_index* x);
int ft_index_unique_id(ft_index* x, int64_t* out);
int ft_index_store(ft_index* x, int64_t data_id, int node, int gpu, double size_bytes, double now_ms,
                   const char* producer, int response, double* global_visible_ms);
int ft_index_resolve(ft_index* x, int64_t data_id, int node, double now_ms, int* e_node, int* e_gpu,
                     double* cost_ms, double* ready_ms, double* size_bytes);
int ft_index_drop(ft_index* x, int64_t data_id);
int ft_index_relocate(ft_index* x, int64_t data_id, int node, int gpu);

/* link ids (dataplane.py:112-133) */
enum ft_link_kind { FT_LINK_H2D = 0, FT_LINK_D2H = 1, FT_LINK_NV = 2, FT_LINK_NVP_OUT = 3, FT_LINK_NVP_IN = 4, FT_LINK_NET = 5 };
typedef struct { int32_t kind, a, b; } ft_link; /* h2d/d2h: (node, root); nv/net: (u, v); nvp_*: (gpu, -1) */
typedef struct {
  ft_link links[FT_MAX_LINKS];
  double hop_caps[FT_MAX_LINKS];
  int32_t n_links, n_caps;
  double bytes_share, cap_gbps /* NaN = None */, reserved_gbps /* NaN = None */, fill_ms;
} ft_branch;
enum ft_method { FT_INTRA_GPU = 0, FT_INTER_GPU = 1, FT_HOST_GPU = 2, FT_INTER_NODE = 3 };
typedef struct ft_plane ft_plane;
typedef struct ft_plan ft_plan;
/* Dataplane(topo, strategy, matrix, chunk_bytes, intra_gpu_map_ms)  dataplane.py:166-173 */
int ft_plane_create(const ft_topo* t, const ft_strategy* s, ft_matrix* m, double chunk_bytes,
                    double intra_gpu_map_ms, ft_plane** out);
void ft_plane_destroy(ft_plane* p);
/* fetch_plan (gpu -1 = host)                        dataplane.py:176-186 */
int ft_fetch_plan(ft_plane* p, int src_node, int src_gpu, int dst_node, int dst_gpu, double size_bytes,
                  ft_plan** out);
void ft_plan_destroy(ft_plan* plan);
int ft_plan_method(const ft_plan* plan, int* method, double* fixed_ms, int* n_stages);
int ft_plan_add_fixed_ms(ft_plan* plan, double ms); /* engine.py:451-452 */
int ft_plan_stage(const ft_plan* plan, int stage, int* managed, double* pinned_bytes, int* n_branches);
int ft_plan_branch(const ft_plan* plan, int stage, int branch, ft_branch* out);
/* every stage and branch in one call, as doubles (the request path reads
 * these): [n_stages, {managed, pinned_bytes, n_branches, {n_links, {kind, a, b}
 * x n_links, n_caps, caps..., bytes_share, cap_gbps, reserved_gbps, fill_ms}
 * x n_branches} x n_stages]; FT_E_TRUNCATED with *need set when cap is short */
int ft_plan_pack(const ft_plan* plan, double* buf, size_t cap, size_t* need);
/* full plan as JSON (method, size_bytes, fixed_ms, claimed_func, note, stages, latency) */
int ft_plan_json(const ft_plan* plan, char* buf, size_t cap, size_t* need);
/* plan_latency_model                                dataplane.py:351-369 */
int ft_plan_latency(const ft_plan* plan, double* out);
/* Dataplane.release_claim                           dataplane.py:346-348 */
int ft_release_claim(ft_plane* p, const ft_plan* plan);

/* ------------- bandwidth-share scheduler: managed PCIe stages (engine.py) */
typedef struct ft_arbiter ft_arbiter;
/* one per (node, direction); bw_all = pcie_gbps x roots            engine.py:186-190 */
int ft_arbiter_create(double bw_all_gbps, int batch_chunks, int64_t chunk_bytes, ft_arbiter** out);
void ft_arbiter_destroy(ft_arbiter* a);
/* _start_managed_stage (slo fallback 1e12 on InfeasibleDemand)      engine.py:537-575 */
int ft_arbiter_start(ft_arbiter* a, double now_ms, const char* key, double total_bytes, double slo_ms,
                     double infer_ms, double arrival_ms, double per_branch_cap_gbps, int n_branches);
/* _on_boundary                                                      engine.py:637-646 */
int ft_arbiter_boundary(ft_arbiter* a, double now_ms, const char* key);
/* stage drained (flow_complete)                                     engine.py:558-564 */
int ft_arbiter_finish(ft_arbiter* a, double now_ms, const char* key);
/* decisions of the last call: [["partition",{..}],["set_rate",k,rate,per_branch],["pending",k,want],["arm",k,t]] */
int ft_arbiter_decisions_json(const ft_arbiter* a, char* buf, size_t cap, size_t* need);
/* {key: [rate, started, pending|null, anchor, armed|null]} */
int ft_arbiter_state_json(const ft_arbiter* a, char* buf, size_t cap, size_t* need);
/* live state of one stage (pending / armed NaN when None) */
int ft_arbiter_stage(const ft_arbiter* a, const char* key, double* rate, int* started, double* pending,
                     double* armed);
/* earliest armed boundary over all stages (NaN if none) — the live driver's next wake-up */
int ft_arbiter_next_event(const ft_arbiter* a, double* t_ms, char* key, size_t key_cap);

/* ================================================= device side (sm_100a) */
int ft_device_count(int* out);
/* enable peer access dev -> peer (no-op when same device)              */
int ft_peer_enable(int device, int peer);

/* ---- elastic VMM pool (replaces the host-memory store)
 * One reserved VA range per GPU; each block is a cuMemCreate physical
 * allocation (2 MiB granularity) mapped into that range, readable/writable
 * from every peer GPU; exportable as a POSIX fd for other processes.     */
typedef struct ft_vmm_pool ft_vmm_pool;
int ft_vmm_pool_create(int device, uint64_t va_bytes, ft_vmm_pool** out);
void ft_vmm_pool_destroy(ft_vmm_pool* p);
int ft_vmm_granularity(int device, uint64_t* out);
/* blocks are ranges of arenas (one cuMemCreate each, mapped once with every
 * peer's access): map/unmap of a block is bookkeeping; a new arena (FT_POOL_ARENA_BYTES,
 * default 1 GiB, or the block if larger) is mapped only when none has room */
int ft_vmm_block_map(ft_vmm_pool* p, uint64_t bytes, uint64_t* block, void** dptr);
int ft_vmm_block_unmap(ft_vmm_pool* p, uint64_t block);
/* map an arena of `bytes` now, never trimmed (the pool's up-front reservation) */
int ft_vmm_pool_reserve(ft_vmm_pool* p, uint64_t bytes);
/* unmap every unreserved arena no block uses; their ids out (call when idle) */
int ft_vmm_pool_trim(ft_vmm_pool* p, uint64_t* arenas, int cap, int* n);
/* the arena a block lives in, its offset there, the arena's size */
int ft_vmm_block_locate(ft_vmm_pool* p, uint64_t block, uint64_t* arena, uint64_t* offset, uint64_t* arena_bytes);
/* POSIX fd of the block's ARENA (map it whole, add the block's offset) */
int ft_vmm_block_export_fd(ft_vmm_pool* p, uint64_t block, int* fd);
int ft_vmm_pool_stats(const ft_vmm_pool* p, uint64_t* mapped_bytes, uint64_t* reserved_bytes, int* blocks);
/* import a block exported by another process; map it for `device` */
int ft_vmm_import_fd(int device, int fd, uint64_t bytes, void** dptr, uint64_t* handle);
int ft_vmm_unimport(uint64_t handle);
/* SCM_RIGHTS fd passing over a connected AF_UNIX socket (PAPER.md:568 channel) */
/* interprocess CUDA events (function <-> daemon ordering without host syncs):
 * create one exportable event (64-byte handle out) / open a peer's handle; use
 * them with ft_event_record / ft_stream_wait_events / ft_event_destroy */
/* stream memory operations on a word of device memory (cuStreamWriteValue32 after the
 * stream's prior work, with a memory barrier / cuStreamWaitValue32 GEQ, cyclic): the
 * function <-> daemon ordering of the native lane — a cross-process CUDA event
 * dependency takes ~110 us to resolve on B200, a polled word a few us
 * (tools/probe_ipc_latency.py) */
int ft_stream_write32(void* stream, void* addr, uint32_t value);
int ft_stream_wait32(void* stream, const void* addr, uint32_t value);
int ft_ipc_event_create(int device, void** ev, void* handle64);
int ft_ipc_event_open(int device, const void* handle64, void** ev);
int ft_fd_send(int sock, int fd, uint64_t tag);
int ft_fd_recv(int sock, int* fd, uint64_t* tag);
/* shared-memory message channel between a function process and the daemon
 * (PAPER.md:568 fast local channel; replaces the reference's in-process calls of
 * engine.py:342-511 by a cross-process request/reply): two SPSC rings of
 * `slots` slots of `slot_bytes` (dir 0 requests, dir 1 replies) in a memfd the
 * creator passes to the peer (SCM_RIGHTS). recv spins `spin_us`, then sleeps
 * on a futex; timeouts in us (<0: none). FT_E_CLOSED once the peer closed. */
typedef struct ft_chan ft_chan;
int ft_chan_create(uint32_t slot_bytes, uint32_t slots, int* memfd, ft_chan** out);
/* maps a peer's ring pair: its geometry is checked against the memfd's size and kept
 * privately (the peer can write the shared header) */
int ft_chan_attach(int memfd, ft_chan** out);
int ft_chan_send(ft_chan* c, int dir, const void* buf, uint32_t n, int64_t timeout_us);
int ft_chan_recv(ft_chan* c, int dir, void* buf, uint32_t cap, uint32_t* n, int64_t spin_us, int64_t timeout_us);
int ft_chan_close(ft_chan* c);

/* The daemon's native lane (csrc/lane.cc): one C++ worker
 * per function connection serves the hot requests that arrive as binary messages on
 * the connection's rings — unique_id (dataplane.py:69-70), commit of a lent pool
 * block = FaaSTube.store zero copy (engine.py:342-360) + the lend of the producer's
 * next block, same-GPU zero-copy fetch (dataplane.py:184-185, engine.py:667-679) and
 * its release — and hands every other request to the connection's Python thread
 * (ft_lane_conn_next, then one of reply / reply_bin / finish). The tube's decisions
 * for lane objects (histogram sample, accounting, shrink timer, cap check, pool
 * frees, stock refills) run in Python from the ordered event queue (ft_lane_events);
 * index entries are written by the lane at once. The tube adopts a lane object into
 * its own table with ft_lane_take. */
typedef struct ft_lane ft_lane;
typedef struct ft_lane_conn ft_lane_conn;
#pragma pack(push, 1)
typedef struct {         /* one event record (+ name_len bytes of producer name)         */
  uint32_t kind;         /* 1 committed, 2 retired, 3 freed, 4 stock, 5 unpin            */
                         /* (stock: data_id = the connection id, consumers = blocks wanted) */
  uint32_t name_len;
  int64_t data_id;
  int32_t gpu, consumers;
  int64_t block_id;      /* pool policy block id                                          */
  uint64_t nbytes;       /* object bytes (stock: the size class wanted)                   */
  double now_ms;         /* committed: the store time on the tube's clock                 */
  uint64_t event;        /* freed / unpin: cudaEvent_t fence, owned by the receiver       */
} ft_lane_event;
#pragma pack(pop)
typedef struct {
  int64_t data_id, block_id;
  uint64_t nbytes;
  double stored_at_ms;
  void* ready;           /* cudaEvent_t, owned by the taker */
  int32_t gpu, dtype, ndim, remaining, pins, consumers;
} ft_lane_obj;
int ft_lane_create(ft_index* index, int node, double t0_s, ft_lane** out);
int ft_lane_set_pool(ft_lane* lane, int gpu, ft_vmm_pool* pool);
int ft_lane_destroy(ft_lane* lane);
int ft_lane_attach(ft_lane* lane, ft_chan* ch, int sock, ft_lane_conn** out);
/* after hello: the client's GPU, the connection stream and the connection's two sync
 * words in pool memory the client maps (c2d: the client's marks, d2c: the daemon's) */
int ft_lane_conn_set_gpu(ft_lane_conn* c, int gpu, void* stream, void* c2d, void* d2c);
/* the connection stream waits for the client's mark `seq` (Python's slow paths) */
int ft_lane_conn_wait(ft_lane_conn* c, uint32_t seq);
int ft_lane_conn_next(ft_lane_conn* c, void* buf, uint32_t cap, uint32_t* n, int64_t timeout_us);
int ft_lane_conn_served(ft_lane_conn* c, uint32_t* next_acked);
int ft_lane_conn_reply(ft_lane_conn* c, const void* msg, uint32_t n);
int ft_lane_conn_reply_bin(ft_lane_conn* c, const void* payload, uint32_t n, int ok, int fd);
int ft_lane_conn_finish(ft_lane_conn* c);
int ft_lane_conn_mark(ft_lane_conn* c, int* ev);
int ft_lane_conn_known(ft_lane_conn* c, int gpu, uint64_t arena, int* known);
int ft_lane_conn_take_drops(ft_lane_conn* c, uint64_t* arenas, int cap, int* n);
int ft_lane_conn_release(ft_lane_conn* c, uint64_t token);
int ft_lane_conn_close(ft_lane_conn* c);
int ft_lane_dropped(ft_lane* lane, int gpu, uint64_t arena);
int ft_lane_lend(ft_lane_conn* c, int64_t block_id, uint64_t vmm_block, void* ptr, uint64_t class_bytes,
                 uint64_t arena, uint64_t offset, uint64_t arena_bytes, uint64_t* token);
int ft_lane_take_lend(ft_lane_conn* c, uint64_t token, int64_t* block_id);
/* a lendable block for connection conn_id's stock (FT_E_KEY: the connection is gone) */
int ft_lane_stock_put(ft_lane* lane, uint64_t conn_id, int gpu, int64_t block_id, uint64_t vmm_block, void* ptr,
                      uint64_t class_bytes, uint64_t arena, uint64_t offset, uint64_t arena_bytes,
                      void* const* fences, int n_fences);
int ft_lane_conn_id(ft_lane_conn* c, uint64_t* id);
int ft_lane_events(ft_lane* lane, void* buf, uint64_t cap, uint64_t* n, int64_t timeout_us);
int ft_lane_take(ft_lane* lane, int64_t data_id, ft_lane_obj* out, int64_t* shape, char* producer, int producer_cap);
int ft_lane_ids(ft_lane* lane, int gpu, int64_t* ids, int cap, int* n);
/* commits, fetches, dones, unique ids, handed to Python, stock hits, stock misses, adopted, recycled,
 * lost (committed by a client that died before its copy ran: dropped) */
int ft_lane_stats(ft_lane* lane, uint64_t* out, int cap);

/* The function-process side of the lane (csrc/client.cc): one call per hot request
 * of Listing 1 through the daemon — rings, the copy into / out of the mapped block,
 * the sync-word ordering. Views are DLPack tensors whose deleter releases the block. */
typedef struct ft_client ft_client;
/* sock: the connection's socket, read only to tell whether the daemon is alive (-1: never) */
int ft_client_create(ft_chan* ch, int sock, void* c2d, void* d2c, int device, ft_client** out);
int ft_client_destroy(ft_client* cl);
/* the daemon is gone: later sends fail, our streams' waits on its marks are released */
int ft_client_abandon(ft_client* cl);
int ft_client_sent(ft_client* cl, uint64_t* out);
int ft_client_views(ft_client* cl, int* out);  /* live DLPack views */
int ft_client_send(ft_client* cl, const void* msg, uint32_t n);
int ft_client_call(ft_client* cl, const void* req, uint32_t n, void* rep, uint32_t cap, uint32_t* rep_len,
                   int64_t spin_us);
int ft_client_recv(ft_client* cl, void* rep, uint32_t cap, uint32_t* rep_len, int64_t spin_us);
int ft_client_mark(ft_client* cl, void* stream, int32_t* ev);
int ft_client_wait(ft_client* cl, void* stream, int32_t ev);
int ft_client_store(ft_client* cl, void* stream, int32_t wait_ev, void* dst, const void* src, uint64_t n, int engine,
                    const void* req, uint32_t req_len, void* rep, uint32_t cap, uint32_t* rep_len, int64_t spin_us);
int ft_client_fetch(ft_client* cl, void* stream, const void* req, uint32_t req_len, void* rep, uint32_t cap,
                    uint32_t* rep_len, int64_t spin_us);
int ft_client_copy_done(ft_client* cl, void* stream, void* dst, const void* src, uint64_t n, int engine,
                        uint64_t token);
int ft_client_done(ft_client* cl, void* stream, uint64_t token, int ordered);
int ft_client_view(ft_client* cl, void* ptr, int dtype, int ndim, const int64_t* shape, uint64_t token,
                   void** dlmanaged);

/* ---- movers
 * K1/K3 ft_copy: SM-driven bulk copy (TMA cp.async.bulk global->smem->global,
 * mbarrier ring, persistent grid) for same-GPU handoff copies and NVLink
 * peer copies (dst or src may be a peer-mapped pointer). Runs on `device`.
 * fingerprint (optional, device u64[2]): fused integrity digest of the bytes.  */
int ft_copy(void* dst, const void* src, uint64_t bytes, int device, void* stream);
/* same, with explicit engine: 0 auto, 1 TMA bulk, 2 vector ld/st (peer-safe) */
int ft_copy_ex(void* dst, const void* src, uint64_t bytes, int device, void* stream, int engine, int grid);
/* TMA-bulk copy with L2 policies: hints bits 0-1 = source, bits 2-3 = destination
 * (0 evict_normal, 1 evict_first, 2 evict_last) — e.g. a store keeps the pool block
 * L2-resident (dst evict_last) for a same-GPU fetch that follows.            */
int ft_copy_hint(void* dst, const void* src, uint64_t bytes, int device, void* stream, uint32_t hints);
/* stream-ordered doorbells on (peer-)mapped device memory (cross-process handoff
 * without host round trips): ft_signal stores `value` with system-scope release
 * after all prior work on `stream`; ft_wait parks `stream` until *flag >= value
 * (wrap-around compare). */
int ft_signal(uint32_t* flag, uint32_t value, int device, void* stream);
int ft_wait(const uint32_t* flag, uint32_t value, int device, void* stream);  /* gives up after 30 s */
/* as ft_wait, giving up after timeout_ns; then writes the awaited value (or 1) to *err if err != NULL */
int ft_wait_timeout(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* err, int device,
                    void* stream);
/* batched small-message copies: every segment in one launch per 64 segments
 * (local or peer pointers, any alignment) — the launch is paid once per batch */
typedef struct {
  void* dst;
  const void* src;
  uint64_t bytes;
} ft_segment;
int ft_copy_batch(const ft_segment* segs, int n, int device, void* stream);
/* a private non-blocking stream on `device` (torch's stream pool aliases streams) */
int ft_stream_create(int device, void** stream);
int ft_stream_destroy(void* stream);
/* raw CUDA events for stream ordering on the request path (no torch objects) */
int ft_event_create(int device, void** ev);
int ft_event_destroy(void* ev);
int ft_event_record(void* ev, void* stream);
int ft_event_query(void* ev, int* done);
int ft_event_synchronize(void* ev);
int ft_stream_wait_events(void* stream, void* const* evs, int n);
/* a request-path copy in one call: `stream` waits on `waits` (NULL entries skipped),
 * TMA-bulk copy with L2 `hints` (as ft_copy_hint), then records `done` (may be NULL) */
int ft_copy_ordered(void* dst, const void* src, uint64_t bytes, int device, void* stream, uint32_t hints,
                    void* const* waits, int nwaits, void* done);
/* occupy `stream` for `ns` nanoseconds of wall time (global timer, clock independent):
 * the synthetic gFunc compute of the workflow runtime (harness compute_latency_ms) */
int ft_spin_ns(uint64_t ns, int device, void* stream);
/* position-keyed digest of `bytes` (u64 sum of mixed words + xor), device u64[2] out */
int ft_fingerprint(const void* src, uint64_t bytes, uint64_t* out_dev, int device, void* stream);
/* host-side digest of the same definition (for checking against ft_fingerprint) */
int ft_fingerprint_host(const void* src, uint64_t bytes, uint64_t out[2]);
/* one PCIe leg: pinned host -> device (or device -> host) by the copy engine, in batches of
 * batch_bytes (0 = one op), on `stream`. Returns after enqueueing.           */
int ft_pcie_copy(void* dst, const void* src, uint64_t bytes, int to_device, int device, void* stream,
                 uint64_t batch_bytes);
/* host->gFunc striped pass (dataplane.py:203-250 routes):
 * k routes, route i moves [off_i, off_i+len_i) of host_src. A route with
 * staging[i] == NULL is a direct link (CE straight into dst, e.g. the
 * target's own root). A route with a staging buffer lands each chunk in
 * staging[i] on stage_dev[i] by CE, then the staging GPU forwards it to dst
 * over NVLink with ft_copy as soon as that chunk's CE op completes (event
 * chained; chunk ring of ring_chunks slots per staging GPU).
 * streams: 2*k cudaStream_t (CE stream, forward stream per route).       */
int ft_h2g_striped(void* dst, int dst_dev, const void* host_src, uint64_t bytes, int k, const int32_t* stage_dev,
                   const uint64_t* off, const uint64_t* len, void* const* staging, uint64_t chunk_bytes,
                   int ring_chunks, void* const* streams);

/* ---- live PCIe mover + bandwidth-share scheduler (native runtime)
 * Replaces the engine's managed-stage loop (engine.py:537-646) and the pinned
 * staging ring (pcie_sched.py:122-162) on real copy engines. Every host->GPU
 * leg of a fetch is one stage of k routes (dataplane.py:203-250 / _pcie_branches):
 * route i moves [off, off+len) of the host object into dst, straight by the CE
 * of dst's own root (stage_dev == dst_dev) or through a chunk ring on stage_dev
 * with an NVLink forward kernel (fw_stream) into dst. Managed stages join the
 * arbiter's SLO partition and are issued in 5 x 2 MB batches at the stage rate,
 * rate changes on batch boundaries, finished when the last byte lands;
 * unmanaged stages are issued at once. submit() never blocks the host: it
 * parks `consumer_stream` (cuStreamWaitValue32) until the stage's completion
 * word is written after its last byte; route streams first wait for
 * `consumer_stream`'s prior work. Pageable host objects (host_pinned = 0) go
 * through the shared pinned ring (host_ring_bytes, worker threads). The caller
 * keeps host and dst alive until ft_pacer_done reports the ticket. Thread-safe. */
typedef struct ft_pacer ft_pacer;
typedef struct {
  int32_t stage_dev;     /* GPU whose PCIe link carries the route (== dst_dev: direct)   */
  int32_t force_staging; /* stage through the ring even when stage_dev == dst_dev      */
  uint64_t off, len;     /* byte range of the object                                     */
  void* ce_stream;       /* cudaStream_t on stage_dev for the PCIe leg                   */
  void* fw_stream;       /* cudaStream_t on stage_dev for the NVLink forward (staged)    */
} ft_route;
/* bw_all = pcie_gbps x links (engine.py:186-190); staging_slots chunk slots per staging GPU.
 * flags: 1 = log every arbiter call and a trace; 2 = keep bw_all fixed (no link estimator:
 * by default bw_all follows the measured service rate of uncontended direct batches,
 * re-partitioning with an extra "bw" call in the log when it moves >5% up or >15% down) */
int ft_pacer_create(double bw_all_gbps, int links, int batch_chunks, int64_t chunk_bytes, int staging_slots,
                    uint64_t host_ring_bytes, int flags, ft_pacer** out);
/* drains in-flight stages (FT_E_TIMEOUT after 120 s: remaining stages are failed) */
int ft_pacer_destroy(ft_pacer* p);
/* _start_edge_transfer -> _run_stage for a host_gpu plan       engine.py:440-475, 537-575 */
int ft_pacer_submit(ft_pacer* p, const char* key, int managed, double slo_ms, double infer_ms,
                    double per_branch_cap_gbps, void* dst, int dst_dev, const void* host, uint64_t bytes,
                    int host_pinned, int k, const ft_route* routes, void* consumer_stream, uint64_t* ticket);
/* the GPU->host direction (responses, host fetches): k routes move [off, off+len) of the
 * device buffer `src` on src_dev into the PINNED host buffer `host_dst` — CE straight out
 * of src_dev's own root (stage_dev == src_dev), or forward kernel into a staging GPU's ring
 * and its CE to the host; paced by the d2h arbiter (log calls prefixed "d2h:"). The route
 * streams first wait for `producer_stream`'s prior work; host-wait with ft_pacer_wait. */
int ft_pacer_submit_d2h(ft_pacer* p, const char* key, int managed, double slo_ms, double infer_ms,
                        double per_branch_cap_gbps, void* host_dst, const void* src, int src_dev, uint64_t bytes,
                        int k, const ft_route* routes, void* producer_stream, uint64_t* ticket);
/* the routes of a host->GPU fetch in one call (tube._host_to_gpu's planning step):
 * plan it (ft_fetch_plan, dataplane.py:190-250), cut the object into each branch's
 * byte range (shares accumulated in float64, boundaries floored to 256 B), take each
 * route's stream pair on the GPU whose PCIe root carries it from the pairs registered
 * with ft_plane_set_pairs (slot keyed by the consumer stream). Out: k routes, whether
 * the stage is managed (strategy.pcie_sched && stage.managed), the smallest hop cap,
 * bytes the routes forward over NVLink. Feed them to ft_pacer_submit. */
int ft_plane_set_pairs(ft_plane* p, int gpu, int n, void* const* ce_streams, void* const* fw_streams);
int ft_h2g_routes(ft_plane* p, int node, int dst_gpu, uint64_t bytes, void* consumer_stream, ft_route* routes,
                  int cap, int* k, int* managed, double* per_branch_cap, uint64_t* nvlink_bytes);
/* host wait for a ticket's last byte (timeout_ms < 0: forever); returns the stage's status */
int ft_pacer_wait(ft_pacer* p, uint64_t ticket, double timeout_ms);
int ft_pacer_done(ft_pacer* p, uint64_t ticket, int* done);
/* out[0..6] = stages, managed stages, batches, bytes issued, active, failed, blocking-mode */
int ft_pacer_stats(ft_pacer* p, uint64_t* out, int cap);
int ft_pacer_now_ms(ft_pacer* p, double* out);
/* logging = 1: [[t, ticket, "start"|"rate"|"issue"|"land", value], ...] */
int ft_pacer_trace_json(ft_pacer* p, char* buf, size_t cap, size_t* need);
/* logging = 1: every arbiter call [[t, "start"|"boundary"|"finish"|"bw", key, decisions, arg], ...] with
 * arg = the per-branch cap a start used / the new bw_all of a "bw" (= set_bw) call; GPU->host calls
 * are prefixed "d2h:". Replayable through the arbiter. */
int ft_pacer_log_json(ft_pacer* p, char* buf, size_t cap, size_t* need);
/* arbiter state, as ft_arbiter_state_json */
int ft_pacer_state_json(ft_pacer* p, char* buf, size_t cap, size_t* need);

#ifdef __cplusplus
}
#endif
#endif /* FAASTUBE_H */
