"""ctypes binding of libfaastube.so (include/faastube.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2411_01830_b200/csrc``). There is no fallback: if the library
is missing every entry point raises ``LibraryMissing``.

Status codes map onto the exception types the reference raises
(``tubesim`` topology.py:40, pcie_sched.py:19, dataplane.py:26-31,
datastore.py:134-136/188).
"""

from __future__ import annotations

import ctypes as C
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FAASTUBE_LIB", os.path.join(_HERE, "libfaastube.so"))

MAX_PATH = 8
MAX_LINKS = 8
MAX_CONSUMERS = 16


class LibraryMissing(RuntimeError):
    pass


class FaasTubeError(RuntimeError):
    code = -1


class TopologyError(ValueError):
    """topology.py:40"""


class InfeasibleDemand(ValueError):
    """pcie_sched.py:19"""


class MissingData(KeyError):
    """dataplane.py:26"""


class DuplicateStore(ValueError):
    """dataplane.py:30"""


class HardPressure(RuntimeError):
    """datastore.py:188"""


class CudaError(RuntimeError):
    pass


class Truncated(RuntimeError):
    pass


class NotSupported(RuntimeError):
    pass


class WaitTimeout(TimeoutError):
    pass


_ERRORS = {
    1: TopologyError,
    2: InfeasibleDemand,
    3: MissingData,
    4: DuplicateStore,
    5: HardPressure,
    6: MemoryError,
    7: CudaError,
    8: ValueError,
    9: Truncated,
    10: KeyError,
    11: NotSupported,
    12: WaitTimeout,
    13: ConnectionError,
}

i32, i64, u64, dbl, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
P = C.POINTER
vp = C.c_void_p
cstr = C.c_char_p


class NvPathC(C.Structure):
    _fields_ = [("gpus", i32 * MAX_PATH), ("n", i32), ("held", i32), ("b_min_gbps", dbl)]


class StoredObjectC(C.Structure):
    _fields_ = [("data_id", i64), ("size_bytes", dbl), ("stored_at_ms", dbl), ("location", i32),
                ("live", i32), ("n_consumers", i32), ("consumer_pos", i32 * MAX_CONSUMERS)]


class StrategyC(C.Structure):
    _fields_ = [("host_oriented", i32), ("parallel_pcie", i32), ("unified_interface", i32),
                ("pcie_sched", i32), ("nvlink_sched", i32), ("pool", i32), ("migration", i32)]


class LinkC(C.Structure):
    _fields_ = [("kind", i32), ("a", i32), ("b", i32)]


class RouteC(C.Structure):
    _fields_ = [("stage_dev", i32), ("force_staging", i32), ("off", u64), ("len", u64), ("ce_stream", vp),
                ("fw_stream", vp)]


class SegmentC(C.Structure):
    _fields_ = [("dst", vp), ("src", vp), ("bytes", u64)]


class BranchC(C.Structure):
    _fields_ = [("links", LinkC * MAX_LINKS), ("hop_caps", dbl * MAX_LINKS), ("n_links", i32),
                ("n_caps", i32), ("bytes_share", dbl), ("cap_gbps", dbl), ("reserved_gbps", dbl),
                ("fill_ms", dbl)]


# name: (restype, argtypes); restype None means the int status convention
_SIGS = {
    "ft_last_error": (cstr, []),
    "ft_version": (cstr, []),
    "ft_topo_create": (None, [cstr, P(vp)]),
    "ft_topo_destroy": (C.c_void_p, [vp]),
    "ft_topo_gpu_count": (None, [vp, P(C.c_int)]),
    "ft_topo_node_of": (None, [vp, C.c_int, P(C.c_int)]),
    "ft_topo_root_of": (None, [vp, C.c_int, P(C.c_int)]),
    "ft_topo_nvlink_gbps": (None, [vp, C.c_int, C.c_int, P(dbl)]),
    "ft_topo_neighbors": (None, [vp, C.c_int, P(i32), C.c_int, P(C.c_int)]),
    "ft_topo_pair_kind": (None, [vp, C.c_int, C.c_int, P(C.c_int)]),
    "ft_topo_switch_port_gbps": (None, [vp, C.c_int, P(dbl)]),
    "ft_topo_degree_gbps": (None, [vp, C.c_int, P(dbl)]),
    "ft_topo_pair_bandwidth": (None, [vp, C.c_int, C.c_int, P(dbl)]),
    "ft_topo_rate": (None, [vp, C.c_int, P(dbl)]),
    "ft_topo_roots": (None, [vp, P(i32), C.c_int, P(C.c_int)]),
    "ft_matrix_create": (None, [vp, P(vp)]),
    "ft_matrix_destroy": (C.c_void_p, [vp]),
    "ft_matrix_hold": (None, [vp, cstr, P(i32), C.c_int, dbl]),
    "ft_matrix_release": (None, [vp, cstr]),
    "ft_matrix_release_path": (None, [vp, cstr, P(i32), C.c_int]),
    "ft_matrix_residual": (None, [vp, C.c_int, C.c_int, P(dbl)]),
    "ft_matrix_budgets": (None, [vp, C.c_int, P(dbl), P(dbl)]),
    "ft_matrix_aggregate_of": (None, [vp, cstr, P(dbl)]),
    "ft_matrix_state_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_candidate_paths": (None, [vp, C.c_int, C.c_int, C.c_int, P(NvPathC), C.c_int, P(C.c_int)]),
    "ft_select_paths": (None, [vp, cstr, C.c_int, C.c_int, C.c_int, P(NvPathC), C.c_int, P(C.c_int),
                               C.c_char_p, sz]),
    "ft_release_paths": (None, [vp, cstr]),
    "ft_claim_direct": (None, [vp, P(i32), C.c_int, cstr, C.c_char_p, sz, P(sz)]),
    "ft_distribute_chunks": (None, [i64, P(dbl), C.c_int, P(i64)]),
    "ft_min_rate": (None, [dbl, dbl, dbl, P(dbl)]),
    "ft_pcie_state_create": (None, [dbl, C.c_int, i64, P(vp)]),
    "ft_pcie_state_destroy": (C.c_void_p, [vp]),
    "ft_pcie_state_add": (None, [vp, cstr, dbl, dbl, dbl, dbl]),
    "ft_pcie_state_remove": (None, [vp, cstr]),
    "ft_pcie_rate_idle": (None, [vp, P(dbl)]),
    "ft_demand_slack": (None, [vp, cstr, dbl, P(dbl)]),
    "ft_rate_demand": (None, [dbl, dbl, dbl, dbl, dbl, P(dbl), P(dbl)]),
    "ft_partition": (None, [vp, dbl, P(dbl), P(i32), C.c_int, P(C.c_int)]),
    "ft_trigger_batches": (None, [dbl, i64, C.c_int, P(dbl), C.c_int, P(C.c_int)]),
    "ft_ring_create": (None, [dbl, dbl, C.c_int, P(vp)]),
    "ft_ring_destroy": (C.c_void_p, [vp]),
    "ft_ring_acquire": (None, [vp, dbl, P(dbl)]),
    "ft_ring_state": (None, [vp, P(dbl), P(dbl)]),
    "ft_default_ring_capacity": (i64, [C.c_int, i64]),
    "ft_pipeline_latency": (None, [dbl, P(dbl), C.c_int, dbl, P(dbl)]),
    "ft_pipeline_fill_ms": (None, [P(dbl), C.c_int, dbl, P(dbl)]),
    "ft_nearest_rank": (None, [P(dbl), C.c_int, dbl, P(dbl)]),
    "ft_size_class": (None, [dbl, P(i64)]),
    "ft_p99": (None, [P(dbl), C.c_int, P(dbl)]),
    "ft_hist_create": (None, [cstr, C.c_int, P(vp)]),
    "ft_hist_destroy": (C.c_void_p, [vp]),
    "ft_hist_record": (None, [vp, dbl, dbl, dbl]),
    "ft_hist_get": (None, [vp, P(dbl), P(dbl), P(dbl), P(dbl)]),
    "ft_hist_reservation": (None, [vp, P(dbl)]),
    "ft_hist_window_active": (None, [vp, dbl, P(C.c_int)]),
    "ft_pool_target": (None, [P(vp), C.c_int, dbl, dbl, P(dbl)]),
    "ft_pool_policy_create": (None, [C.c_int, C.c_int, dbl, dbl, dbl, P(vp)]),
    "ft_pool_policy_destroy": (C.c_void_p, [vp]),
    "ft_pool_policy_allocate": (None, [vp, dbl, P(i64), P(i64), P(dbl)]),
    "ft_pool_policy_free": (None, [vp, i64]),
    "ft_pool_policy_record": (None, [vp, cstr, dbl, dbl, dbl]),
    "ft_pool_policy_shrink": (None, [vp, dbl, P(i64), C.c_int, P(C.c_int)]),
    "ft_pool_policy_target": (None, [vp, dbl, P(dbl)]),
    "ft_pool_policy_hist": (None, [vp, cstr, P(dbl), P(dbl)]),
    "ft_pool_policy_state_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_migration_plan": (None, [P(StoredObjectC), C.c_int, dbl, C.c_int, P(i32), P(i32), C.c_int, P(C.c_int)]),
    "ft_prefetch_back": (None, [P(StoredObjectC), C.c_int, dbl, P(i32), C.c_int, P(C.c_int)]),
    "ft_strategy_preset": (None, [cstr, P(StrategyC)]),
    "ft_index_create": (None, [dbl, dbl, dbl, P(vp)]),
    "ft_index_destroy": (C.c_void_p, [vp]),
    "ft_index_unique_id": (None, [vp, P(i64)]),
    "ft_index_store": (None, [vp, i64, C.c_int, C.c_int, dbl, dbl, cstr, C.c_int, P(dbl)]),
    "ft_index_resolve": (None, [vp, i64, C.c_int, dbl, P(C.c_int), P(C.c_int), P(dbl), P(dbl), P(dbl)]),
    "ft_index_drop": (None, [vp, i64]),
    "ft_index_relocate": (None, [vp, i64, C.c_int, C.c_int]),
    "ft_plane_create": (None, [vp, P(StrategyC), vp, dbl, dbl, P(vp)]),
    "ft_plane_destroy": (C.c_void_p, [vp]),
    "ft_fetch_plan": (None, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dbl, P(vp)]),
    "ft_plan_destroy": (C.c_void_p, [vp]),
    "ft_plan_method": (None, [vp, P(C.c_int), P(dbl), P(C.c_int)]),
    "ft_plan_add_fixed_ms": (None, [vp, dbl]),
    "ft_plan_stage": (None, [vp, C.c_int, P(C.c_int), P(dbl), P(C.c_int)]),
    "ft_plan_branch": (None, [vp, C.c_int, C.c_int, P(BranchC)]),
    "ft_plan_pack": (None, [vp, P(dbl), sz, P(sz)]),
    "ft_plan_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_plan_latency": (None, [vp, P(dbl)]),
    "ft_release_claim": (None, [vp, vp]),
    "ft_arbiter_create": (None, [dbl, C.c_int, i64, P(vp)]),
    "ft_arbiter_destroy": (C.c_void_p, [vp]),
    "ft_arbiter_start": (None, [vp, dbl, cstr, dbl, dbl, dbl, dbl, dbl, C.c_int]),
    "ft_arbiter_boundary": (None, [vp, dbl, cstr]),
    "ft_arbiter_finish": (None, [vp, dbl, cstr]),
    "ft_arbiter_decisions_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_arbiter_state_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_arbiter_stage": (None, [vp, cstr, P(dbl), P(C.c_int), P(dbl), P(dbl)]),
    "ft_arbiter_next_event": (None, [vp, P(dbl), C.c_char_p, sz]),
    # device side
    "ft_device_count": (None, [P(C.c_int)]),
    "ft_peer_enable": (None, [C.c_int, C.c_int]),
    "ft_vmm_pool_create": (None, [C.c_int, u64, P(vp)]),
    "ft_vmm_pool_destroy": (C.c_void_p, [vp]),
    "ft_vmm_granularity": (None, [C.c_int, P(u64)]),
    "ft_vmm_block_map": (None, [vp, u64, P(u64), P(vp)]),
    "ft_vmm_block_unmap": (None, [vp, u64]),
    "ft_vmm_block_export_fd": (None, [vp, u64, P(C.c_int)]),
    "ft_vmm_pool_reserve": (None, [vp, u64]),
    "ft_vmm_pool_trim": (None, [vp, P(u64), C.c_int, P(C.c_int)]),
    "ft_vmm_block_locate": (None, [vp, u64, P(u64), P(u64), P(u64)]),
    "ft_vmm_pool_stats": (None, [vp, P(u64), P(u64), P(C.c_int)]),
    "ft_vmm_import_fd": (None, [C.c_int, C.c_int, u64, P(vp), P(u64)]),
    "ft_vmm_unimport": (None, [u64]),
    "ft_ipc_event_create": (None, [C.c_int, P(vp), C.c_char_p]),
    "ft_ipc_event_open": (None, [C.c_int, C.c_char_p, P(vp)]),
    "ft_fd_send": (None, [C.c_int, C.c_int, u64]),
    "ft_fd_recv": (None, [C.c_int, P(C.c_int), P(u64)]),
    "ft_plane_set_pairs": (None, [vp, C.c_int, C.c_int, P(vp), P(vp)]),
    "ft_h2g_routes": (None, [vp, C.c_int, C.c_int, u64, vp, vp, C.c_int, P(C.c_int), P(C.c_int), P(dbl),
                             P(u64)]),
    "ft_lane_create": (None, [vp, C.c_int, dbl, P(vp)]),
    "ft_lane_set_pool": (None, [vp, C.c_int, vp]),
    "ft_lane_destroy": (None, [vp]),
    "ft_lane_attach": (None, [vp, vp, C.c_int, P(vp)]),
    "ft_lane_conn_set_gpu": (None, [vp, C.c_int, vp, vp, vp]),
    "ft_lane_conn_wait": (None, [vp, C.c_uint32]),
    "ft_stream_write32": (None, [vp, vp, C.c_uint32]),
    "ft_stream_wait32": (None, [vp, vp, C.c_uint32]),
    "ft_lane_conn_next": (None, [vp, vp, C.c_uint32, P(C.c_uint32), i64]),
    "ft_lane_conn_served": (None, [vp, P(C.c_uint32)]),
    "ft_lane_conn_reply": (None, [vp, C.c_char_p, C.c_uint32]),
    "ft_lane_conn_reply_bin": (None, [vp, C.c_char_p, C.c_uint32, C.c_int, C.c_int]),
    "ft_lane_conn_finish": (None, [vp]),
    "ft_lane_conn_mark": (None, [vp, P(C.c_int)]),
    "ft_lane_conn_known": (None, [vp, C.c_int, u64, P(C.c_int)]),
    "ft_lane_conn_take_drops": (None, [vp, P(u64), C.c_int, P(C.c_int)]),
    "ft_lane_conn_release": (None, [vp, u64]),
    "ft_lane_conn_close": (None, [vp]),
    "ft_lane_dropped": (None, [vp, C.c_int, u64]),
    "ft_lane_lend": (None, [vp, i64, u64, vp, u64, u64, u64, u64, P(u64)]),
    "ft_lane_take_lend": (None, [vp, u64, P(i64)]),
    "ft_lane_stock_put": (None, [vp, u64, C.c_int, i64, u64, vp, u64, u64, u64, u64, P(vp), C.c_int]),
    "ft_lane_conn_id": (None, [vp, P(u64)]),
    "ft_lane_events": (None, [vp, vp, u64, P(u64), i64]),
    "ft_lane_take": (None, [vp, i64, vp, P(i64), C.c_char_p, C.c_int]),
    "ft_lane_ids": (None, [vp, C.c_int, P(i64), C.c_int, P(C.c_int)]),
    "ft_lane_stats": (None, [vp, P(u64), C.c_int]),
    "ft_client_create": (None, [vp, C.c_int, vp, vp, C.c_int, P(vp)]),
    "ft_client_abandon": (None, [vp]),
    "ft_client_destroy": (None, [vp]),
    "ft_client_sent": (None, [vp, P(u64)]),
    "ft_client_views": (None, [vp, P(C.c_int)]),
    "ft_client_send": (None, [vp, C.c_char_p, C.c_uint32]),
    "ft_client_call": (None, [vp, C.c_char_p, C.c_uint32, vp, C.c_uint32, P(C.c_uint32), i64]),
    "ft_client_recv": (None, [vp, vp, C.c_uint32, P(C.c_uint32), i64]),
    "ft_client_mark": (None, [vp, vp, P(C.c_int32)]),
    "ft_client_wait": (None, [vp, vp, C.c_int32]),
    "ft_client_store": (None, [vp, vp, C.c_int32, vp, vp, u64, C.c_int, C.c_char_p, C.c_uint32, vp, C.c_uint32,
                               P(C.c_uint32), i64]),
    "ft_client_fetch": (None, [vp, vp, C.c_char_p, C.c_uint32, vp, C.c_uint32, P(C.c_uint32), i64]),
    "ft_client_copy_done": (None, [vp, vp, vp, vp, u64, C.c_int, u64]),
    "ft_client_done": (None, [vp, vp, u64, C.c_int]),
    "ft_client_view": (None, [vp, vp, C.c_int, C.c_int, P(i64), u64, P(vp)]),
    "ft_chan_create": (None, [C.c_uint32, C.c_uint32, P(C.c_int), P(vp)]),
    "ft_chan_attach": (None, [C.c_int, P(vp)]),
    "ft_chan_send": (None, [vp, C.c_int, C.c_char_p, C.c_uint32, i64]),
    "ft_chan_recv": (None, [vp, C.c_int, vp, C.c_uint32, P(C.c_uint32), i64, i64]),
    "ft_chan_close": (None, [vp]),
    "ft_copy": (None, [vp, vp, u64, C.c_int, vp]),
    "ft_copy_ex": (None, [vp, vp, u64, C.c_int, vp, C.c_int, C.c_int]),
    "ft_copy_hint": (None, [vp, vp, u64, C.c_int, vp, C.c_uint32]),
    "ft_signal": (None, [vp, C.c_uint32, C.c_int, vp]),
    "ft_wait": (None, [vp, C.c_uint32, C.c_int, vp]),
    "ft_wait_timeout": (None, [vp, C.c_uint32, u64, vp, C.c_int, vp]),
    "ft_copy_batch": (None, [vp, C.c_int, C.c_int, vp]),
    "ft_store_commit": (None, [vp, vp, i64, C.c_int, C.c_int, dbl, dbl, cstr, C.c_int, dbl, P(dbl), P(dbl)]),
    "ft_retire_commit": (None, [vp, vp, i64, i64, cstr, P(dbl), P(dbl)]),
    "ft_store_local": (None, [vp, vp, i64, C.c_int, C.c_int, dbl, dbl, cstr, C.c_int, dbl, vp, vp, vp, C.c_uint32,
                              P(vp), C.c_int, vp, P(dbl), P(dbl)]),
    "ft_fetch_local": (None, [vp, vp, i64, i64, cstr, C.c_int, vp, vp, u64, C.c_int, vp, C.c_uint32, P(vp), C.c_int,
                              vp, P(dbl), P(dbl)]),
    "ft_retire_many": (None, [vp, vp, C.c_int, vp, vp, vp, vp, vp]),
    "ft_stream_create": (None, [C.c_int, P(vp)]),
    "ft_stream_destroy": (None, [vp]),
    "ft_event_create": (None, [C.c_int, P(vp)]),
    "ft_event_destroy": (None, [vp]),
    "ft_event_record": (None, [vp, vp]),
    "ft_event_query": (None, [vp, P(C.c_int)]),
    "ft_event_synchronize": (None, [vp]),
    "ft_stream_wait_events": (None, [vp, P(vp), C.c_int]),
    "ft_copy_ordered": (None, [vp, vp, u64, C.c_int, vp, C.c_uint32, P(vp), C.c_int, vp]),
    "ft_spin_ns": (None, [u64, C.c_int, vp]),
    "ft_fingerprint": (None, [vp, u64, vp, C.c_int, vp]),
    "ft_fingerprint_host": (None, [vp, u64, P(u64)]),
    "ft_pcie_copy": (None, [vp, vp, u64, C.c_int, C.c_int, vp, u64]),
    "ft_h2g_striped": (None, [vp, C.c_int, vp, u64, C.c_int, P(i32), P(u64), P(u64), P(vp), u64, C.c_int,
                              P(vp)]),
    # live PCIe mover + bandwidth-share scheduler
    "ft_pacer_create": (None, [dbl, C.c_int, C.c_int, i64, C.c_int, u64, C.c_int, P(vp)]),
    "ft_pacer_destroy": (None, [vp]),
    "ft_pacer_submit": (None, [vp, cstr, C.c_int, dbl, dbl, dbl, vp, C.c_int, vp, u64, C.c_int, C.c_int,
                               P(RouteC), vp, P(u64)]),
    "ft_pacer_submit_d2h": (None, [vp, cstr, C.c_int, dbl, dbl, dbl, vp, vp, C.c_int, u64, C.c_int, P(RouteC), vp,
                                   P(u64)]),
    "ft_pacer_wait": (None, [vp, u64, dbl]),
    "ft_pacer_done": (None, [vp, u64, P(C.c_int)]),
    "ft_pacer_stats": (None, [vp, P(u64), C.c_int]),
    "ft_pacer_now_ms": (None, [vp, P(dbl)]),
    "ft_pacer_trace_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_pacer_log_json": (None, [vp, C.c_char_p, sz, P(sz)]),
    "ft_pacer_state_json": (None, [vp, C.c_char_p, sz, P(sz)]),
}

HEADER_SYMBOLS = tuple(_SIGS)


class _Lib:
    def __init__(self):
        self._dll = None

    def load(self):
        if self._dll is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_2411_01830_b200/csrc` (no CPU fallback exists)")
            dll = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(dll, name)
                fn.argtypes = args
                fn.restype = C.c_int if res is None else res
            self._dll = dll
        return self._dll

    def raw(self, name):
        return getattr(self.load(), name)

    def __getattr__(self, name):
        if not name.startswith("ft_"):
            raise AttributeError(name)
        fn = self.raw(name)
        res = _SIGS[name][0]
        if res is not None:
            setattr(self, name, fn)          # cached: later lookups skip __getattr__
            return fn

        def call(*args):
            rc = fn(*args)
            if rc != 0:
                raise_status(rc)
            return rc
        call.__name__ = name
        setattr(self, name, call)
        return call


LIB = _Lib()


def destroyer(name):
    """A finalizer for handles released by ``name``: holds the library itself, so it
    still works while the interpreter tears module globals down (no stray
    "NoneType has no attribute" errors at exit) and never raises."""
    lib = LIB

    def destroy(h):
        try:
            lib.raw(name)(h)
        except Exception:  # noqa: BLE001 - best effort in finalizers
            pass
    return destroy


def raise_status(rc):
    msg = LIB.raw("ft_last_error")()
    msg = msg.decode() if msg else f"status {rc}"
    exc = _ERRORS.get(rc, FaasTubeError)
    raise exc(msg)


def call_status(name, *args):
    """Call returning the raw status (for truncation retries)."""
    return LIB.raw(name)(*args)


def json_out(name, *args):
    """Call a (…, buf, cap, need) JSON producer with automatic sizing."""
    cap = 1 << 14
    while True:
        buf = C.create_string_buffer(cap)
        need = sz()
        rc = LIB.raw(name)(*args, buf, cap, C.byref(need))
        if rc == 9 and need.value > cap:
            cap = need.value
            continue
        if rc != 0:
            raise_status(rc)
        return json.loads(buf.value.decode())


def enc(s):
    return s.encode() if isinstance(s, str) else s


def none_if_nan(x):
    return None if x != x else x


def nan_if_none(x):
    return float("nan") if x is None else float(x)
