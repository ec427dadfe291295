"""Latency model and percentile — mirror of tubesim ``simcore.py:21-50,
247-252`` over libfaastube. (The reference's event queue and fluid network
simulate links; this build drives the real links, so they are not mirrored.)
"""

from __future__ import annotations

import ctypes as C

from ._lib import LIB

GBPS_TO_BYTES_PER_MS = 1e6
PHASES = ("queuing", "host_to_gfunc", "gfunc_to_gfunc", "compute", "internode")


def ms_for(bytes_count: float, gbps: float) -> float:
    return bytes_count / (gbps * GBPS_TO_BYTES_PER_MS)


def _arr(xs):
    return (C.c_double * max(1, len(xs)))(*[float(x) for x in xs])


def pipeline_latency(size_bytes: float, hop_gbps: list, chunk_bytes: float) -> float:
    """simcore.py:25-42"""
    x = C.c_double()
    LIB.ft_pipeline_latency(float(size_bytes), _arr(hop_gbps), len(hop_gbps), float(chunk_bytes), C.byref(x))
    return x.value


def pipeline_fill_ms(hop_gbps: list, chunk_bytes: float) -> float:
    """simcore.py:45-50"""
    x = C.c_double()
    LIB.ft_pipeline_fill_ms(_arr(hop_gbps), len(hop_gbps), float(chunk_bytes), C.byref(x))
    return x.value


def nearest_rank(sorted_values: list, pct: float) -> float:
    """simcore.py:247-252 (the p99 estimator every report uses)"""
    x = C.c_double()
    LIB.ft_nearest_rank(_arr(sorted_values), len(sorted_values), float(pct), C.byref(x))
    return x.value
