"""Per-function PCIe bandwidth-share scheduler (isolation quotas) — the
engine's managed-stage logic (tubesim ``engine.py:116-142, 537-646``) in
libfaastube (``ft_arbiter_*``).

Two drivers share this state machine:

* replay: feed the reference engine's event times (start / boundary /
  finish) and compare decisions — the parity tests do this;
* live: ``tube.FaaSTube`` starts a stage per host<->GPU fetch, paces each
  stage's batches at the arbiter's rate on the copy engines, delivers
  boundary events when ``next_event`` says, and finishes stages when their
  last batch lands.
"""

from __future__ import annotations

import ctypes as C

from ._lib import LIB, destroyer, enc, json_out


class StageArbiter:
    def __init__(self, bw_all_gbps: float, batch_chunks: int = 5, chunk_bytes: int = 2 * 10**6):
        self.bw_all_gbps = bw_all_gbps
        self.batch_bytes = batch_chunks * chunk_bytes
        h = C.c_void_p()
        LIB.ft_arbiter_create(float(bw_all_gbps), int(batch_chunks), int(chunk_bytes), C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_arbiter_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def start(self, now_ms, key, total_bytes, slo_ms, infer_ms, arrival_ms, per_branch_cap_gbps, n_branches):
        LIB.ft_arbiter_start(self._h, float(now_ms), enc(key), float(total_bytes), float(slo_ms), float(infer_ms),
                             float(arrival_ms), float(per_branch_cap_gbps), int(n_branches))
        return self.decisions()

    def boundary(self, now_ms, key):
        LIB.ft_arbiter_boundary(self._h, float(now_ms), enc(key))
        return self.decisions()

    def finish(self, now_ms, key):
        LIB.ft_arbiter_finish(self._h, float(now_ms), enc(key))
        return self.decisions()

    def decisions(self) -> list:
        return json_out("ft_arbiter_decisions_json", self._h)

    def state(self) -> dict:
        return json_out("ft_arbiter_state_json", self._h)

    def stage(self, key):
        r, s, p, a = C.c_double(), C.c_int(), C.c_double(), C.c_double()
        LIB.ft_arbiter_stage(self._h, enc(key), C.byref(r), C.byref(s), C.byref(p), C.byref(a))
        return {"rate": r.value, "started": bool(s.value), "pending": None if p.value != p.value else p.value,
                "armed": None if a.value != a.value else a.value}

    def next_event(self):
        t = C.c_double()
        key = C.create_string_buffer(256)
        LIB.ft_arbiter_next_event(self._h, C.byref(t), key, 256)
        return (None, None) if t.value != t.value else (t.value, key.value.decode())
