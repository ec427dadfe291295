"""TEST INFRASTRUCTURE ONLY — replayable restatement of the reference engine's
managed PCIe stages (the per-function bandwidth-share scheduler).

Restates ``engine.py:116-142`` (``_ManagedStage``) and ``engine.py:537-646``
(``_start_managed_stage``, ``_pcie_resync``, ``_set_stage_rate``,
``_earliest_boundary``, ``_arm_boundary``, ``_on_boundary``) for ONE
(node, direction) scheduler, with the engine's clock passed in explicitly.
The reference's event queue and fluid network are replaced by the caller:
``arm`` decisions are boundary events the caller must deliver back through
``boundary(now, key)``; ``finish(now, key)`` is the engine's
"all flows of the stage completed" callback (``engine.py:558-564``).

Every call returns the decisions it made, in order:
  ("partition", {func: rate})          pcie_sched.partition result
  ("set_rate", key, rate, per_branch)  engine.py:614-622
  ("pending", key, want)               engine.py:609-611
  ("arm", key, boundary_ms)            engine.py:628-635 (only when pushed)
"""

from __future__ import annotations

import math

from .decisions import Demand, Infeasible, LinkShare, ms_for, split_rates

EPS = 1e-9  # engine.py:26


class _Stage:  # engine.py:116-142
    def __init__(self, demand, n_flows, cap, batch_bytes):
        self.key = demand.func
        self.demand = demand
        self.n_flows = n_flows
        self.cap = cap
        self.batch_bytes = batch_bytes
        self.rate = 0.0
        self.pending = None
        self.anchor = 0.0
        self.armed = None
        self.started = False

    def next_boundary(self, after):
        if not self.started or self.rate <= EPS:
            return None
        dur = ms_for(self.batch_bytes, self.rate)
        k = max(1, math.floor((after - self.anchor) / dur + 1e-9) + 1)
        return self.anchor + k * dur


class Arbiter:
    def __init__(self, bw_all, batch_chunks=5, chunk=2 * 10**6):
        self.share = LinkShare(bw_all, batch_chunks, chunk)
        self.batch_bytes = chunk * batch_chunks
        self.stages = {}
        self.risk_flags = 0
        self._out = None

    # engine.py:537-575 (the per-branch cap is min hop cap over branches)
    def start(self, now, name, total, slo, infer, arrival, per_branch_cap, n_branches):
        self._out = []
        try:
            d = Demand(name, total, slo, infer, arrival)
        except Infeasible:
            d = Demand(name, total, 1e12, 0.0, arrival)
            d.at_risk = True
            self.risk_flags += 1
        st = _Stage(d, n_branches, per_branch_cap * n_branches, self.batch_bytes)
        self.stages[st.key] = st
        self.share.demands[d.func] = d
        self._resync(now)
        return self._out

    def set_bw(self, now, bw_all, link_gbps):
        """Live pacer only (no engine counterpart): the measured link capacity
        changed; stage caps rise to at least the link per flow; re-partition."""
        self._out = []
        self.share.bw_all = bw_all
        for st in self.stages.values():
            st.cap = max(st.cap, link_gbps * st.n_flows)
        self._resync(now)
        return self._out

    def finish(self, now, key):  # engine.py:558-564
        self._out = []
        self.share.demands.pop(key, None)
        self.stages.pop(key, None)
        self._resync(now)
        return self._out

    def boundary(self, now, key):  # engine.py:637-646
        self._out = []
        st = self.stages.get(key)
        if st is None:
            return self._out
        st.armed = None
        if st.pending is not None:
            others = sum(x.rate for x in self.stages.values() if x.started and x.key != st.key)
            self._set(now, st, min(st.pending, max(0.0, self.share.bw_all - others)))
        self._resync(now)
        return self._out

    def _resync(self, now):  # engine.py:581-612
        stages = list(self.stages.values())
        targets = split_rates(self.share, now)
        self._out.append(("partition", dict(targets)))
        committed = sum(m.rate for m in stages if m.started)
        order = sorted(stages, key=lambda m: (m.demand.slack(now), m.demand.arrival, m.demand.func))
        leftover = 0.0
        for m in order:
            target = targets.get(m.demand.func, 0.0) + leftover
            want = min(target, m.cap)
            leftover = max(0.0, target - want)
            if not m.started:
                room = self.share.bw_all - committed
                rate = min(want, room)
                if rate > EPS and (rate >= want - EPS or committed <= EPS):
                    self._set(now, m, rate)
                    committed += rate
                else:
                    b = self._earliest(stages, now)
                    if b is not None:
                        self._arm(now, m, b)
            elif abs(want - m.rate) > 1e-6:
                m.pending = want
                self._out.append(("pending", m.key, want))
                self._arm(now, m, m.next_boundary(now))

    def _set(self, now, m, rate):  # engine.py:614-622
        m.rate = rate
        m.started = True
        m.pending = None
        m.anchor = now
        self._out.append(("set_rate", m.key, rate, rate / m.n_flows))

    @staticmethod
    def _earliest(stages, now):  # engine.py:624-626
        ts = [b for b in (m.next_boundary(now) for m in stages) if b is not None]
        return min(ts) if ts else None

    def _arm(self, now, m, t):  # engine.py:628-635
        if t is None or t <= now + EPS:
            return
        if m.armed is not None and m.armed <= t + 1e-9:
            return
        m.armed = t
        self._out.append(("arm", m.key, t))
