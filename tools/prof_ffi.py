"""Per-entry-point time of libfaastube calls on the same-GPU put/get path."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import _lib
from paper_2411_01830_b200.tube import FaaSTube

acc = collections.defaultdict(lambda: [0, 0.0])
orig_getattr = _lib._Lib.__getattr__
def getattr_(self, name):
    fn = orig_getattr(self, name)
    def timed(*a, _fn=fn, _n=name):
        t0 = time.perf_counter()
        try:
            return _fn(*a)
        finally:
            e = acc[_n]; e[0] += 1; e[1] += time.perf_counter() - t0
    object.__setattr__(self, name, timed)
    return timed
_lib._Lib.__getattr__ = getattr_
for k in list(vars(_lib.LIB)):
    if k.startswith("ft_"):
        delattr(_lib.LIB, k)

tube = FaaSTube("faastube")
x = torch.ones(4096, dtype=torch.uint8, device="cuda:0")
out = torch.empty_like(x)
def loop(n, zero_copy):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        d = tube.unique_id()
        tube.store(d, x)
        v = tube.fetch(d, device=0) if zero_copy else tube.fetch(d, device=0, out=out)
        ts.append(time.perf_counter() - t0)
        del v
    return sorted(ts)
loop(300, False); loop(300, True)
acc.clear()
N = 3000
ts = loop(N, False)
print(f"store+fetch(out) host us p50 {1e6*ts[N//2]:.1f} p99 {1e6*ts[int(N*.99)]:.1f}")
tot = 0
for k, (c, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    tot += t
    print(f"  {k:32s} calls/iter {c/N:5.2f}  us/iter {1e6*t/N:7.2f}  us/call {1e6*t/max(c,1):6.2f}")
print(f"  total ffi us/iter {1e6*tot/N:.1f}")
ts = loop(N, True)
print(f"store+fetch(view) host us p50 {1e6*ts[N//2]:.1f} p99 {1e6*ts[int(N*.99)]:.1f}")
