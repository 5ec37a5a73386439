"""Small decode steps for compute-sanitizer beyond smoke(): GQA groups (qk5 tensor-core
kernel, pv quad path), forced tiers and truncation.  Exits non-zero on a parity failure."""
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from gpu_helpers import Case, close  # noqa: E402

from paper_2409_16546_b200 import attention_decode as AD  # noqa: E402

for g, n, kw in [(4, 600, {}), (8, 300, {}), (4, 300, {"force_tier": 12})]:
    c = Case(B=1, Hkv=2, g=g, n=n, seed=5)
    r = c.gpu(**kw)
    o = r.o.cpu().numpy()
    for u, b, hq, j in c.units():
        ref = c.oracle(u, j, force_tier=kw.get("force_tier"))
        assert close(o[b, hq], ref.o), (g, n, kw, u, j)
    print(f"g={g} n={n} {kw} ok")

# the serving path (no v-tier export): pv stage fast path / GQA quad path, qk5 ring
for g, n in [(1, 600), (4, 600), (8, 300)]:
    c = Case(B=1, Hkv=2, g=g, n=n, seed=9)
    o = AD.decode_step(c.q, c.store).o.cpu().numpy()
    for u, b, hq, j in c.units():
        assert close(o[b, hq], c.oracle(u, j).o), ("fast", g, n, u, j)
    print(f"fast path g={g} n={n} ok")

# round 2: paper-like scales (pv6 DENSE stages, SIMD rule), the prefill writer (Case uses
# KVStore.append -> akv_append_ws), akv_append_at, metered reads
for g, n in [(1, 600), (2, 300), (4, 300)]:
    c = Case(B=1, Hkv=2, g=g, n=n, seed=13, lo=-0.5, hi=0.5)
    o = AD.decode_step(c.q, c.store).o.cpu().numpy()
    for u, b, hq, j in c.units():
        assert close(o[b, hq], c.oracle(u, j).o), ("paper-like", g, n, u, j)
    print(f"paper-like g={g} n={n} ok")

import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_2409_16546_b200 import _lib  # noqa: E402

c = Case(B=1, Hkv=2, n=300, seed=17)
k = torch.zeros(1, 2, 128, dtype=torch.int16, device="cuda")
v = torch.zeros(1, 2, 128, dtype=torch.int16, device="cuda")
_lib.check(_lib.lib().akv_append_at(ctypes.byref(c.store.c_store), k.data_ptr(), v.data_ptr(), 299,
                                    c.store.status_dev.data_ptr(), torch.cuda.current_stream().cuda_stream),
           "akv_append_at")
torch.cuda.synchronize()
from paper_2409_16546_b200 import AccessCounter  # noqa: E402
w = c.store.read_element(0, 0, 5, 0, 16, AccessCounter())
print("append_at + metered read ok", w)
