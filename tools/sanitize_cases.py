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
