import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2409_16546_b200 import KVStore
from paper_2409_16546_b200 import attention_decode as AD
from paper_2409_16546_b200.synth import generate_batch
import os
B, H, n = 16, 32, 4096
K, V, Q = generate_batch(B, H, n, 128, 1, 7, workers=len(os.sched_getaffinity(0)))
st = KVStore(B, H, 128, n, strict=False)
for t0 in range(0, n - 1, 1024):
    t1 = min(n - 1, t0 + 1024)
    st.append(torch.from_numpy(np.ascontiguousarray(K[:, t0:t1]).view(np.int16)).view(B, H, -1, 128),
              torch.from_numpy(np.ascontiguousarray(V[:, t0:t1]).view(np.int16)).view(B, H, -1, 128))
st.check()
q = torch.from_numpy(Q.view(np.int16)).view(B, H, 128)
kn = torch.from_numpy(np.ascontiguousarray(K[:, n - 1]).view(np.int16)).view(B, H, 128)
vn = torch.from_numpy(np.ascontiguousarray(V[:, n - 1]).view(np.int16)).view(B, H, 128)
res = {}
for zin in (False, True):
    for zout in (False, True):
        dg = AD.DecodeGraph(st, 1, rewind_to=n - 1, zero_copy_out=zout, zero_copy_in=zin).capture()
        dg.host_q.copy_(q); dg.host_k.copy_(kn); dg.host_v.copy_(vn)
        for _ in range(10): o = dg.step()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(50): o = dg.step()
        dt = (time.perf_counter() - t0) / 50 * 1e6
        res[f"in{int(zin)}_out{int(zout)}"] = (round(dt, 1), float(o.abs().sum()))
print(json.dumps(res))
