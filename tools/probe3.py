"""Cycle accounting of the QK ring (measurement aid; needs build/probe/libakv_probe3.so)."""
import ctypes, os, sys
os.environ["AKV_LIB_PROBE"] = os.path.join(os.path.dirname(__file__), "..", "build", "probe", "libakv_probe3.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_2409_16546_b200 import KVStore, _lib
from paper_2409_16546_b200 import attention_decode as AD
from paper_2409_16546_b200.synth import generate_batch

B, H, n = 16, 32, 4096
K, V, Q = generate_batch(B, H, n, 128, 1, 7, workers=len(os.sched_getaffinity(0)))
st = KVStore(B, H, 128, n, strict=False)
for t0 in range(0, n, 1024):
    st.append(torch.from_numpy(np.ascontiguousarray(K[:, t0:t0+1024]).view(np.int16)).view(B, H, -1, 128),
              torch.from_numpy(np.ascontiguousarray(V[:, t0:t0+1024]).view(np.int16)).view(B, H, -1, 128))
st.check()
q = torch.from_numpy(Q.view(np.int16)).view(B, H, 128).cuda()
L = _lib.lib()
buf = (ctypes.c_ulonglong * 16)()
for force in (None, 16):
    for _ in range(3):
        AD.decode(q, st, force_tier=force)
    torch.cuda.synchronize()
    L.akv_probe_read_qk(buf)
    R = 5
    for _ in range(R):
        AD.decode(q, st, force_tier=force)
    torch.cuda.synchronize()
    L.akv_probe_read_qk(buf)
    v = list(buf)
    warps = 1184 * R
    ctas = 148 * R
    print(f"   per-stage: meta {v[11]/ctas/110:.0f} bulk {v[8]/ctas/110:.0f} rows {v[9]/ctas/110:.0f} "
          f"arrive {v[10]/ctas/110:.0f} cyc (stages/CTA ~110)")
    print(f"force={force}: producer/CTA: wait_empty {v[0]/ctas:.0f} issue {v[1]/ctas:.0f} total {v[2]/ctas:.0f} cyc; "
          f"consumer/warp: wait_full {v[3]/warps:.0f} compute {v[4]/warps:.0f} total {v[5]/warps:.0f} cyc (warps {warps/R:.0f})")
