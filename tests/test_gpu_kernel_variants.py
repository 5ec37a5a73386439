"""The opt-in kernel variants run the same GPU parity checks (in a child process: the
kernel choice is read from the environment once per process).

* AKV_QK_KERNEL=qk9: the tcgen05 / TMEM GQA score kernel (akv_qk9.cuh).
* AKV_QK5_TMA=1: qk5 staged by TMA gather4 instead of cp.async.
"""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"AKV_QK_KERNEL": "qk9"}, {"AKV_QK5_TMA": "1"}])
def test_variant_parity(env):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sel = "gqa or forced or truncated or flat_scales or config_parity or unknown_target or fast_path"
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", sel]
    res = subprocess.run(cmd, cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert " passed" in res.stdout
