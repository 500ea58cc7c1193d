"""One cluster-kernel variant (tfft_tune_select) on a small fp32 N = 8192
batch, checked against numpy; run under `timeout` per variant."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_02520_b200 import _lib, make_plan
from paper_2405_02520_b200.fft_core import fit_group_size
from paper_2405_02520_b200.fft_core.plan import native_plan
v = int(sys.argv[1]); b = int(sys.argv[2]) if len(sys.argv) > 2 else 64
lib = _lib.load()
n = 8192
plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
h = native_plan(plan, 0)
x = torch.randn(b, n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
_lib.check(lib.tfft_tune_select(_lib.FP32, 13, v))
_lib.check(lib.tfft_execute(h.handle, x.data_ptr(), y.data_ptr(), b, 0, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
ref = np.fft.fft(x.cpu().numpy().astype(np.complex128), axis=1)
err = np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref)
print("variant", v, "batch", b, "rel err", err, flush=True)
