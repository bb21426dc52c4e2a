"""Bisect the thread-target CNOT folds on cfg4 golden rows (debug helper)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_2404_06314_b200 import configs
from paper_2404_06314_b200.engine import BatchEngine, BatchRequest
g = np.load(os.path.join(ROOT, "tests", "golden", "cfg4.npz"))
spec = configs.CONFIGS[4]
circ, obs, wrt = configs.build(spec, configs.native_api())
NR = int(os.environ.get("NR", "8"))
x = g["x_rows"][:NR]
for mode in ("jac", "fwd"):
    eng = BatchEngine(device="cuda:0")
    r = eng.run_batch(BatchRequest(circ, obs, {"w": g["w"]}, x, wrt=wrt if mode == "jac" else ()))
    e = np.abs(r.expectations - (g["expect"] if mode == "jac" else g["expect_fwd"])[:NR]).max(axis=1)
    msg = f"{os.environ.get('VQC_FOLD_THREAD_TARGETS')} {os.environ.get('VQC_FWD_REG','')} {mode} expect err per row {np.array2string(e, precision=2)}"
    if mode == "jac":
        j = np.abs(r.gradients["w"] - g["jac_w"][:NR]).max(axis=(1, 2))
        msg += f" jac_w err {np.array2string(j, precision=2)}"
    print(msg, flush=True)
