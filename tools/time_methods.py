"""Time param-shift / SPSA through BatchEngine.run_batch on the GPU (host
numpy in/out, like the reference's run_batch). Prints one JSON line per case."""

import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

import torch  # noqa: E402

from paper_2404_06314_b200 import configs  # noqa: E402
from paper_2404_06314_b200.engine import BatchEngine, BatchRequest  # noqa: E402

CASES = [(2, "param-shift", 1024), (2, "spsa", 1024), (3, "param-shift", 256), (3, "spsa", 4096),
         (4, "param-shift", 64), (4, "spsa", 1024)]

eng = BatchEngine(device="cuda:0")
for cfg_id, method, rows in CASES:
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec)
    req = BatchRequest(circ, obs, {"w": w}, x[:rows], method=method, wrt=wrt, spsa_samples=8)
    eng.run_batch(req)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        eng.run_batch(req)
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({"config": f"cfg{cfg_id}", "method": method, "rows": rows,
                      "s_per_call": dt, "samples_per_s": rows / dt}), flush=True)
