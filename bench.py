#!/usr/bin/env python
"""Benchmark: batched statevector forward + adjoint gradients on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0. One step = one forward + adjoint-gradient pass (VJP,
upstream = ones, the autograd semantics) over the whole batch of the
headline workload, BASELINE.json config 4 (16 qubits, 10 layers, batch
16384 sharded over the GPUs, 16 per-qubit <Z_i>, gradients w.r.t. weights and
inputs), plus the one NCCL all-reduce of the weight gradients for N > 1.

* ``value``: samples/s over the whole job, device-timed with CUDA events on
  the launching stream (max over ranks), inputs resident in HBM, L2 flushed
  between timed steps.
* ``e2e``: the same metric through the host-buffer C ABI call
  (``vqc_run_batch_host``: H2D inputs, run, D2H results, synchronise).
* ``roofline``: FP64 bound; algorithmic flops per sample
  F = 2^n [6R + 6R(1+K) + 4 Rn K] over the state-evolution kernels' measured
  time; peak = measured DFMA throughput (profiles/peaks_fp64.json).
* ``cpu_baseline``: the CPU oracle (C restatement of the reference kernels,
  OpenMP over rows like the reference's thread pool) on a bounded row sample.
* ``--impl reference``: that CPU path alone, as the reference arm.
* ``--gpus N`` without an outer torchrun re-launches this script under
  ``torch.distributed.run`` with N ranks (one per GPU, NCCL); rows shard
  with the reference's split and the weight gradient is all-reduced once
  per step. ``--dry-run`` runs the same launcher / sharding / all-reduce /
  max-over-ranks path on gloo with a host-only step (CPU test of the N > 1
  plumbing).
* ``parity``: the bench checks its own timed outputs: the first 8 rows
  against the reference's goldens (tests/golden) and, at N = 1, the last
  rows against the oracle rows the cpu_baseline leg computes anyway.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QNN fwd+adjoint-grad samples/sec vs qubits/layers; % of HBM/FP64 roofline"
HEADLINE_CFG = 4
FP64_PEAK_FALLBACK = 37.1  # TFLOP/s, tools/probe_peaks.cu on this pool (profiles/peaks_fp64.json)


def fp64_peak() -> tuple[float, str]:
    path = os.path.join(ROOT, "profiles", "peaks_fp64.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["fp64_fma_tflops"]), "measured (tools/probe_peaks.cu DFMA loop, profiles/peaks_fp64.json)"
    except Exception:
        return FP64_PEAK_FALLBACK, "measured earlier on this pool (tools/probe_peaks.cu)"


def fp32_peak() -> tuple[float, str]:
    """FFMA throughput (complex64 mode's pipe): measured by tools/probe_peaks.cu
    when profiles/peaks_fp64.json carries it, else twice the FP64 figure
    (B200: 128 FP32 vs 64 FP64 lanes per SM)."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_fp64.json")) as fh:
            return float(json.load(fh)["fp32_fma_tflops"]), "measured (tools/probe_peaks.cu FFMA loop)"
    except Exception:
        return 2.0 * fp64_peak()[0], "2 x the measured FP64 DFMA figure (128 vs 64 lanes per SM)"


def hbm_peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def workload_desc(spec) -> str:
    ent = {"cnot_ring": "CNOT ring", "cz_chain": "CZ chain", "cz_all": "CZ all-to-all"}[spec.entangler]
    obs = {"zzzz": "<Z0Z1Z2Z3>", "per_qubit": f"{spec.n} per-qubit <Z_i>", "sum_z": "sum_i <Z_i>",
           "z0z1": "<Z0 Z1>"}[spec.observables]
    wrt = "weights and inputs" if spec.wrt_inputs else "weights"
    return (f"cfg{spec.cfg_id}: {spec.n} qubits, {spec.layers} layers ({spec.enc} encoding, "
            f"{'/'.join(spec.trainable)} trainable, {ent}), batch {spec.batch}, {obs}, "
            f"forward + adjoint VJP grads w.r.t. {wrt}, complex128")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """``--gpus N`` (N > 1) outside torchrun: run this script under
    ``torch.distributed.run`` with N ranks on this node (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def nccl_log_setup() -> str | None:
    """NCCL_DEBUG=INFO into per-job files (not stdout, which carries the one
    JSON line); rank 0 summarises the communicator lines afterwards."""
    if "NCCL_DEBUG" in os.environ and "NCCL_DEBUG_FILE" not in os.environ:
        return None
    d = f"/tmp/vqc_bench_nccl_{os.environ.get('MASTER_PORT', 'x')}_{os.getppid()}"
    os.makedirs(d, exist_ok=True)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(d, "%h.%p.log"))
    return d


def nccl_summary(d: str | None) -> dict | None:
    """Communicator evidence (version, nRanks, NVLS / channel lines)."""
    import glob
    if not d:
        return None
    files = sorted(glob.glob(os.path.join(d, "*.log")))
    keep = ("NCCL version", "Init COMPLETE", "NVLS", "nRanks", "P2P/CUMEM", "via P2P")
    lines = []
    for f in files:
        try:
            with open(f) as fh:
                lines += [ln.strip()[-220:] for ln in fh if any(k in ln for k in keep)]
        except OSError:
            pass
    return {"files": len(files), "lines": lines[:16]}


def host_cpu() -> dict:
    """Host CPU identity: physical cores (the reference's default thread
    count, batch.py:47-51), logical cores and the model string."""
    try:
        import psutil
        physical = psutil.cpu_count(logical=False)
    except Exception:
        physical = None
    logical = os.cpu_count() or 1
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = logical
    return {"physical": physical or logical, "logical": logical, "usable": usable, "model": model}


# ----------------------------------------------------------------------------- CPU arms

def cpu_reference_rows(spec, xs, threads: int, combined: bool = False):
    """Reference semantics on the CPU oracle for rows ``xs``.

    combined=False: run_batch(method='adjoint', wrt) (the Jacobian, M+1
    reverse sweeps per row; batch.py:147-217) + the backward einsum
    (model.py:140-142) — what the reference's QuantumModule.backward costs.
    combined=True: the best-case VJP-equivalent reference call, one
    observable sum_m O_m (observables.py:21-47; valid for the bench's
    row-uniform upstream) — 2 reverse sweeps per row.
    Returns (seconds, per-row VJP rows (len(xs), n_cols), expectations)."""
    from paper_2404_06314_b200 import configs
    from paper_2404_06314_b200.observables import Observable
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import oracle_batch
    circ, obs, wrt = configs.build(spec, configs.native_api())
    _, w = configs.inputs_and_weights(spec, batch=1)
    if combined:
        obs = [Observable(tuple(t for o in obs for t in o.terms))]
    t0 = time.perf_counter()
    e, jac = oracle_batch(circ, obs, {"w": w}, xs, wrt, threads=threads)
    up = np.ones((len(xs), len(obs)))
    vjp_rows = np.concatenate([np.einsum("bm,bmp->bp", up, jac[k]) for k in wrt], axis=1)
    _ = vjp_rows.sum(axis=0)
    return time.perf_counter() - t0, vjp_rows, e


def cpu_rows_for(spec, threads: int, target_s: float, min_rounds: int = 4) -> int:
    """Bounded sample: a multiple of ``threads`` rows (>= min_rounds rows per
    thread, SURVEY §8d asks >= 4T on cfg4) taking about target_s."""
    x, _ = configs_inputs(spec)
    t1, _, _ = cpu_reference_rows(spec, x[:threads], threads)   # one row per thread
    rounds = max(min_rounds, int(target_s / max(t1, 1e-4)))
    return int(min(spec.batch, rounds * threads))


def configs_inputs(spec):
    from paper_2404_06314_b200 import configs
    return configs.inputs_and_weights(spec)


def cpu_baseline(spec, target_s: float = 10.0) -> tuple[dict, dict]:
    """Both CPU numbers on the LAST rows of the batch (so the bench's own GPU
    outputs for those rows can be checked against them): the reference's
    Jacobian + einsum backward, and its VJP-equivalent combined-observable
    call. Returns (cpu_baseline dict, oracle rows for the parity check)."""
    cpu = host_cpu()
    threads = cpu["physical"]
    rows = cpu_rows_for(spec, threads, target_s)
    x, _ = configs_inputs(spec)
    lo = spec.batch - rows
    dt, vjp_rows, e = cpu_reference_rows(spec, x[lo:], threads)
    dtc, vjp_c, _ = cpu_reference_rows(spec, x[lo:], threads, combined=True)
    out = {"value": rows / dt, "unit": "samples/s", "cores": threads, "kind": "port",
           "sample": f"rows {lo}..{spec.batch - 1} ({rows} of {spec.batch}) of cfg{spec.cfg_id}; "
                     f"oracle = C restatement of vqckit _kernels.py + run_batch, reference "
                     f"backward semantics (Jacobian, M+1 reverse sweeps per row, + einsum), "
                     f"{threads} OpenMP threads = physical cores, {dt:.1f} s",
           "cpu_model": cpu["model"], "physical_cores": cpu["physical"],
           "logical_cores": cpu["logical"],
           "vjp_equivalent": {"value": rows / dtc, "unit": "samples/s", "seconds": dtc,
                              "call": "one combined observable sum_m O_m (observables.py:21-47), "
                                      "2 reverse sweeps per row; valid for upstream = ones"},
           "rows_measured": rows, "extrapolation": "linear in rows (rows are independent)"}
    check = {"lo": lo, "vjp_rows": vjp_rows, "vjp_rows_combined": vjp_c, "expect": e}
    return out, check


def config_block(spec, world: int) -> dict:
    """The ``config`` object both arms print (same keys, so the driver can
    match the lines)."""
    return {"workload": workload_desc(spec), "batch": spec.batch, "qubits": spec.n,
            "layers": spec.layers, "observables": len(configs_terms(spec)),
            "mode": "vjp (upstream = ones)",
            "parallelism": f"dp{world} (row shards, split_workload; 1 NCCL all-reduce of the "
                           "weight grads per step)" if world > 1 else "dp1",
            "l2": "flushed between timed steps (256 MiB write); states stream through "
                  "a >1 GiB HBM workspace"}


def configs_terms(spec):
    from paper_2404_06314_b200 import configs
    return configs.observable_terms(spec)


def run_reference(args, spec):
    """Reference arm: the oracle (reference kernels restated in C) on all
    physical cores, a bounded row sample per step; rank 0 only."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    cpu = host_cpu()
    threads = cpu["physical"]
    rows = cpu_rows_for(spec, threads, target_s=args.ref_step_s, min_rounds=1)
    x, _ = configs_inputs(spec)
    for _ in range(args.warmup):
        cpu_reference_rows(spec, x[:threads], threads)
    times = [cpu_reference_rows(spec, x[:rows], threads)[0] for _ in range(args.steps)]
    per_step = statistics.mean(times)
    value = rows / per_step
    dtc = cpu_reference_rows(spec, x[:rows], threads, combined=True)[0]
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(spec, max(world, args.gpus)),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": f"{rows} rows per step of cfg{spec.cfg_id} (bounded sample; "
                                   "rows are independent so samples/s extrapolates linearly); "
                                   "reference backward semantics (Jacobian + einsum)",
                         "cpu_model": cpu["model"], "physical_cores": cpu["physical"],
                         "logical_cores": cpu["logical"],
                         "vjp_equivalent": {"value": rows / dtc, "unit": "samples/s",
                                            "call": "combined observable sum_m O_m"}},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

class GpuWorkload:
    def __init__(self, spec, rank: int, world: int, device, precision: str = "complex128"):
        import torch

        from paper_2404_06314_b200 import configs, native
        from paper_2404_06314_b200.engine import BatchEngine, split_workload
        self.spec = spec
        self.torch = torch
        circ, obs, wrt = configs.build(spec, configs.native_api())
        x, w = configs.inputs_and_weights(spec)
        lo, hi = split_workload(spec.batch, world)[rank]
        self.lo, self.hi = lo, hi
        self.rows = hi - lo
        self.precision = precision
        self.engine = BatchEngine(device=device, precision=precision)
        self.plan, self.layout = self.engine.plans.get(circ, obs, wrt, torch.device(device))
        self.flat = self.engine.base_flat(circ, {"w": w})
        self.x_host = np.ascontiguousarray(x[lo:hi])
        self.M = len(obs)
        dev = torch.device(device)
        self.dev = dev
        self.d_x = torch.from_numpy(self.x_host).to(dev)
        self.d_w = torch.from_numpy(self.flat).to(dev)
        self.d_up = torch.ones((self.rows, self.M), dtype=torch.float64, device=dev)
        self.expect = torch.empty((self.rows, self.M), dtype=torch.float64, device=dev)
        self.vsum = torch.empty((self.layout.n_cols,), dtype=torch.float64, device=dev)
        self.rows_out = torch.empty((self.rows, self.layout.n_cols), dtype=torch.float64, device=dev)
        self.ws = torch.empty(self.plan.workspace_bytes(self.rows, native.VQC_MODE_VJP),
                              dtype=torch.uint8, device=dev)
        self.native = native

        # e2e host buffers in pinned (page-locked) memory: inputs, upstream and
        # the step's results (expectations, per-row VJP rows, weight VJP)
        def pinned(shape):
            return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

        xh = pinned(self.x_host.shape)
        xh[...] = self.x_host
        self.x_host = xh
        self.up_host = pinned((self.rows, self.M))
        self.up_host[...] = 1.0
        self.out_host = (pinned((self.rows, self.M)), pinned((self.rows, self.layout.n_cols)),
                         pinned((self.layout.n_cols,)))

    def step(self, world: int):
        stream = self.torch.cuda.current_stream(self.dev).cuda_stream
        self.plan.adjoint(self.d_x, self.d_w, self.d_up, self.expect, None, self.rows_out,
                          self.vsum, self.ws, stream)
        launches = self.native.last_launch_count()
        if world > 1:
            self.torch.distributed.all_reduce(self.vsum)
        return launches

    def step_host(self, world: int):
        e, _, rows, vsum = self.plan.run_batch_host(self.x_host, self.flat, upstream=self.up_host,
                                                    out=self.out_host)
        if world > 1:
            t = self.torch.from_numpy(vsum).to(self.dev)
            self.torch.distributed.all_reduce(t)
            vsum = t.cpu().numpy()
        return e, rows, vsum

    def e2e_bytes(self):
        h2d = self.x_host.nbytes + self.flat.nbytes + self.up_host.nbytes
        d2h = self.rows * self.M * 8 + self.rows * self.layout.n_cols * 8 + self.layout.n_cols * 8
        return h2d, d2h


def roofline_from_profile(spec, prof: dict, steps: int, rows_total: int,
                          precision: str = "complex128") -> dict:
    from paper_2404_06314_b200 import configs
    peak, how = fp64_peak() if precision == "complex128" else fp32_peak()
    evo = {k: v for k, v in prof.items() if k.startswith("pass_") or k.startswith("smem_")}
    evo_ms = sum(v[0] for v in evo.values()) / steps
    evo_launches = sum(v[1] for v in evo.values()) / steps
    flops = configs.flops_per_sample(spec, K=1) * rows_total
    achieved = flops / (evo_ms * 1e-3) / 1e12 if evo_ms > 0 else 0.0
    total_ms = sum(v[0] for v in prof.values()) / steps
    out = {
        "bound": "fp64" if precision == "complex128" else "fp32", "achieved": achieved, "peak": peak,
        "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": None,
        "kernel": "+".join(sorted(evo)) if evo else None,
        "kernel_share_of_step": evo_ms / total_ms if total_ms > 0 else None,
        "launches_per_step": evo_launches,
        "algorithmic_flops_per_sample": configs.flops_per_sample(spec, K=1),
        "peak_source": how,
    }
    # measured DRAM traffic (ncu dram__bytes_read.sum + dram__bytes_write.sum
    # over every launch of one fwd+adjoint call, profiles/r0N/traffic_cfg<id>.json:
    # the latest round that captured this config)
    try:
        rnd = next(r for r in ("r02", "r01")
                   if os.path.exists(os.path.join(ROOT, "profiles", r, f"traffic_cfg{spec.cfg_id}.json")))
        with open(os.path.join(ROOT, "profiles", rnd, f"traffic_cfg{spec.cfg_id}.json")) as fh:
            tr = json.load(fh)
        per_sample = sum(v.get("dram_bytes_per_sample", 0.0) for k, v in tr["kernels"].items()
                         if k.startswith("pass_") or k.startswith("smem_"))
        if per_sample > 0:
            out["traffic"] = per_sample * rows_total / max(evo_launches, 1.0)
            out["traffic_unit"] = "DRAM bytes per state-evolution launch (ncu, scaled to this step's rows)"
            out["traffic_bytes_per_sample"] = per_sample
            out["traffic_source"] = f"profiles/{rnd}/traffic_cfg{spec.cfg_id}.json"
    except (OSError, KeyError, ValueError, StopIteration):
        pass
    hb = configs.hbm_bytes_per_sample(spec, K=1)
    if hb > 0 and evo_ms > 0:
        gbs = hb * rows_total / (evo_ms * 1e-3) / 1e9
        out["hbm_model"] = {"bytes_per_sample": hb, "achieved_gbs": gbs, "peak_gbs": hbm_peak(),
                            "frac": gbs / hbm_peak()}
    return out


def _rel_err(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float((np.abs(a - b) / np.maximum(1.0, np.abs(b))).max())


def parity_check(spec, wl, oracle_rows=None) -> dict:
    """The timed step's own outputs (expectations and per-row VJP rows of
    the LAST timed step) against (a) the reference's goldens for the first
    rows of the batch this rank holds and (b) oracle rows from the
    cpu_baseline leg (last rows of the batch, N = 1). Tolerance 1e-10."""
    out = {"tol": 1e-10 if wl.precision == "complex128" else 1e-5, "checked_rows": []}
    errs = []
    exp = wl.expect.cpu().numpy()
    rows = wl.rows_out.cpu().numpy()
    P = spec.num_weights
    try:
        g = np.load(os.path.join(ROOT, "tests", "golden", f"cfg{spec.cfg_id}.npz"))
        lo, hi = wl.lo, min(wl.hi, wl.lo + 8, int(g["expect"].shape[0]))
        if hi > lo:
            ref_w = g["jac_w"][lo:hi].sum(axis=1)
            errs += [_rel_err(exp[:hi - lo], g["expect"][lo:hi]),
                     _rel_err(rows[:hi - lo, :P], ref_w)]
            if "vjp_x_rows" in g.files:
                errs.append(_rel_err(rows[:hi - lo, P:], g["vjp_x_rows"][lo:hi]))
            out["checked_rows"].append(f"{lo}..{hi - 1} vs reference goldens")
    except (OSError, KeyError):
        pass
    if oracle_rows is not None:
        c_lo = oracle_rows["lo"]
        if wl.lo <= c_lo and wl.hi == spec.batch:
            k = c_lo - wl.lo
            errs += [_rel_err(exp[k:], oracle_rows["expect"]), _rel_err(rows[k:], oracle_rows["vjp_rows"])]
            out["checked_rows"].append(f"{c_lo}..{spec.batch - 1} vs oracle (cpu_baseline leg)")
    out["max_err"] = max(errs) if errs else None
    out["ok"] = bool(errs) and max(errs) <= out["tol"]
    return out


def measure_gpu(spec, args, rank, world, device, flush_buf, with_e2e: bool, steps: int, warmup: int,
                oracle_rows_fn=None, precision: str = "complex128"):
    import torch
    import torch.distributed as dist

    from paper_2404_06314_b200 import native
    wl = GpuWorkload(spec, rank, world, device, precision)
    for _ in range(warmup):
        wl.step(world)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device()).start()
    native.profile_enable(True)
    launches = 0
    for k in range(steps):
        flush_buf.add_(1)               # L2 flush (256 MiB write), outside the events
        ev[k][0].record()
        launches += wl.step(world)
        ev[k][1].record()
    torch.cuda.synchronize()
    prof = native.profile_report()
    native.profile_enable(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / steps
    value = spec.batch / (ms_per_step * 1e-3)
    res = {"value": value, "ms_per_step": ms_per_step, "gpu_launches": launches, "clocks": clk,
           "kernels": {k: {"ms_per_step": v[0] / steps, "launches_per_step": v[1] / steps}
                       for k, v in prof.items()},
           "roofline": roofline_from_profile(spec, prof, steps, wl.rows, precision)}
    if with_e2e:
        for _ in range(max(1, warmup)):
            wl.step_host(world)
        if world > 1:
            dist.barrier()
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            wl.step_host(world)
            times.append(time.perf_counter() - t0)
        tt = torch.tensor([sum(times)], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item()) / steps
        h2d, d2h = wl.e2e_bytes()
        res["e2e"] = {"value": spec.batch / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                      "path": "vqc_run_batch_host (numpy in/out, pinned host buffers)"}
    res["plan"] = json.loads(wl.plan.describe())
    # e2e overwrote the device outputs only through host buffers: re-run one
    # device step so wl.expect / wl.rows_out hold this configuration's result
    wl.step(1)
    torch.cuda.synchronize()
    res["parity"] = parity_check(spec, wl, oracle_rows_fn() if oracle_rows_fn else None)
    del wl
    torch.cuda.empty_cache()
    return res


def measure_jacobian(spec, rows: int, device: str) -> dict:
    """Jacobian mode (reference run_batch semantics: one adjoint sweep per
    observable, (B, M, cols) output), device-timed; SURVEY §8d asks for it on
    cfg2 / cfg4 next to the VJP headline."""
    import torch

    from paper_2404_06314_b200 import configs, native
    from paper_2404_06314_b200.engine import BatchEngine
    circ, obs, wrt = configs.build(spec, configs.native_api())
    x, w = configs.inputs_and_weights(spec, batch=rows or spec.batch)
    eng = BatchEngine(device=device)
    dev = torch.device(device)
    plan, layout = eng.plans.get(circ, obs, wrt, dev)
    flat = eng.base_flat(circ, {"w": w})
    B, M, C = len(x), len(obs), layout.n_cols
    d_x, d_w = torch.from_numpy(x).to(dev), torch.from_numpy(flat).to(dev)
    e = torch.empty((B, M), dtype=torch.float64, device=dev)
    j = torch.empty((B, M, C), dtype=torch.float64, device=dev)
    ws = torch.empty(plan.workspace_bytes(B, native.VQC_MODE_JACOBIAN), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    plan.adjoint(d_x, d_w, None, e, j, None, None, ws, st)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    t0.record()
    for _ in range(reps):
        plan.adjoint(d_x, d_w, None, e, j, None, None, ws, st)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    peak, _ = fp64_peak()
    flops = configs.flops_per_sample(spec, K=M) * B
    out = {"config": workload_desc(spec).replace("VJP grads", "Jacobians"), "rows": B, "ms_per_call": ms,
           "value": B / (ms * 1e-3), "unit": "samples/s",
           "roofline_frac_fp64": flops / (ms * 1e-3) / 1e12 / peak}
    del ws, j
    torch.cuda.empty_cache()
    return out


def run_dry(args, spec) -> None:
    """--dry-run: the N > 1 plumbing without kernels (gloo): ranks shard the
    rows with split_workload, a host-only step reduces each shard and the
    partial sums are all-reduced once per step; max-over-ranks timing and the
    rank-0 line are the GPU arm's."""
    import torch
    import torch.distributed as dist

    from paper_2404_06314_b200.engine import split_workload
    world, rank, _ = dist_setup()
    if world > 1:
        dist.init_process_group("gloo")
    x, _ = configs_inputs(spec)
    lo, hi = split_workload(spec.batch, world)[rank]
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        part = torch.from_numpy(np.array([x[lo:hi].sum(), float(hi - lo)]))
        if world > 1:
            dist.all_reduce(part)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item()) / max(1, args.steps) * 1e3
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms,
                          "config": config_block(spec, world),
                          "check": {"rows": float(part[1]), "sum": float(part[0]),
                                    "expected_sum": float(x.sum())}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(args, spec):
    import torch
    import torch.distributed as dist

    from paper_2404_06314_b200 import build, configs
    world, rank, local = dist_setup()
    if world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    nccl_dir = None
    if world > 1:
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench: {world} ranks need {world} visible GPUs, "
                             f"found {torch.cuda.device_count()}")
        nccl_dir = nccl_log_setup()
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = f"cuda:{local if world > 1 else 0}"
    torch.cuda.set_device(device)
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    flush = torch.zeros(256 << 20 >> 3, dtype=torch.float64, device=device)
    cpu, oracle_rows = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        def oracle_rows_fn():
            nonlocal cpu, oracle_rows
            cpu, oracle_rows = cpu_baseline(spec, target_s=args.cpu_target_s)
            return oracle_rows
    else:
        oracle_rows_fn = None
    res = measure_gpu(spec, args, rank, world, device, flush, True, args.steps, args.warmup,
                      oracle_rows_fn)
    sweep = []
    if world == 1 and not args.no_sweep:
        for cid in (1, 2, 3, 5):
            s = configs.CONFIGS[cid]
            r = measure_gpu(s, args, rank, world, device, flush, False, 3, 2)
            sweep.append({"config": workload_desc(s), "value": r["value"], "unit": "samples/s",
                          "ms_per_step": r["ms_per_step"],
                          "roofline_frac_fp64": r["roofline"]["frac"],
                          "achieved_tflops": r["roofline"]["achieved"],
                          "parity_max_err": r["parity"]["max_err"],
                          "kernels": r["kernels"], "plan": r["plan"]})
    if world == 1 and not args.no_sweep:
        # the optional complex64 mode (north star: 1e-5), same workloads
        for cid in (3, 4, 5):
            s = configs.CONFIGS[cid]
            r = measure_gpu(s, args, rank, world, device, flush, False, 3, 2, precision="complex64")
            sweep.append({"config": workload_desc(s).replace("complex128", "complex64"),
                          "precision": "complex64", "value": r["value"], "unit": "samples/s",
                          "ms_per_step": r["ms_per_step"],
                          "roofline_frac_fp32": r["roofline"]["frac"],
                          "achieved_tflops": r["roofline"]["achieved"],
                          "parity_max_err": r["parity"]["max_err"], "parity_tol": r["parity"]["tol"],
                          "kernels": r["kernels"], "plan": r["plan"]})
    jac = []
    if world == 1 and not args.no_sweep:
        for cid, rows in ((2, 0), (4, 2048)):
            jac.append(measure_jacobian(configs.CONFIGS[cid], rows, device))
    line = None
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded: x ~ U(-pi,pi) (B,n), weights ~ U(0,2pi); BASELINE cfg4)",
            "config": config_block(spec, world),
            "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
            "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
            "parity": res["parity"], "parity_max_err": res["parity"]["max_err"],
            "kernels": res["kernels"], "plan": res["plan"],
        }
        if world > 1:
            line["nccl"] = nccl_summary(nccl_dir)
        if sweep:
            line["sweep"] = sweep
        if jac:
            line["jacobian_mode"] = jac
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=HEADLINE_CFG)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-target-s", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="host-only N-rank plumbing check on gloo (no kernels)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    from paper_2404_06314_b200 import configs
    spec = configs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, spec)
    elif args.dry_run:
        run_dry(args, spec)
    else:
        run_ours(args, spec)


if __name__ == "__main__":
    main()
