"""Generate golden fixtures by running the REFERENCE implementation (vqckit).

Run here (the reference is mounted read-only at /root/reference):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz. Reference caches are redirected to /tmp so
nothing is written into the reference tree. The reference has no CZ gate, so
CZ(c,t) is spelled H(t) CNOT(c,t) H(t). Only tests read these
files; the GPU box never imports the reference.
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vqc_numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import numpy as np  # noqa: E402
import vqckit  # noqa: E402
from vqckit import (AngleExpression, BatchEngine, BatchRequest, Circuit, Gate,  # noqa: E402
                    GateKind, Observable, ParameterSet, adjoint_gradients, evolve)

from paper_2404_06314_b200 import configs  # noqa: E402

# SURVEY §8(c) parity protocol: full batch for cfg1-3 comes from the oracle
# (pinned to these rows); cfg4 the first 64 rows, cfg5 the first 8
ROWS = {1: 32, 2: 64, 3: 32, 4: 64, 5: 8}
THREADS = 8


def ref_api():
    from types import SimpleNamespace
    return SimpleNamespace(GateKind=GateKind, Gate=Gate, AngleExpression=AngleExpression,
                           ParameterSet=ParameterSet, Circuit=Circuit, Observable=Observable)


def compiled_arrays(circuit):
    c = circuit.compiled()
    return dict(kinds=c.kinds, q0=c.q0, q1=c.q1, gen_axis=c.gen_axis, coeff=c.coeff,
                f_offs=c.f_offs, f_idx=c.f_idx)


def golden_config(cfg_id: int, engine: BatchEngine) -> None:
    spec = configs.CONFIGS[cfg_id]
    circuit, observables, wrt = configs.build(spec, ref_api(), cz_decompose=True)
    x, w = configs.inputs_and_weights(spec)
    rows = ROWS[cfg_id]
    xs = x[:rows]
    t0 = time.time()
    fwd = engine.run_batch(BatchRequest(circuit, observables, {"w": w}, xs, wrt=()))
    res = engine.run_batch(BatchRequest(circuit, observables, {"w": w}, xs, wrt=wrt))
    dt = time.time() - t0
    up = np.ones((rows, len(observables)))
    out = dict(x_rows=xs, w=w, expect_fwd=fwd.expectations, expect=res.expectations,
               jac_w=res.gradients["w"], vjp_w=np.einsum("bm,bmp->p", up, res.gradients["w"]),
               x_checksum=np.array([x.sum(), (x * x).sum()]), batch=np.array(spec.batch),
               **{"ref_" + k: v for k, v in compiled_arrays(circuit).items()})
    if "x" in res.gradients:
        out["jac_x"] = res.gradients["x"]
        out["vjp_x_rows"] = np.einsum("bm,bmf->bf", up, res.gradients["x"])
    if len(observables) > 1:
        # the reference's VJP-equivalent call: one combined
        # observable sum_m u_m O_m (observables.py:21-47), u = ones
        combined = Observable(tuple(t for o in observables for t in o.terms))
        comb = engine.run_batch(BatchRequest(circuit, [combined], {"w": w}, xs, wrt=wrt))
        out["comb_expect"] = comb.expectations
        out["comb_vjp_w"] = comb.gradients["w"].sum(axis=(0, 1))
        if "x" in comb.gradients:
            out["comb_vjp_x_rows"] = comb.gradients["x"][:, 0, :]
    np.savez_compressed(os.path.join(HERE, f"cfg{cfg_id}.npz"), **out)
    print(f"cfg{cfg_id}: {rows} rows in {dt:.1f}s", flush=True)


def random_case(rng, n: int, n_gates: int, general_obs: bool):
    """Random circuit over RX RY RZ CNOT H X with 0-2 factor expressions that
    share parameters across gates (own generator; same coverage goals as the
    reference's conftest: every gate kind, shared references, encoding set)."""
    sets = (ParameterSet("s", 3, "encoding"), ParameterSet("theta", 4, "trainable"),
            ParameterSet("lam", 2, "trainable"))
    kinds = [GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.CNOT, GateKind.H, GateKind.X]
    pool = [(s.name, i) for s in sets for i in range(s.size)]
    gates = []
    for _ in range(n_gates):
        kind = kinds[int(rng.integers(len(kinds)))]
        if kind == GateKind.CNOT and n < 2:
            kind = GateKind.X
        if kind == GateKind.CNOT:
            a, b = rng.permutation(n)[:2]
            gates.append(Gate(kind, (int(a), int(b))))
            continue
        q = int(rng.integers(n))
        if kind in (GateKind.RX, GateKind.RY, GateKind.RZ):
            nf = int(rng.integers(0, 3))
            picks = []
            for _ in range(nf):
                ref = pool[int(rng.integers(len(pool)))]
                if ref not in picks:
                    picks.append(ref)
            gates.append(Gate(kind, (q,), AngleExpression(float(rng.uniform(-2, 2)), tuple(picks))))
        else:
            gates.append(Gate(kind, (q,)))
    circuit = Circuit(n, tuple(gates), sets)
    letters = "IXYZ" if general_obs else "IZ"
    observables = []
    for _ in range(int(rng.integers(1, 4))):
        terms = []
        for _ in range(int(rng.integers(1, 4))):
            s = "".join(letters[int(rng.integers(len(letters)))] for _ in range(n))
            terms.append((float(rng.uniform(-2, 2)), s))
        observables.append(Observable(tuple(terms)))
    values = {s.name: rng.uniform(-1.5, 1.5, s.size) for s in sets}
    return circuit, observables, values


def golden_random(engine: BatchEngine) -> None:
    rng = np.random.default_rng(20261020)
    cases = {}
    idx = 0
    for general in (False, True):
        for n in (1, 2, 3, 4, 5, 6, 7, 9):
            for rep in range(3):
                circuit, observables, values = random_case(rng, n, int(rng.integers(1, 40)), general)
                B = int(rng.integers(1, 6))
                inputs = rng.uniform(-1.5, 1.5, (B, 3))
                trainable = {k: v for k, v in values.items() if k != "s"}
                res = engine.run_batch(BatchRequest(circuit, observables, trainable, inputs,
                                                    wrt=("theta", "lam", "s")))
                fwd = engine.run_batch(BatchRequest(circuit, observables, trainable, inputs))
                binding = dict(values)
                binding["s"] = inputs[0]
                state = evolve(circuit, binding)
                single = adjoint_gradients(circuit, binding, observables, ["lam", "theta"])
                ca = compiled_arrays(circuit)
                obs_pack = vqckit.observables.ObservablePack.from_observables(observables, n)
                pre = f"c{idx}_"
                cases.update({pre + k: v for k, v in ca.items()})
                cases.update({
                    pre + "n": np.array(n), pre + "general": np.array(general),
                    pre + "term_offs": obs_pack.term_offs, pre + "t_coeffs": obs_pack.coeffs,
                    pre + "t_xmask": obs_pack.x_masks, pre + "t_smask": obs_pack.sign_masks,
                    pre + "t_phases": np.stack([obs_pack.phases.real, obs_pack.phases.imag], -1),
                    pre + "theta": values["theta"], pre + "lam": values["lam"], pre + "s0": values["s"],
                    pre + "inputs": inputs, pre + "expect": res.expectations,
                    pre + "expect_fwd": fwd.expectations,
                    pre + "jac_theta": res.gradients["theta"], pre + "jac_lam": res.gradients["lam"],
                    pre + "jac_s": res.gradients["s"], pre + "state0": state,
                    pre + "single_expect": single.expectations,
                    pre + "single_lam": single.gradients["lam"],
                    pre + "single_theta": single.gradients["theta"],
                })
                # serialise the circuit itself for the product-side compiler test
                cases[pre + "doc"] = np.array(repr(vqckit.circuit_to_dict(circuit)))
                cases[pre + "obs"] = np.array(repr([o.terms for o in observables]))
                idx += 1
    cases["count"] = np.array(idx)
    np.savez_compressed(os.path.join(HERE, "random.npz"), **cases)
    print(f"random: {idx} cases", flush=True)


METHOD_ROWS = {1: 16, 2: 8}
SPSA = dict(seed=5, spsa_c=0.01, spsa_samples=3)


def golden_methods(engine: BatchEngine) -> None:
    """param-shift and SPSA through the reference's run_batch (batch.py:193-201)
    on the first rows of cfg1 / cfg2 (wrt = (w, x))."""
    out = {}
    for cfg_id, rows in METHOD_ROWS.items():
        spec = configs.CONFIGS[cfg_id]
        circuit, observables, wrt = configs.build(spec, ref_api(), cz_decompose=True)
        x, w = configs.inputs_and_weights(spec)
        xs = x[:rows]
        ps = engine.run_batch(BatchRequest(circuit, observables, {"w": w}, xs,
                                           method="param-shift", wrt=wrt))
        sp = engine.run_batch(BatchRequest(circuit, observables, {"w": w}, xs,
                                           method="spsa", wrt=wrt, **SPSA))
        for name, res in (("ps", ps), ("spsa", sp)):
            out[f"cfg{cfg_id}_{name}_expect"] = res.expectations
            for k, v in res.gradients.items():
                out[f"cfg{cfg_id}_{name}_jac_{k}"] = v
        out[f"cfg{cfg_id}_rows"] = np.array(rows)
    out["spsa_seed"], out["spsa_c"], out["spsa_samples"] = (
        np.array(SPSA["seed"]), np.array(SPSA["spsa_c"]), np.array(SPSA["spsa_samples"]))
    np.savez_compressed(os.path.join(HERE, "methods.npz"), **out)
    print("methods: done", flush=True)


def golden_training() -> None:
    """The reference's train_classifier (training.py:59-94) with Adam on a
    4-qubit re-uploading classifier over a seeded synthetic dataset."""
    from vqckit.datasets import Dataset
    from vqckit.model import Constant, QuantumModule, Uniform
    from vqckit.optim import Adam
    from vqckit.training import train_classifier
    rng = np.random.default_rng(2024)
    feats = rng.uniform(-1.0, 1.0, (40, 4))
    labels = (feats[:, 0] * feats[:, 1] > 0).astype(np.int64)
    ds = Dataset(feats, labels, np.arange(32), np.arange(32, 40), 2)
    circuit = vqckit.build_reuploading_ansatz(4, 2, num_features=4)
    obs = [Observable(((2.0, "ZIII"),)), Observable(((2.0, "IZII"),))]
    mod = QuantumModule(circuit, obs, "s", [("theta", Uniform()), ("lambda", Constant(1.0))],
                        seed=11, threads=1)
    opt = Adam(lr=0.05, per_set={"lambda": 0.01})
    recs = train_classifier(ds, mod, epochs=3, batch_size=8, optimizer=opt, seed=3)
    np.savez_compressed(os.path.join(HERE, "training.npz"), features=feats, labels=labels,
                        loss=np.array([r.loss for r in recs]),
                        metric=np.array([r.metric for r in recs]),
                        theta=mod.parameters()["theta"], lam=mod.parameters()["lambda"])
    print("training: done", flush=True)


def main(which=None):
    if which == "training":
        golden_training()
        return
    engine = BatchEngine(threads=THREADS)
    if which in (None, "random"):
        golden_random(engine)
    if which in (None, "methods"):
        golden_methods(engine)
    for cfg_id in (1, 2, 3, 4, 5):
        if which in (None, f"cfg{cfg_id}"):
            golden_config(cfg_id, engine)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
