"""Per-plan specialisation (csrc/jit.cpp), checked on the CPU: the generated
source covers every op of the scheduled program and compiles for sm_100a
with NVRTC (no GPU needed). Numerics of the JIT kernels are the -m gpu parity
tests (HBM plans run JIT kernels by default)."""

import numpy as np
import pytest

from paper_2404_06314_b200 import configs, native
from paper_2404_06314_b200.engine import WrtLayout, encoding_set


def _src(circ, wrt, compile=False):
    compiled = circ.compiled()
    layout = WrtLayout.build(compiled, wrt)
    off, size = compiled.offsets[encoding_set(circ).name]
    return native.jit_source(compiled, layout.wrt_col, off, size, compile=compile)


def test_hbm_plan_has_one_kernel_pair_per_pass():
    spec = configs.CONFIGS[4]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    src, _ = _src(circ, wrt)
    n_pf = src.count("void __launch_bounds__") // 2
    assert n_pf >= 10 and src.count("vqc_jit_pf") == n_pf and src.count("vqc_jit_pa") == n_pf
    # every fused set of cfg4 is emitted with compile-time slots
    # adjoint schedule: 3 register slots, both states per thread
    # gradient partials per thread, reduced per warp; thread-group barriers
    assert "jop_u2<R, MODE_FWD, 0, true>(f, f, T, " in src and "jop_ip3w_set<R, 7>(a, f, pr + 0);" in src
    assert "wr_split<9, 4>(q0_v, wl_, " in src and "seg_end_g<R, MODE>" in src and "wred_outputs(E, jb0_out" in src
    assert "vqc::KM_DUAL" in src
    assert "exec_op" not in src


@pytest.mark.parametrize("fold", ["0", "1"])
def test_random_hbm_circuit_compiles_for_sm100a(monkeypatch, fold):
    """Every gate kind (and so every op the scheduler emits) through NVRTC;
    with thread-target CNOT folds (default) boundary CNOTs become address
    maps (tile_ld / thread bases), without them some run in registers."""
    monkeypatch.setenv("VQC_JIT_CACHE", "0")  # really compile (no cubin cache)
    monkeypatch.setenv("VQC_FOLD_THREAD_TARGETS", fold)
    from test_scheduler_sim import _random
    rng = np.random.default_rng(7)
    circ, _, _ = _random(rng, 13, 60)
    src, secs = _src(circ, ("a", "b", "s"), compile=True)
    assert secs is not None and secs > 0
    for op in (("jop_cnot",) if fold == "0" else ()) + ("jop_u2", "jop_ip"):
        assert op in src, op
    if fold == "1":
        assert "__popc(tb & " in src     # a fold controlled by a tile bit


def test_on_chip_plan_shares_code_per_segment_shape(monkeypatch):
    """cfg3 kept on chip (VQC_SMEM_MAX_QUBITS=12; by default 11- and 12-qubit
    plans run the pass kernels on one whole-state tile): 48 segments of two
    shapes -> one switch case per shape and unit, compiled in seconds
    (minutes as one copy per segment)."""
    monkeypatch.setenv("VQC_JIT_CACHE", "0")
    monkeypatch.setenv("VQC_SMEM_MAX_QUBITS", "12")
    spec = configs.CONFIGS[3]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    src, secs = _src(circ, wrt, compile=True)
    # forward-only unit (1 shape) + forward/adjoint unit (1 + 2 shapes: the
    # adjoint segments of the first layer keep only their inner products)
    assert src.count("case 0:") == 3 and src.count("case 1:") == 1 and "case 2:" not in src
    assert "__constant__ int sab0_opnd" in src and "vqc_jit_sa" in src and "vqc_jit_sf" in src
    assert secs < 120


def test_whole_state_tile_plan_for_12_qubits(monkeypatch):
    """cfg3 by default: one pass whose tile is the whole 12-qubit state, pass
    kernels with thread-group barriers and per-warp reductions."""
    spec = configs.CONFIGS[3]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    src, _ = _src(circ, wrt)
    assert src.count("vqc_jit_pa") == 1 and "vqc_jit_sa" not in src
    assert "__launch_bounds__(512, 1) vqc_jit_pa0" in src and "seg_end_g<R, MODE>" in src and "wr_split<" in src


def test_constant_observable_terms_compile(monkeypatch):
    """Z-string observables as compile-time constants of the observing pass
    (skeleton.cuh observe<..., TMS>): the unrolled expectation / seed loops
    compile for sm_100a."""
    monkeypatch.setenv("VQC_JIT_CACHE", "0")
    monkeypatch.setenv("VQC_JIT_SOURCE_TERMS", "1")
    from test_scheduler_sim import _random
    circ, _, _ = _random(np.random.default_rng(11), 13, 40)
    src, secs = _src(circ, ("a", "b", "s"), compile=True)
    assert secs is not None and "static constexpr bool kConst = true" in src and "using Terms = TM" in src


def test_cubin_cache_round_trip(tmp_path, monkeypatch):
    """The on-disk cubin cache returns what NVRTC produced (second call reads)."""
    monkeypatch.setenv("VQC_JIT_CACHE", str(tmp_path))
    from test_scheduler_sim import _random
    circ, _, _ = _random(np.random.default_rng(3), 13, 30)
    _, t1 = _src(circ, ("a", "b", "s"), compile=True)
    n_files = len(list(tmp_path.glob("*.cubin")))
    _, t2 = _src(circ, ("a", "b", "s"), compile=True)
    assert n_files >= 1 and len(list(tmp_path.glob("*.cubin"))) == n_files
    assert t2 < t1


def test_unusable_cache_dir_still_compiles(tmp_path, monkeypatch):
    """A cache path that cannot be a directory only costs the cache."""
    blocker = tmp_path / "not_a_dir"
    blocker.write_text("x")
    monkeypatch.setenv("VQC_JIT_CACHE", str(blocker / "sub"))
    from test_scheduler_sim import _random
    circ, _, _ = _random(np.random.default_rng(5), 13, 20)
    src, secs = _src(circ, ("a", "b", "s"), compile=True)
    assert secs is not None and "vqc_jit_pa0" in src


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_complex64_units_compile_for_sm100a(monkeypatch, cfg_id):
    """complex64 plans (precision 1) compile their JIT units with VQC_C64:
    on-chip (cfg2) and HBM passes (cfg4), 8-byte state elements."""
    monkeypatch.setenv("VQC_JIT_CACHE", "0")
    monkeypatch.setenv("VQC_JIT_SOURCE_PRECISION", "1")
    spec = configs.CONFIGS[cfg_id]
    circ, obs, wrt = configs.build(spec, configs.native_api())
    src, secs = _src(circ, wrt, compile=True)
    assert src.count("#define VQC_C64 1") >= 1 and secs is not None
