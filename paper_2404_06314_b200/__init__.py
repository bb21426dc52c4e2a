"""B200-native batched statevector forward + adjoint gradients.

Drop-in for the hot path of the reference package ``vqckit`` (arXiv
2404.06314, Qiskit-Torch-Module ideas): circuits lower to a flat gate list
(``ir``), libvqc.so runs them on sm_100a (``native``), ``BatchEngine`` /
``QuantumModule`` keep the reference's API.
"""

from .ir import (MAX_QUBITS, AngleExpression, Circuit, CompiledCircuit, Gate, GateKind,
                 ParameterSet, build_reuploading_ansatz, circuit_from_dict, circuit_to_dict,
                 evaluate_expression, load_circuit, save_circuit, validate_binding)
from .observables import Observable, ObservablePack, parse_observable, pauli_masks, z_observable
from .engine import (BatchEngine, BatchInputError, BatchRequest, BatchResult, WrtLayout,
                     default_engine, mix_seed, run_batch, split_workload)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so the IR is importable without CUDA
    if name in ("QuantumModule", "QuantumFunction", "HybridModule", "Uniform", "Constant", "Normal"):
        from . import module
        return getattr(module, name)
    raise AttributeError(name)
