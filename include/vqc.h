/*
 * vqc.h — C ABI of the B200-native batched statevector engine (libvqc.so).
 *
 * Drop-in boundary for the reference's batched adjoint path
 * (vqckit, /root/reference/pkg/src/vqckit):
 *
 *   reference interface                                  replaced by
 *   ---------------------------------------------------  -------------------------
 *   CompiledCircuit.from_circuit arrays (circuit.py:168-216)  VqcCircuit
 *   ObservablePack.from_observables (observables.py:132-167)  VqcObservables
 *   WrtLayout.build -> wrt_col (gradients.py:58-77)           vqc_plan_create(wrt_col)
 *   BatchEngine.run_batch, wrt=() (batch.py:147-217, 475-477) vqc_forward
 *   BatchEngine.run_batch, method="adjoint" (batch.py:478-480,
 *     gradients.py:104-118, _kernels.py:241-281)              vqc_adjoint (jac != NULL)
 *   QuantumModule.backward einsum("bm,bmp->p") (model.py:651-662)
 *     and engine_server.py:125-138 input VJP                 vqc_adjoint (upstream != NULL)
 *   numpy-in/numpy-out call of the whole batch                vqc_run_batch_host
 *
 * Conventions (statevector.py:1-11, _kernels.py:16-27): gate codes RX=0 RY=1
 * RZ=2 CNOT=3 H=4 X=5, plus CZ=6 (new); U(theta)=exp(-i theta P/2); qubit 0 is
 * the least-significant index bit; angle_g = coeff_g * prod flat[f_idx].
 * All numeric buffers are float64 (complex128 states live only in the
 * caller-provided workspace). Device pointers (d_*) are CUDA global memory on
 * the plan's device; host pointers (h_*) are ordinary host memory.
 *
 * Errors: every entry point returns 0 on success or a negative VQC_E* code;
 * vqc_last_error() returns a thread-local message. No exception crosses the
 * ABI. Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default stream) except vqc_run_batch_host, which synchronises.
 */
#ifndef VQC_H_
#define VQC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQC_ABI_VERSION 1

enum {
  VQC_OK = 0,
  VQC_E_INVALID = -1,     /* bad argument (shape, range, null pointer)        */
  VQC_E_UNSUPPORTED = -2, /* valid for the reference but not on this path     */
  VQC_E_CUDA = -3,        /* CUDA runtime error                                */
  VQC_E_WORKSPACE = -4,   /* workspace too small                               */
  VQC_E_NOMEM = -5        /* host / device allocation failed                   */
};

enum { VQC_GATE_RX = 0, VQC_GATE_RY = 1, VQC_GATE_RZ = 2, VQC_GATE_CNOT = 3,
       VQC_GATE_H = 4, VQC_GATE_X = 5, VQC_GATE_CZ = 6 };

/* circuit.py:168-216 (CompiledCircuit) plus the encoding slot of
 * batch.py:440-458. f_offs has n_gates+1 entries (CSR into f_idx). */
typedef struct {
  int32_t n_qubits;          /* 1..24 (statevector.py:21) */
  int64_t n_gates;
  const int64_t* kinds;
  const int64_t* q0;         /* target (rotations/H/X), control (CNOT), first qubit (CZ) */
  const int64_t* q1;         /* CNOT target / CZ second qubit, else ignored */
  const double* coeff;       /* per gate; ignored for non-rotations */
  const int64_t* f_offs;
  const int64_t* f_idx;      /* flat parameter indices, <= 4 per gate */
  int64_t total_params;
  int64_t enc_offset;        /* flat offset of the one encoding set (batch.py:400-405) */
  int64_t enc_size;
} VqcCircuit;

/* observables.py:132-167 (ObservablePack): M observables, T terms total;
 * phases are (T, 2) re/im of i^{#Y}. Z strings (x_mask == 0) run on every
 * path; X/Y strings on the on-chip path (n <= 12) — vqc_plan_create returns
 * VQC_E_UNSUPPORTED for them when n > 12. */
typedef struct {
  int64_t n_obs;
  const int64_t* term_offs;  /* n_obs + 1 */
  const double* coeffs;
  const int64_t* x_masks;
  const int64_t* sign_masks;
  const double* phases;
} VqcObservables;

typedef struct VqcPlan VqcPlan;

/* Lower the circuit to the device program: validates like circuit.py:73-101,
 * builds the rotation/angle tables, the WrtLayout chain-rule table
 * (gradients.py:58-77, _kernels.py:269-278) and the pass/segment schedule,
 * and uploads them to the current device. wrt_col has total_params entries,
 * each an output column or -1. precision: 0 = complex128 states, 1 = complex64
 * states (JIT kernels; angles, block matrices, reductions and all outputs stay
 * float64; parity target 1e-5 against the complex128 reference). */
int vqc_plan_create(const VqcCircuit* circuit, const VqcObservables* obs, const int64_t* wrt_col,
                    int precision, VqcPlan** out);
void vqc_plan_destroy(VqcPlan* plan);

/* Introspection for hosts and tests. */
int64_t vqc_plan_num_cols(const VqcPlan* plan);     /* output columns (WrtLayout.n_cols) */
int64_t vqc_plan_num_obs(const VqcPlan* plan);
int vqc_plan_mode(const VqcPlan* plan);             /* 0 = on-chip (smem) state, 1 = HBM passes */
/* Writes a short JSON description (schedule stats) into buf; returns needed length. */
int64_t vqc_plan_describe(const VqcPlan* plan, char* buf, int64_t cap);

enum { VQC_MODE_FORWARD = 0, VQC_MODE_VJP = 1, VQC_MODE_JACOBIAN = 2 };
/* Bytes of device workspace a call with batch B in the given mode needs. */
size_t vqc_workspace_bytes(const VqcPlan* plan, int64_t B, int mode);

/* Forward: d_expect (B, M) = <psi_b|O_m|psi_b> (batch.py:475-477).
 * d_inputs (B, enc_size); d_weights = the flat parameter vector
 * (total_params; its encoding slice is ignored). */
int vqc_forward(VqcPlan* plan, const double* d_inputs, const double* d_weights, int64_t B,
                double* d_expect, void* d_workspace, size_t workspace_bytes, void* stream);

/* Forward + adjoint backward in one call (the reference's
 * run_batch(method="adjoint") includes its own forward).
 *  - Jacobian mode: d_upstream == NULL; d_jac (B, M, n_cols) receives
 *    d<O_m>/dp like batch.py:463-505 (before the per-set split).
 *  - VJP mode: d_upstream (B, M); d_vjp_rows (B, n_cols) receives
 *    sum_m u[b,m] J[b,m,:] per row (engine_server.py:135-136) and
 *    d_vjp_sum (n_cols) the batch sum (model.py:661), each optional (NULL).
 * d_expect (B, M) is optional. */
int vqc_adjoint(VqcPlan* plan, const double* d_inputs, const double* d_weights, int64_t B,
                const double* d_upstream, double* d_expect, double* d_jac, double* d_vjp_rows,
                double* d_vjp_sum, void* d_workspace, size_t workspace_bytes, void* stream);

/* Host-buffer drop-in for BatchEngine.run_batch (batch.py:147-217): copies
 * inputs H2D, runs forward / adjoint on the plan's device with a plan-owned
 * workspace, copies results D2H and synchronises. Same output conventions as
 * vqc_adjoint; with h_upstream == NULL and h_jac == NULL it is forward-only. */
int vqc_run_batch_host(VqcPlan* plan, const double* h_inputs, const double* h_weights, int64_t B,
                       const double* h_upstream, double* h_expect, double* h_jac,
                       double* h_vjp_rows, double* h_vjp_sum);

/* Number of kernels the last call on this thread launched (for bench claims). */
/* Per-plan kernel specialisation (no reference counterpart: the reference's
 * numba kernels are compiled once per gate kind, _kernels.py:32-141). The
 * CUDA source that vqc_plan_create compiles with NVRTC for this circuit;
 * with compile != 0 it is also compiled for sm_100a (no GPU needed) and the
 * compile time stored in *compile_s. Returns the source length or < 0. */
int64_t vqc_jit_source(const VqcCircuit* circuit, const int64_t* wrt_col, int compile, char* buf, int64_t cap,
                       double* compile_s);

int64_t vqc_last_launch_count(void);

/* SPSA direction draws for rows row0 .. row0 + rows - 1 of a batch (host
 * arithmetic, no GPU): out (rows, samples, cols) receives +1 / -1, bit for
 * bit the reference's 2 * rng.integers(0, 2, size=cols) - 1 per sample
 * (gradients.py:180-201) with rng = numpy default_rng(mix_seed(seed, row))
 * per row (batch.py:75-81, 197); per_row_seed == 0 draws every row from
 * default_rng(seed) itself, the single-binding form (gradients.py:243-266). */
int vqc_spsa_signs(uint64_t seed, int64_t row0, int64_t rows, int64_t samples, int64_t cols,
                   int per_row_seed, int8_t* out);

/* Per-kernel CUDA-event timing of this thread's launches (bench/profiling):
 * enable resets the totals; report synchronises pending events and writes
 * {"kernel": [total_ms, launches], ...} into buf, returning the JSON length. */
void vqc_profile_enable(int on);
int64_t vqc_profile_report(char* buf, int64_t cap);

const char* vqc_last_error(void);
int vqc_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VQC_H_ */
