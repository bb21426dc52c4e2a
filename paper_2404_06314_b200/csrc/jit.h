// Per-plan specialisation: the device program of a plan (scheduler.cpp) is
// emitted as straight-line CUDA (every op a call with compile-time slots,
// kinds and table offsets — kernels.cuh jop_*), compiled for sm_100a with
// NVRTC at plan creation and loaded through the driver API. The interpreter
// kernels in engine.cu run the same ops with run-time decoding; both paths
// share the skeleton (skeleton.cuh) and the arithmetic.
#pragma once
#include <cuda.h>

#include <string>
#include <vector>

#include "scheduler.h"

namespace vqc {

struct JitKernels {
  CUfunction smem_fwd = nullptr, smem_adj = nullptr;  // n <= 12
  std::vector<CUfunction> pass_fwd, pass_adj;         // per HBM pass
  double compile_s = 0.0;
  size_t cubin_bytes = 0;
  bool cached = false;
};

// CUDA source of a plan's kernels (split: the on-chip adjoint runs on
// (psi, phi) thread pairs).
std::string jit_source(const HostProgram& P, bool split);

// NVRTC-compile a plan's units without loading them (CPU-side checks). Returns "".
std::string jit_compile_only(const HostProgram& P, bool split, double* seconds);

// Generate, compile (NVRTC, sm_100a) and load. Returns "" on success.
std::string jit_build(const HostProgram& P, bool split, JitKernels* out);

// Driver-API launch of a JIT kernel with (DevProgram, RunArgs) arguments.
struct DevProgram;
struct RunArgs;
CUresult jit_launch(CUfunction f, unsigned gx, unsigned gy, unsigned bx, size_t smem, CUstream st,
                    const DevProgram& D, const RunArgs& A);

}  // namespace vqc
