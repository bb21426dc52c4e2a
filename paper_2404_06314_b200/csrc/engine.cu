// libvqc.so: kernels, launch orchestration and the C ABI declared in
// include/vqc.h. See kernels.cuh for the execution model and DESIGN.md for the
// roofline accounting.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vqc.h"
#include "jit.h"
#include "scheduler.h"
#include "skeleton.cuh"

namespace vqc {

// Interpreter kernels: the device program decoded at run time (InterpSegs).
// Plans normally run JIT-specialised kernels (jit.cpp); these serve
// VQC_JIT=0 and the interpreter parity tests.
template <int R, int KM>
__global__ void __launch_bounds__(smem_max_threads(R, KM)) k_smem(DevProgram D, RunArgs A) {
  smem_body<R, KM, InterpSegs>(D, A);
}
template <int R, int KM>
__global__ void __launch_bounds__(pass_max_threads(R), 1) k_pass(DevProgram D, RunArgs A) {
  pass_body<R, KM, InterpSegs>(D, A);
}

// Per-sample angle / fused-block tables for every pass, once per call (HBM
// mode): [cos/sin per rotation][U per block][gradient vector per member].
__global__ void __launch_bounds__(256) k_tables(DevProgram D, RunArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t bl = blockIdx.x;
  const int64_t b = A.b0 + bl;
  PassDesc all{};
  all.rot_begin = 0;
  all.rot_end = D.n_rot;
  all.blk_begin = 0;
  all.blk_end = D.n_blk;
  all.av_begin = 0;
  all.av_end = D.n_av;
  double2* cs = reinterpret_cast<double2*>(smem_raw);
  double2* u = cs + D.n_rot;
  double* av = reinterpret_cast<double*>(u + 4 * (size_t)D.n_blk);
  build_tables(D, A, &all, b, true, cs, u, av, threadIdx.x, blockDim.x);
  const double* src = reinterpret_cast<const double*>(smem_raw);
  double* dst = const_cast<double*>(A.tables) + (size_t)bl * A.table_stride;
  for (int64_t i = threadIdx.x; i < A.table_stride; i += blockDim.x) dst[i] = src[i];
}

// out[i] = sum_t in[i * n_tiles + t], fixed order (one warp per output)
__global__ void k_tile_reduce(const double* __restrict__ in, double* __restrict__ out, int64_t count,
                              int n_tiles) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  double v = 0.0;
  for (int t = lane; t < n_tiles; t += 32) v += in[w * n_tiles + t];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) out[w] = v;
}

// chain rule (_kernels.py:269-278): out[b,k,col] = sum_e ip[b,k,gslot_e] * dangle/dp
__global__ void k_chain(DevProgram D, RunArgs A, const double* __restrict__ ip, int64_t nb, int K,
                        const int32_t* __restrict__ col_offs, const ChainEntry* __restrict__ chain,
                        int ncols, double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nb * K * ncols) return;
  const int col = (int)(idx % ncols);
  const int64_t bk = idx / ncols;
  const int64_t b = A.b0 + bk / K;
  double acc = 0.0;
  for (int e = col_offs[col]; e < col_offs[col + 1]; ++e) {
    const ChainEntry ce = chain[e];
    double partial = ce.coeff;
    for (int u = 0; u < ce.nother; ++u) partial *= flat_val(D, A, b, ce.other[u]);
    acc += ip[bk * D.NG + ce.gslot] * partial;
  }
  out[idx] = acc;
}

// out[col] = sum_b rows[b, col] in fixed order (model.py:661 einsum over rows)
__global__ void k_batch_sum(const double* __restrict__ rows, int64_t nb, int ncols,
                            double* __restrict__ out) {
  __shared__ double part[32][33];
  const int col = blockIdx.x * 32 + threadIdx.x;
  double v0 = 0.0, v1 = 0.0;  // 32 row slices per column, two chains each
  if (col < ncols) {
    int64_t b = threadIdx.y;
    for (; b + 32 < nb; b += 64) {
      v0 += rows[b * ncols + col];
      v1 += rows[(b + 32) * ncols + col];
    }
    if (b < nb) v0 += rows[b * ncols + col];
  }
  part[threadIdx.y][threadIdx.x] = v0 + v1;
  __syncthreads();
  if (threadIdx.y == 0 && col < ncols) {
    double s = 0.0;
    for (int w = 0; w < 32; ++w) s += part[w][threadIdx.x];
    out[col] = s;
  }
}

using KFn = void (*)(DevProgram, RunArgs);

// small registers sets (n < 9) keep both states per thread; larger tiles
// split the adjoint over (psi, phi) thread pairs
bool use_split(int n, int R) { return (n - R) >= 5; }

// JIT-compiled HBM plans: the adjoint sweep runs 3 register slots with both
// states per thread (KM_DUAL: no partner reads, one barrier less per
// segment), the forward sweep its own 4-slot schedule (measured on cfg4:
// adjoint 630 -> 559 ms, forward 191 ms kept; r01 knob sweep in DESIGN.md)
constexpr int kHbmAdjointRegs = 3;
// on-chip plans up to this size take their per-sample tables from k_tables
// (few threads per sample would build them through serial global loads)
constexpr int kSmemTablesMaxN = 10;
constexpr int kHbmForwardRegs = 4;
// complex64 HBM plans: 4 slots, both states per thread (float2 states need
// half the registers), 12-qubit tiles; one program for both sweeps
// (measured on cfg4: 36.4k -> 38.9k samples/s, profiles/r02/knobs_c8_complex64.log)
constexpr int kHbmTileC64 = 12;
constexpr int kHbmRegsC64 = 4;
// on-chip JIT plans this small run 3 register slots with both states per
// thread (measured: cfg2 158 -> 98 us, cfg1 52 -> 31 us per call); n = 11, 12
// keep 4 slots on thread pairs (cfg3: 5.95 vs 6.40 ms). VQC_SMEM_DUAL=1 / 0
// forces it on / off for 4 <= n <= 12.
constexpr int kSmemDualMaxN = 10;
// JIT plans from this size up run the pass kernels (schedule_circuit): one
// sample per CTA with 2^(n-3) threads, i.e. at least a full warp per sample.
// Up to kPassFusedMaxQubits the forward sweep shares the adjoint schedule and
// kernel (one launch: cfg2 97 -> 39 us per 1024-row call); above, the forward
// sweep has its own 4-slot schedule.
constexpr int kPassMinQubits = 8;
constexpr int kPassFusedMaxQubits = 10;
bool smem_dual(int n) {
  auto env = [](const char* name) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : -1;
  };
  if (n < 4 || n > kSmemMaxQubits || env("VQC_JIT") == 0) return false;
  const int e = env("VQC_SMEM_DUAL");
  return e < 0 ? n <= kSmemDualMaxN : e != 0;
}

// Plans use R = min(4, n) register slots (schedule_circuit), so only these
// interpreter instantiations exist (each is a large unrolled kernel).
KFn smem_kernel(int R, bool dual, bool split) {
  if (!dual) {
    switch (R) {
      case 1: return k_smem<1, KM_FWD>;
      case 2: return k_smem<2, KM_FWD>;
      case 3: return k_smem<3, KM_FWD>;
      default: return k_smem<4, KM_FWD>;
    }
  }
  if (split) return k_smem<4, KM_SPLIT>;
  switch (R) {
    case 1: return k_smem<1, KM_DUAL>;
    case 2: return k_smem<2, KM_DUAL>;
    case 3: return k_smem<3, KM_DUAL>;
    default: return k_smem<4, KM_DUAL>;
  }
}
KFn pass_kernel(int, bool dual) { return dual ? k_pass<4, KM_SPLIT> : k_pass<4, KM_FWD>; }

// a kernel to launch: prebuilt interpreter (fn) or plan-specialised JIT (cu)
struct Kern {
  KFn fn = nullptr;
  CUfunction cu = nullptr;
};

}  // namespace vqc

// ------------------------------------------------------------------ host side

using namespace vqc;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

// Optional per-kernel CUDA-event timing (vqc_profile_enable / _report): one
// event pair around each launch on the launching stream.
struct ProfPending {
  const char* name;
  cudaEvent_t e0, e1;
};
struct ProfAgg {
  std::string name;
  double ms;
  int64_t count;
};
thread_local bool g_prof = false;
thread_local std::vector<ProfPending> g_prof_pending;
thread_local std::vector<cudaEvent_t> g_prof_pool;
thread_local std::vector<ProfAgg> g_prof_agg;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
    if (g_prof) {
      e0 = prof_event();
      cudaEventRecord(e0, st);
    }
  }
  ~ProfScope() {
    if (e0) {
      cudaEvent_t e1 = prof_event();
      cudaEventRecord(e1, st);
      g_prof_pending.push_back({name, e0, e1});
    }
  }
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(VQC_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr int kMaxSmemBytes = 232448;  // 227 KiB opt-in per CTA on sm_100

template <class T>
cudaError_t upload(const std::vector<T>& v, T** d) {
  *d = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(d), v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

int env_int(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return (s && *s) ? std::atoi(s) : dflt;
}

}  // namespace

// ThrEntry rows of every segment (program.h): for each thread group gi the
// global bits its index contributes, and the swizzled load / store bases
// with the folded CNOT translations controlled by thread bits applied.
static std::vector<ThrEntry> build_thr_table(std::vector<SegDesc>& segs) {
  std::vector<ThrEntry> tab;
  for (SegDesc& sd : segs) {
    sd.thr_off = (int32_t)tab.size();
    const int nthr = sd.nthr;
    for (uint32_t gi = 0; gi < (1u << nthr); ++gi) {
      uint32_t j0 = 0, p0 = 0;
      for (int i = 0; i < nthr; ++i)
        if ((gi >> i) & 1u) {
          p0 ^= sd.tsw[i];
          j0 |= 1u << sd.thr_g[i];
        }
      uint32_t lp0 = p0, sp0 = p0;
      for (int t = 0; t < kMaxR; ++t) {
        if (__builtin_popcount(j0 & sd.ld_k[t]) & 1) lp0 ^= sd.ps[t];
        if (__builtin_popcount(j0 & sd.st_k[t]) & 1) sp0 ^= sd.ps[t];
      }
      tab.push_back(ThrEntry{j0, lp0, sp0, 0u});
    }
  }
  return tab;
}

// device copies of one scheduled program's tables
struct ProgTabs {
  Op* ops = nullptr;
  SegDesc* segs = nullptr;
  IpOut* ipouts = nullptr;
  BlockDesc* blocks = nullptr;
  MemberDesc* members = nullptr;
  DiagRun* diag = nullptr;
  int16_t* setids = nullptr;
  ThrEntry* thr_tab = nullptr;
  PassDesc* passes = nullptr;
  RotDesc* rots = nullptr;
  cudaError_t upload_all(std::vector<SegDesc>& segs_h, const HostProgram& P) {
    const std::vector<ThrEntry> thr = build_thr_table(segs_h);
    cudaError_t e = upload(thr, &thr_tab);
    if (e == cudaSuccess) e = upload(P.ops, &ops);
    if (e == cudaSuccess) e = upload(P.segs, &segs);
    if (e == cudaSuccess) e = upload(P.ipouts, &ipouts);
    if (e == cudaSuccess) e = upload(P.blocks, &blocks);
    if (e == cudaSuccess) e = upload(P.members, &members);
    if (e == cudaSuccess) e = upload(P.diag, &diag);
    if (e == cudaSuccess) e = upload(P.setids, &setids);
    if (e == cudaSuccess) e = upload(P.passes, &passes);
    if (e == cudaSuccess) e = upload(P.rots, &rots);
    return e;
  }
  void free_all() {
    cudaFree(ops);
    cudaFree(segs);
    cudaFree(ipouts);
    cudaFree(blocks);
    cudaFree(members);
    cudaFree(diag);
    cudaFree(setids);
    cudaFree(thr_tab);
    cudaFree(passes);
    cudaFree(rots);
    *this = ProgTabs();
  }
};

// a second scheduled program (forward sweep) with its tables and kernels
struct ProgDev {
  HostProgram prog;
  ProgTabs tabs;
  DevProgram D{};
  JitKernels jit;
};

struct VqcPlan {
  int circuit_qubits = 0;  // the circuit's own qubit count (the plan may hold idle qubits, VQC_PAD_QUBITS)
  int device = 0;
  int sms = 148;
  HostProgram prog;
  int64_t total_params = 0, enc_off = 0, enc_size = 0;
  int M = 0;
  std::vector<int32_t> term_offs;
  std::vector<uint32_t> smask, xmask;
  std::vector<int32_t> tphase;
  std::vector<double> tcoeff;
  std::vector<int32_t> tobs;  // observable of each term
  bool has_xy = false;
  // device tables
  ProgTabs tabs;  // device tables of `prog`
  int32_t* d_term_offs = nullptr;
  uint32_t* d_smask = nullptr;
  uint32_t* d_xmask = nullptr;
  int32_t* d_tphase = nullptr;
  double* d_tcoeff = nullptr;
  int32_t* d_tobs = nullptr;
  int32_t* d_col_offs = nullptr;
  ChainEntry* d_chain = nullptr;
  DevProgram D{};
  size_t state_budget = 0;
  bool use_jit = false;
  JitKernels jit;
  // Separate forward schedule for HBM plans (its own tile size / register
  // slots, VQC_FWD_TILE / VQC_FWD_REG); null = `prog` runs forward and adjoint
  ProgDev* fwd = nullptr;
  unsigned* d_check = nullptr;  // VQC_CHECKS: device bounds-check failure bits
  // host-call cache
  std::mutex mu;
  cudaStream_t stream = nullptr;
  void* h_dev = nullptr;
  size_t h_dev_bytes = 0;
};

namespace {

struct Layout {
  size_t ip = 0, rows = 0, psi = 0, phi = 0, fin = 0, ipart = 0, epart = 0, tables = 0, ftables = 0, total = 0;
  int64_t table_stride = 0;   // doubles per sample (0: tables rebuilt per CTA)
  int64_t ftable_stride = 0;  // same for the separate forward program
  int64_t chunk = 0;
  int n_tiles = 1;
  int K = 1;
};

Layout make_layout(const VqcPlan* p, int64_t B, int mode) {
  Layout L;
  const HostProgram& P = p->prog;
  const int64_t N = (int64_t)1 << P.n;
  const int M = p->M;
  L.K = mode == VQC_MODE_JACOBIAN ? std::max(M, 1) : 1;
  const size_t esz = P.precision == 1 ? 8 : 16;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  const bool adj = mode != VQC_MODE_FORWARD;
  L.ip = take(adj ? (size_t)B * L.K * P.NG * sizeof(double) : 0);
  L.rows = take(mode == VQC_MODE_VJP ? (size_t)B * P.n_cols * sizeof(double) : 0);
  if (!P.hbm) {
    L.chunk = B;
    L.fin = take(mode == VQC_MODE_JACOBIAN && M > 1 ? (size_t)B * N * esz : 0);
    // small on-chip states: per-sample tables from k_tables (one CTA per sample,
    // rotations in parallel) instead of a serial dependent-load chain per CTA
    const int64_t st = 2 * (int64_t)P.n_rot + 8 * (int64_t)P.n_blk + 4 * (int64_t)P.n_av;
    if (P.n <= kSmemTablesMaxN && st > 0 && st * 8 <= 160 * 1024) {
      L.table_stride = st;
      L.tables = take((size_t)B * st * 8);
    }
  } else {
    L.n_tiles = 1 << (P.n - P.k);
    const int nstates = mode == VQC_MODE_FORWARD ? 1 : (mode == VQC_MODE_VJP ? 2 : 3);
    const size_t per = (size_t)nstates * N * esz + (size_t)L.K * P.NG * L.n_tiles * 8 +
                       (size_t)M * L.n_tiles * 8;
    int64_t chunk = (int64_t)(p->state_budget / std::max<size_t>(per, 1));
    // rows are the grid's y dimension (at most 65535 per launch)
    chunk = std::max<int64_t>(1, std::min<int64_t>({chunk, B, (int64_t)65535}));
    L.chunk = chunk;
    L.psi = take((size_t)chunk * N * esz);
    L.phi = take(adj ? (size_t)chunk * N * esz : 0);
    L.fin = take(mode == VQC_MODE_JACOBIAN ? (size_t)chunk * N * esz : 0);
    L.ipart = take(adj ? (size_t)chunk * L.K * P.NG * L.n_tiles * 8 : 0);
    const int ftiles = p->fwd ? 1 << (p->fwd->prog.n - p->fwd->prog.k) : L.n_tiles;
    L.epart = take((size_t)chunk * M * std::max(L.n_tiles, ftiles) * 8);
    auto stride_of = [](const HostProgram& Q) {
      const int64_t st = 2 * (int64_t)Q.n_rot + 8 * (int64_t)Q.n_blk + 4 * (int64_t)Q.n_av;
      return (st > 0 && st * 8 <= 160 * 1024) ? st : (int64_t)0;
    };
    if ((L.table_stride = stride_of(P)) > 0) L.tables = take((size_t)chunk * L.table_stride * 8);
    if (p->fwd && (L.ftable_stride = stride_of(p->fwd->prog)) > 0)
      L.ftables = take((size_t)chunk * L.ftable_stride * 8);
  }
  L.total = off + 256;
  return L;
}

// reduction slots of the shared-memory partial buffer (slots x threads
// doubles). Per-warp reductions keep one row of the pass's slots per warp:
// warps x max_red_per_pass doubles = (max_red_per_pass / 32) slots x threads.
// JIT HBM adjoint passes with both states per thread reduce their gradient
// partials per warp when the scheduler planned thread groups and a pass's
// slots fit a small table (deep passes keep the per-segment CTA reductions)
bool use_warp_red(const HostProgram& P) {
  return P.hbm && P.group_sync && P.adj_dual && P.pingpong == 0 && P.max_red_per_pass <= 512 && P.k - P.R >= 5;
}

int red_slots(const VqcPlan* p) {
  int rs = std::max(1, std::max(p->M, p->prog.max_red_per_seg));
  if (p->prog.warp_red) rs = std::max(rs, (p->prog.max_red_per_pass + 31) / 32);
  return rs;
}

// bytes per state element: complex128 or complex64
int elem_bytes(const VqcPlan* p) { return p->prog.precision == 1 ? 8 : 16; }

// samples per CTA in smem mode
int smem_samples(const VqcPlan* p, int64_t B, bool dual, size_t* smem_bytes, int* threads_per_sample) {
  const HostProgram& P = p->prog;
  const int TPS = 1 << (P.n - P.R);
  const bool split = dual && use_split(P.n, P.R) && !P.adj_dual;
  const int TT = split ? 2 * TPS : TPS;
  *threads_per_sample = TT;
  auto bytes_for = [&](int S) {
    return SmemLayout(S, 1 << P.n, dual, P.n_rot, P.n_blk, P.n_av, red_slots(p), S * TT, p->M,
                      (int)p->smask.size(), elem_bytes(p)).total;
  };
  const int max_threads = P.R >= 5 ? 256 : (split ? 512 : (P.R >= 4 ? 256 : 512));
  int smax = std::max(1, max_threads / TT);
  // samples per CTA: enough CTAs for VQC_SMEM_CTAS_PER_SM (default 2) per SM
  const int64_t cps = std::max(1, env_int("VQC_SMEM_CTAS_PER_SM", 2)) * (int64_t)p->sms;
  const int64_t want = std::max<int64_t>(1, (B + cps - 1) / cps);
  int S = 1;
  // JIT kernels of n >= 12 lag their reductions, which assumes one sample per CTA
  if (p->use_jit && P.n >= 12) smax = 1;
  while (S * 2 <= smax && S * 2 <= want && bytes_for(S * 2) <= (size_t)kMaxSmemBytes) S *= 2;
  *smem_bytes = bytes_for(S);
  return S;
}

// dynamic shared memory of a pass kernel; rs = reduction slots (0 for forward
// passes that neither observe nor reduce: more CTAs fit per SM)
size_t pass_smem(const VqcPlan* p, const HostProgram& P, bool dual, int rs = -1) {
  const int TPS = 1 << (P.k - P.R);
  return SmemLayout(1, 1 << P.k, dual, P.max_rot_per_pass, P.max_blk_per_pass, P.max_av_per_pass,
                    rs < 0 ? red_slots(p) : rs, (dual && !P.adj_dual) ? 2 * TPS : TPS, p->M,
                    (int)p->smask.size(), elem_bytes(p)).total;
}

int launch(const char* name, Kern k, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
           const DevProgram& D, const RunArgs& A) {
  if (smem > (size_t)kMaxSmemBytes) return fail(VQC_E_UNSUPPORTED, "shared-memory footprint too large");
  if (k.cu) {
    ProfScope ps(name, st);
    const CUresult cr = jit_launch(k.cu, grid.x, grid.y, block.x, smem, st, D, A);
    ++g_launches;
    if (cr != CUDA_SUCCESS) return fail(VQC_E_CUDA, "JIT kernel launch failed (CUresult " + std::to_string((int)cr) + ")");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return VQC_OK;
  }
  static std::mutex attr_mu;
  static std::vector<KFn> configured;
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    if (std::find(configured.begin(), configured.end(), k.fn) == configured.end()) {
      cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes);
      configured.push_back(k.fn);
    }
  }
  ProfScope ps(name, st);
  k.fn<<<grid, block, smem, st>>>(D, A);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return VQC_OK;
}

Kern smem_k(const VqcPlan* p, bool adj) {
  Kern k;
  if (p->use_jit) k.cu = adj ? p->jit.smem_adj : p->jit.smem_fwd;
  else k.fn = smem_kernel(p->prog.R, adj, use_split(p->prog.n, p->prog.R));
  return k;
}
Kern pass_k(const VqcPlan* p, bool dual, int pass) {
  Kern k;
  if (p->use_jit) k.cu = dual ? p->jit.pass_adj[pass] : p->jit.pass_fwd[pass];
  else k.fn = pass_kernel(p->prog.R, dual);
  return k;
}

int run_tile_reduce(const double* in, double* out, int64_t count, int n_tiles, cudaStream_t st) {
  if (count <= 0) return VQC_OK;
  const int threads = 256;
  const int64_t blocks = (count * 32 + threads - 1) / threads;
  ProfScope ps("tile_reduce", st);
  k_tile_reduce<<<(unsigned)blocks, threads, 0, st>>>(in, out, count, n_tiles);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VQC_OK : cuda_fail(e, "tile reduce");
}

// run forward (+ adjoint) for all rows; fills ip (B,K,NG) and d_expect
int run_core_impl(VqcPlan* p, const double* d_in, const double* d_w, int64_t B, const double* d_up,
                  double* d_expect, int mode, char* ws, const Layout& L, cudaStream_t st);

// run_core_impl, plus the device bounds checks of VQC_CHECKS plans: the
// failure bits are cleared before the launches and read back after them
int run_core(VqcPlan* p, const double* d_in, const double* d_w, int64_t B, const double* d_up,
             double* d_expect, int mode, char* ws, const Layout& L, cudaStream_t st) {
  if (p->d_check && cudaMemsetAsync(p->d_check, 0, sizeof(unsigned), st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "check reset");
  const int rc = run_core_impl(p, d_in, d_w, B, d_up, d_expect, mode, ws, L, st);
  if (rc || !p->d_check) return rc;
  unsigned bits = 0;
  cudaError_t e = cudaMemcpyAsync(&bits, p->d_check, sizeof bits, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "check read-back");
  if (bits) return fail(VQC_E_CUDA, "device bounds check failed (bits " + std::to_string(bits) + ")");
  return VQC_OK;
}

int run_core_impl(VqcPlan* p, const double* d_in, const double* d_w, int64_t B, const double* d_up,
                  double* d_expect, int mode, char* ws, const Layout& L, cudaStream_t st) {
  const HostProgram& P = p->prog;
  const DevProgram& D = p->D;
  RunArgs A{};
  A.inputs = d_in;
  A.weights = d_w;
  A.upstream = d_up;
  A.K = L.K;
  A.red_slots = red_slots(p);
  A.check = p->d_check;
  static unsigned long long* dbg = nullptr;
  const bool dbg_on = env_int("VQC_DEBUG_TIMING", 0) != 0;
  if (dbg_on) {
    if (!dbg) cudaMalloc(&dbg, DBG_N * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, DBG_N * sizeof(unsigned long long), st);
    A.dbg = dbg;
  }
  struct DbgPrint {
    bool on;
    unsigned long long* d;
    cudaStream_t st;
    ~DbgPrint() {
      if (!on) return;
      unsigned long long h[DBG_N];
      cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double ctas = h[DBG_CTAS] ? (double)h[DBG_CTAS] : 1.0;
      fprintf(stderr, "[vqc timing] per CTA cycles: prologue %.0f fwd %.0f observe %.0f bwd %.0f store %.0f | "
              "segments: load %.0f ops %.0f store %.0f final %.0f (ctas %.0f)\n",
              h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / ctas, h[4] / ctas, h[5] / ctas, h[6] / ctas,
              h[7] / ctas, h[8] / ctas, ctas);
    }
  } dbg_print{dbg_on, dbg, st};
  double* ip = reinterpret_cast<double*>(ws + L.ip);
  const bool adj = mode != VQC_MODE_FORWARD;
  if (!P.hbm) {
    size_t smem = 0;
    int TT = 1;
    const int S = smem_samples(p, B, adj, &smem, &TT);
    A.b0 = 0;
    A.nb = B;
    A.S = S;
    A.bra = -1;
    A.expect = d_expect;
    A.ip = ip;
    A.psi_fin = reinterpret_cast<double2*>(ws + L.fin);
    A.jacobian = mode == VQC_MODE_JACOBIAN;
    A.tables = nullptr;
    A.table_stride = 0;
    if (L.table_stride > 0 && B > 0) {
      A.tables = reinterpret_cast<double*>(ws + L.tables);
      A.table_stride = L.table_stride;
      if (int rc = launch("tables", Kern{k_tables, nullptr}, dim3((unsigned)B), dim3(256),
                          (size_t)L.table_stride * 8, st, D, A))
        return rc;
    }
    const dim3 grid((unsigned)((B + S - 1) / S)), block((unsigned)(S * TT));
    return launch(adj ? "smem_fwd_adjoint" : "smem_forward", smem_k(p, adj), grid,
                  block, smem, st, D, A);
  }
  // HBM passes, chunked over rows. The forward sweep runs the forward program
  // (p->fwd when the plan has a separate forward schedule, else `prog`); the
  // adjoint sweep always runs `prog`. With one program the last pass fuses
  // forward + observe + seed + the first adjoint pass.
  double2* psi = reinterpret_cast<double2*>(ws + L.psi);
  double2* phi = reinterpret_cast<double2*>(ws + L.phi);
  double2* fin = reinterpret_cast<double2*>(ws + L.fin);
  double* ipart = reinterpret_cast<double*>(ws + L.ipart);
  double* epart = reinterpret_cast<double*>(ws + L.epart);
  const bool sep = p->fwd != nullptr;
  const HostProgram& PF = sep ? p->fwd->prog : P;
  const DevProgram& DF = sep ? p->fwd->D : D;
  const int TPS = 1 << (P.k - P.R), TPSF = 1 << (PF.k - PF.R);
  const int NP = (int)P.passes.size(), NPF = (int)PF.passes.size();
  const int tiles_f = 1 << (PF.n - PF.k);
  const size_t smF = pass_smem(p, PF, false), smF0 = pass_smem(p, PF, false, 0), smB = pass_smem(p, P, true);
  for (int64_t b0 = 0; b0 < B; b0 += L.chunk) {
    const int64_t nb = std::min<int64_t>(L.chunk, B - b0);
    A.b0 = b0;
    A.nb = nb;
    A.S = 1;
    A.psi = psi;
    A.phi = phi;
    A.psi_fin = fin;
    // a tile that is the whole state has no per-tile partials to sum: the
    // kernels write expectations and inner products in their final layout
    const bool one_tile = L.n_tiles == 1 && tiles_f == 1;
    A.expect = (one_tile && d_expect) ? d_expect + (size_t)b0 * p->M : epart;
    A.ip = one_tile ? ip + (size_t)b0 * L.K * P.NG : ipart;
    A.bra = -1;
    int rc;
    // per-sample angle / block tables of each program that runs
    RunArgs AF = A;  // forward sweep arguments
    A.tables = nullptr;
    A.table_stride = 0;
    AF.tables = nullptr;
    AF.table_stride = 0;
    // (a whole-state tile is its sample's only CTA: it builds the tables
    // itself, build_tables in pass_body, instead of a k_tables launch)
    if (one_tile) {
    } else if (L.table_stride > 0 && (!sep || mode != VQC_MODE_FORWARD)) {
      A.tables = reinterpret_cast<double*>(ws + L.tables);
      A.table_stride = L.table_stride;
      if ((rc = launch("tables", Kern{k_tables, nullptr}, dim3((unsigned)nb), dim3(256),
                       (size_t)L.table_stride * 8, st, D, A)))
        return rc;
    }
    if (!sep) {
      AF.tables = A.tables;
      AF.table_stride = A.table_stride;
    } else if (L.ftable_stride > 0 && !one_tile) {
      AF.tables = reinterpret_cast<double*>(ws + L.ftables);
      AF.table_stride = L.ftable_stride;
      if ((rc = launch("tables", Kern{k_tables, nullptr}, dim3((unsigned)nb), dim3(256),
                       (size_t)L.ftable_stride * 8, st, DF, AF)))
        return rc;
    }
    // ping-pong JIT kernels: two tile groups per CTA (half the grid, twice
    // the block and its shared memory)
    const int Gb = P.pingpong ? 2 : 1, Gf = PF.pingpong ? 2 : 1;
    const dim3 grid((unsigned)(L.n_tiles / Gb), (unsigned)nb), grid_f((unsigned)(tiles_f / Gf), (unsigned)nb);
    const dim3 block_f((unsigned)(Gf * TPSF)), block2((unsigned)(Gb * (P.adj_dual ? TPS : 2 * TPS)));
    auto fwd_pass = [&](int pi, uint32_t flags) {
      AF.pass = pi;
      AF.flags = flags;
      const bool obs = (flags & F_OBSERVE) != 0;
      AF.red_slots = obs ? A.red_slots : 0;
      Kern k;
      if (sep) k.cu = p->fwd->jit.pass_fwd[pi];
      else k = pass_k(p, false, pi);
      return launch("pass_forward", k, grid_f, block_f, Gf * (obs ? smF : smF0), st, DF, AF);
    };
    auto adj_pass = [&](int pi, uint32_t flags) {
      A.pass = pi;
      A.flags = flags;
      return launch("pass_adjoint", pass_k(p, true, pi), grid, block2, Gb * smB, st, D, A);
    };
    const uint32_t stores = F_STORE_PSI | F_STORE_PHI;
    // forward sweep: all but the last forward pass
    for (int pi = 0; pi < NPF - 1; ++pi)
      if ((rc = fwd_pass(pi, (pi == 0 ? F_INIT : F_LOAD_PSI) | F_FWD | F_STORE_PSI))) return rc;
    const uint32_t first = NPF == 1 ? F_INIT : F_LOAD_PSI;
    int exp_tiles = tiles_f;  // tiles of the kernel that observes (expectation partials)
    if (mode == VQC_MODE_FORWARD) {
      if ((rc = fwd_pass(NPF - 1, first | F_FWD | F_OBSERVE))) return rc;
    } else if (mode == VQC_MODE_VJP) {
      if (!sep) {
        if ((rc = adj_pass(NP - 1, first | F_FWD | F_OBSERVE | F_SEED | F_BWD | (NP > 1 ? stores : 0)))) return rc;
      } else {
        if ((rc = fwd_pass(NPF - 1, first | F_FWD | F_STORE_PSI))) return rc;
        if ((rc = adj_pass(NP - 1, F_LOAD_PSI | F_OBSERVE | F_SEED | F_BWD | (NP > 1 ? stores : 0)))) return rc;
      }
      exp_tiles = L.n_tiles;
      for (int pi = NP - 2; pi >= 0; --pi)
        if ((rc = adj_pass(pi, F_LOAD_PSI | F_LOAD_PHI | F_BWD | (pi > 0 ? stores : 0)))) return rc;
    } else {
      if ((rc = fwd_pass(NPF - 1, first | F_FWD | F_OBSERVE | F_STORE_FIN))) return rc;
      for (int m = 0; m < p->M; ++m) {
        A.bra = m;
        if ((rc = adj_pass(NP - 1, F_LOAD_FIN | F_SEED | F_BWD | (NP > 1 ? stores : 0)))) return rc;
        for (int pi = NP - 2; pi >= 0; --pi)
          if ((rc = adj_pass(pi, F_LOAD_PSI | F_LOAD_PHI | F_BWD | (pi > 0 ? stores : 0)))) return rc;
      }
    }
    if (adj && !one_tile && (rc = run_tile_reduce(ipart, ip + (size_t)b0 * L.K * P.NG, nb * L.K * P.NG, L.n_tiles, st)))
      return rc;
    if (d_expect && !one_tile && (rc = run_tile_reduce(epart, d_expect + (size_t)b0 * p->M, nb * p->M, exp_tiles, st)))
      return rc;
  }
  return VQC_OK;
}

int run_chain(VqcPlan* p, const double* d_in, const double* d_w, const double* ip, int64_t B, int K,
              double* out, cudaStream_t st) {
  const HostProgram& P = p->prog;
  const int64_t total = B * K * P.n_cols;
  if (total <= 0) return VQC_OK;
  RunArgs A{};
  A.inputs = d_in;
  A.weights = d_w;
  A.b0 = 0;
  const int threads = 256;
  ProfScope ps("chain_rule", st);
  k_chain<<<(unsigned)((total + threads - 1) / threads), threads, 0, st>>>(
      p->D, A, ip, B, K, p->d_col_offs, p->d_chain, P.n_cols, out);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VQC_OK : cuda_fail(e, "chain rule");
}

int check_common(const VqcPlan* p, const double* d_in, const double* d_w, int64_t B) {
  if (!p) return fail(VQC_E_INVALID, "plan is NULL");
  if (B < 0) return fail(VQC_E_INVALID, "batch size must be >= 0");
  if (B > 0 && p->enc_size > 0 && !d_in) return fail(VQC_E_INVALID, "inputs pointer is NULL");
  if (p->total_params > 0 && !d_w) return fail(VQC_E_INVALID, "weights pointer is NULL");
  if (B > (int64_t)65535 * 65535) return fail(VQC_E_INVALID, "batch too large");
  return VQC_OK;
}

// flat gate list -> scheduled device program (shared by plan creation and
// the CPU-side JIT source dump)
int schedule_circuit(const VqcCircuit* c, const int64_t* wrt_col, HostProgram* prog,
                     std::vector<uint32_t>* zmask = nullptr, std::vector<double>* zcoeff = nullptr,
                     int tile_override = 0, int regs_override = 0, int precision = 0) {
  // Idle-qubit padding: a circuit of 4-7 qubits is planned on 8, the extra
  // qubits staying in |0>, so it runs the pass kernels (one warp per sample,
  // warp-level synchronisation and reductions) instead of the on-chip kernels,
  // which are latency-bound at a few warps per SM: 16384 rows of 8 layers on
  // 4 / 5 / 6 / 7 qubits 2.9e6 / 4.0e6 / 5.6e6 / 4.2e6 -> 1.46e7 / 1.24e7 /
  // 1.14e7 / 9.6e6 samples/s, cfg1 0.072 -> 0.047 ms per call. Amplitudes
  // with an idle bit set stay exactly zero, so results only move by summation
  // order. VQC_PAD_QUBITS=0 turns it off (the on-chip JIT kernels).
  // VQC_PAD_FROM=1 extends it to 1-3 qubit circuits, which otherwise run the
  // prebuilt interpreter without a JIT compile (16384 rows x 8 layers at 2 /
  // 3 qubits: 5.2e6 / 3.4e6 -> 2.3e7 / 1.5e7 samples/s; 64-row calls lose 5 %).
  const int n_true = c->n_qubits;
  const int pad_to = env_int("VQC_JIT", -1) != 0 ? std::min(kSmemMaxQubits, env_int("VQC_PAD_QUBITS", kPassMinQubits)) : 0;
  const int nq = (n_true >= env_int("VQC_PAD_FROM", 4) && n_true < pad_to) ? pad_to : n_true;
  if (nq != n_true)
    for (int64_t g = 0; g < c->n_gates; ++g) {
      const bool two = c->kinds[g] == G_CNOT || c->kinds[g] == G_CZ;
      if (c->q0[g] < 0 || c->q0[g] >= n_true || (two && (c->q1[g] < 0 || c->q1[g] >= n_true)))
        return fail(VQC_E_INVALID, "gate " + std::to_string(g) + ": qubit out of range");
    }
  std::vector<GateIn> gates((size_t)c->n_gates);
  for (int64_t g = 0; g < c->n_gates; ++g) {
    GateIn& gi = gates[g];
    gi.kind = (int)c->kinds[g];
    gi.q0 = (int)c->q0[g];
    gi.q1 = (int)c->q1[g];
    gi.coeff = c->coeff[g];
    if (gi.kind >= G_RX && gi.kind <= G_RZ) {
      const int64_t lo = c->f_offs[g], hi = c->f_offs[g + 1];
      if (lo < 0 || hi < lo || (hi > lo && !c->f_idx)) return fail(VQC_E_INVALID, "bad f_offs");
      for (int64_t t = lo; t < hi; ++t) gi.fidx.push_back((int32_t)c->f_idx[t]);
      if ((int)gi.fidx.size() > kMaxFactors)
        return fail(VQC_E_UNSUPPORTED, "gate " + std::to_string(g) + ": more than 4 angle factors");
    }
  }
  std::vector<int64_t> wcol((size_t)c->total_params, -1);
  for (int64_t i = 0; i < c->total_params; ++i) wcol[i] = wrt_col[i];
  if (zmask) prog->absorbed = absorb_trailing_gates(&gates, nq, zmask, zcoeff);
  ScheduleOptions opt;
  // HBM tiles: 2^11 complex128 amplitudes (32 KiB per state); complex64
  // elements are half the size, so its tiles hold 2^12 (same bytes)
  opt.tile_qubits = env_int("VQC_TILE_QUBITS", precision == 1 ? kHbmTileC64 : 11);
  // States of more qubits than this run the pass kernels (tile load, register
  // segments with thread-group barriers and per-warp reductions, tile store).
  // With JIT kernels that includes n = 8 ... 12, whose single tile is the
  // whole state (cfg3: 5.87 -> 4.70 ms against the on-chip thread-pair
  // kernel); smaller plans keep several samples per CTA. VQC_SMEM_MAX_QUBITS
  // moves the boundary; interpreter-only plans (VQC_JIT=0) stay on chip to 12.
  opt.smem_max_qubits = env_int("VQC_JIT", -1) != 0
                            ? std::max(3, std::min(kSmemMaxQubits, env_int("VQC_SMEM_MAX_QUBITS", kPassMinQubits - 1)))
                            : kSmemMaxQubits;
  // register slots of a pass plan: 3 with both states per thread; complex64
  // streams 2^12 tiles with 4 (its whole-state tiles of n <= 12 keep 3)
  const int pass_regs = std::max(3, std::min(4, env_int("VQC_REG_SLOTS", (precision == 1 && nq > kSmemMaxQubits)
                                                                               ? kHbmRegsC64 : kHbmAdjointRegs)));
  // (the per-warp reductions of the pass kernels need a full warp per tile)
  if (nq <= kSmemMaxQubits && nq - pass_regs < 5) opt.smem_max_qubits = kSmemMaxQubits;
  if (nq > opt.smem_max_qubits && nq <= kSmemMaxQubits) opt.tile_qubits = nq;
  // whole-state tiles (n <= 12 on the pass kernels): passes of at most this
  // many segments, a bound on the JIT compile time of deep circuits (0: one pass)
  if (nq > opt.smem_max_qubits && nq <= kSmemMaxQubits)
    opt.max_pass_segments = std::max(0, env_int("VQC_PASS_SEGMENTS", 48));
  opt.segment_cost = env_int("VQC_SEGMENT_COST", 4);
  opt.variants = std::max(1, env_int("VQC_SCHED_VARIANTS", 1));
  opt.forced_low = std::max(0, std::min(3, env_int("VQC_FORCED_LOW", 3)));  // contiguous low qubits per pass
  // four register slots (16 amplitudes per thread); the scheduler and its
  // CPU checker also handle 3 and 5 (tests/test_scheduler_sim.py). Other
  // values (VQC_REG_SLOTS) only for JIT-compiled HBM plans: the prebuilt
  // interpreter kernels exist for R = 4 passes only.
  opt.reg_slots = 4;
  if (nq > opt.smem_max_qubits && env_int("VQC_JIT", -1) != 0)
    opt.reg_slots = pass_regs;
  // small on-chip JIT plans: 3 slots, both states per thread (smem_dual)
  if (nq <= opt.smem_max_qubits && smem_dual(nq)) opt.reg_slots = 3;
  // HBM plans run JIT kernels, whose address maps take CNOT folds onto
  // thread-bit targets (boundary CNOTs then need no register slot: cfg4 80 ->
  // 62 adjoint and 62 -> 52 forward segments); VQC_FOLD_THREAD_TARGETS=0 off
  // (2 = forward program only, 3 = adjoint / main program only: bisection knobs)
  const int ftt = env_int("VQC_FOLD_THREAD_TARGETS", 1);
  const bool fwd_prog = tile_override > 0 || regs_override > 0;
  opt.fold_thread_targets = nq > opt.smem_max_qubits && env_int("VQC_JIT", -1) != 0 &&
                            (ftt == 1 || (ftt == 2 && fwd_prog) || (ftt == 3 && !fwd_prog));
  // thread-group barriers and per-warp reductions in the JIT HBM pass kernels
  // (VQC_GROUP_SYNC=0: CTA barriers and per-segment CTA reductions as before)
  opt.group_sync = nq > opt.smem_max_qubits && env_int("VQC_JIT", -1) != 0 &&
                   env_int("VQC_GROUP_SYNC", 1) != 0 && env_int("VQC_PINGPONG", 0) == 0;
  if (tile_override > 0) opt.tile_qubits = tile_override;
  if (regs_override > 0) opt.reg_slots = regs_override;
  const int absorbed = prog->absorbed;
  std::string err = build_program(gates, nq, c->total_params, wcol, opt, prog);
  // Passes keep qubits 0-2 local (128-byte chunks in HBM). Keeping only qubits
  // 0-1 (64-byte chunks) frees a local qubit: worth it only when it saves a
  // pass (cfg4 16 -> 15 passes, +1 %; cfg5 keeps 13 and would lose 1.5 %).
  if (err.empty() && prog->hbm && nq > prog->k && opt.forced_low == 3 && std::getenv("VQC_FORCED_LOW") == nullptr) {
    ScheduleOptions opt2 = opt;
    opt2.forced_low = 2;
    HostProgram alt;
    if (build_program(gates, nq, c->total_params, wcol, opt2, &alt).empty() && alt.passes.size() < prog->passes.size())
      *prog = std::move(alt);
  }
  prog->absorbed = absorbed;
  if (!err.empty())
    return fail(err.find("out of range") != std::string::npos || err.find("duplicate") != std::string::npos
                    ? VQC_E_INVALID
                    : VQC_E_UNSUPPORTED,
                err);
  return VQC_OK;
}

// DevProgram of a scheduled program (its tables + the plan's observables)
void fill_dev(const VqcPlan* p, const HostProgram& P, const ProgTabs& t, DevProgram& D) {
  D.ops = t.ops;
  D.segs = t.segs;
  D.ipouts = t.ipouts;
  D.blocks = t.blocks;
  D.members = t.members;
  D.diag = t.diag;
  D.setids = t.setids;
  D.thr_tab = t.thr_tab;
  D.passes = t.passes;
  D.rots = t.rots;
  D.n_blk = P.n_blk;
  D.n_av = P.n_av;
  D.max_rot_pass = P.max_rot_per_pass;
  D.max_blk_pass = P.max_blk_per_pass;
  D.max_av_pass = P.max_av_per_pass;
  D.term_offs = p->d_term_offs;
  D.t_smask = p->d_smask;
  D.t_xmask = p->d_xmask;
  D.t_phase = p->d_tphase;
  D.has_xy = p->has_xy ? 1 : 0;
  D.t_coeff = p->d_tcoeff;
  D.t_obs = p->d_tobs;
  D.n = P.n;
  D.k = P.k;
  D.R = P.R;
  D.NG = P.NG;
  D.n_rot = P.n_rot;
  D.M = p->M;
  D.T = (int)p->smask.size();
  D.n_pass = (int)P.passes.size();
  D.enc_off = p->enc_off;
  D.enc_size = p->enc_size;
}

}  // namespace

// ------------------------------------------------------------------ C ABI

extern "C" {

int vqc_abi_version(void) { return VQC_ABI_VERSION; }

int64_t vqc_jit_source(const VqcCircuit* c, const int64_t* wrt_col, int compile, char* buf, int64_t cap,
                       double* compile_s) {
  g_err.clear();
  if (!c || (c->total_params > 0 && !wrt_col)) return fail(VQC_E_INVALID, "NULL argument");
  if (c->n_qubits < 1 || c->n_qubits > kMaxQubits) return fail(VQC_E_INVALID, "num_qubits must be in [1, 24]");
  HostProgram prog;
  std::vector<uint32_t> zm;  // as for Z-string observables (trailing gates absorbed)
  std::vector<double> zc;
  const int prec = env_int("VQC_JIT_SOURCE_PRECISION", 0) == 1 ? 1 : 0;  // dump / compile a complex64 plan
  if (int rc = schedule_circuit(c, wrt_col, &prog, &zm, &zc, 0, 0, prec)) return rc;
  if ((prog.hbm || (prog.R <= 3 && smem_dual(prog.n))) &&
      env_int("VQC_ADJ_DUAL", (prog.R <= 3 || (prog.hbm && prec == 1)) ? 1 : 0) != 0)
    prog.adj_dual = true;
  prog.precision = prec;
  prog.pingpong = prog.hbm ? std::max(0, std::min(2, env_int("VQC_PINGPONG", 0))) : 0;
  prog.warp_red = use_warp_red(prog);
  prog.direct_io = prog.hbm && prog.group_sync && prog.pingpong == 0 && env_int("VQC_DIRECT_IO", 0) != 0;
  if (env_int("VQC_JIT_SOURCE_TERMS", 0) != 0) {  // per-qubit <Z_i> as compile-time terms (CPU compile checks)
    for (int q = 0; q < prog.n; ++q) {
      prog.obs_mask.push_back(1u << q);
      prog.obs_coeff.push_back(1.0 + 0.125 * q);
      prog.obs_offs.push_back(q);
    }
    prog.obs_offs.push_back(prog.n);
  }
  build_thr_table(prog.segs);  // per-segment thread-table offsets, as at plan creation
  const bool split = use_split(prog.n, prog.R) && !prog.adj_dual;
  const std::string src = jit_source(prog, split);
  if (compile) {
    std::string err = jit_compile_only(prog, split, compile_s);
    if (!err.empty()) return fail(VQC_E_CUDA, err);
  }
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, (int64_t)src.size());
    memcpy(buf, src.data(), (size_t)n);
    buf[n] = 0;
  }
  return (int64_t)src.size();
}

const char* vqc_last_error(void) { return g_err.c_str(); }

int64_t vqc_last_launch_count(void) { return g_launches; }

void vqc_profile_enable(int on) {
  g_prof = on != 0;
  if (g_prof) g_prof_agg.clear();
}

int64_t vqc_profile_report(char* buf, int64_t cap) {
  for (ProfPending& p : g_prof_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.e1) == cudaSuccess) cudaEventElapsedTime(&ms, p.e0, p.e1);
    bool found = false;
    for (ProfAgg& a : g_prof_agg)
      if (a.name == p.name) { a.ms += ms; a.count += 1; found = true; break; }
    if (!found) g_prof_agg.push_back({p.name, (double)ms, 1});
    g_prof_pool.push_back(p.e0);
    g_prof_pool.push_back(p.e1);
  }
  g_prof_pending.clear();
  std::string js = "{";
  for (size_t i = 0; i < g_prof_agg.size(); ++i) {
    char tmp[160];
    snprintf(tmp, sizeof tmp, "%s\"%s\": [%.6f, %lld]", i ? ", " : "", g_prof_agg[i].name.c_str(),
             g_prof_agg[i].ms, (long long)g_prof_agg[i].count);
    js += tmp;
  }
  js += "}";
  if (buf && cap > 0) {
    const int64_t c = std::min<int64_t>(cap - 1, (int64_t)js.size());
    memcpy(buf, js.data(), (size_t)c);
    buf[c] = 0;
  }
  return (int64_t)js.size();
}

int vqc_plan_create(const VqcCircuit* c, const VqcObservables* obs, const int64_t* wrt_col, int precision,
                    VqcPlan** out) {
  g_err.clear();
  if (!c || !obs || !out) return fail(VQC_E_INVALID, "NULL argument");
  *out = nullptr;
  if (precision != 0 && precision != 1)
    return fail(VQC_E_INVALID, "precision must be 0 (complex128) or 1 (complex64), got " + std::to_string(precision));
  if (precision == 1 && env_int("VQC_JIT", -1) == 0)
    return fail(VQC_E_UNSUPPORTED, "complex64 plans run JIT-compiled kernels only (VQC_JIT=0 set)");
  if (c->n_qubits < 1 || c->n_qubits > kMaxQubits)
    return fail(VQC_E_INVALID, "num_qubits must be in [1, 24], got " + std::to_string(c->n_qubits));
  if (c->n_gates < 0 || c->total_params < 0) return fail(VQC_E_INVALID, "negative sizes");
  if (c->n_gates > 0 && (!c->kinds || !c->q0 || !c->q1 || !c->coeff || !c->f_offs))
    return fail(VQC_E_INVALID, "NULL gate table");
  if (c->enc_offset < 0 || c->enc_size < 0 || c->enc_offset + c->enc_size > c->total_params)
    return fail(VQC_E_INVALID, "encoding slot out of range");
  if (obs->n_obs < 0 || (obs->n_obs > 0 && (!obs->term_offs)))
    return fail(VQC_E_INVALID, "bad observable table");
  if (c->total_params > 0 && !wrt_col) return fail(VQC_E_INVALID, "wrt_col is NULL");

  VqcPlan* p = new VqcPlan();
  p->total_params = c->total_params;
  p->enc_off = c->enc_offset;
  p->enc_size = c->enc_size;
  p->M = (int)obs->n_obs;
  p->circuit_qubits = c->n_qubits;
  p->term_offs.assign((size_t)p->M + 1, 0);
  const uint32_t nmask = c->n_qubits >= 32 ? 0xffffffffu : ((1u << c->n_qubits) - 1u);
  for (int m = 0; m < p->M; ++m) {
    const int64_t lo = obs->term_offs[m], hi = obs->term_offs[m + 1];
    if (lo < 0 || hi < lo) { delete p; return fail(VQC_E_INVALID, "bad term_offs"); }
    for (int64_t t = lo; t < hi; ++t) {
      if (obs->x_masks[t] != 0 && c->n_qubits > kSmemMaxQubits) {
        delete p;
        return fail(VQC_E_UNSUPPORTED,
                    "observable " + std::to_string(m) + ": X/Y Pauli strings are supported for n <= 12 only "
                    "(Z strings only on the HBM path)");
      }
      if (obs->x_masks[t] < 0 || ((uint64_t)obs->x_masks[t] & ~(uint64_t)nmask)) {
        delete p;
        return fail(VQC_E_INVALID, "observable x mask out of range");
      }
      if (obs->sign_masks[t] < 0 || ((uint64_t)obs->sign_masks[t] & ~(uint64_t)nmask)) {
        delete p;
        return fail(VQC_E_INVALID, "observable sign mask out of range");
      }
      // phase = i^{#Y}: recover the power from the (re, im) pair
      const double pr = obs->phases ? obs->phases[2 * t] : 1.0, pim = obs->phases ? obs->phases[2 * t + 1] : 0.0;
      int ph = -1;
      if (pr == 1.0 && pim == 0.0) ph = 0;
      else if (pr == 0.0 && pim == 1.0) ph = 1;
      else if (pr == -1.0 && pim == 0.0) ph = 2;
      else if (pr == 0.0 && pim == -1.0) ph = 3;
      if (ph < 0) { delete p; return fail(VQC_E_INVALID, "Pauli phase must be a power of i"); }
      p->smask.push_back((uint32_t)obs->sign_masks[t]);
      p->xmask.push_back((uint32_t)obs->x_masks[t]);
      p->tphase.push_back(ph);
      p->tcoeff.push_back(obs->coeffs[t]);
      p->tobs.push_back((int32_t)m);
      if (obs->x_masks[t] != 0) p->has_xy = true;
    }
    p->term_offs[m + 1] = (int32_t)p->smask.size();
  }
  // Z-only observables absorb the circuit's trailing CNOT / CZ / X gates
  // (G^dagger O G is again a Z string): fewer state passes, same results
  if (int rc = schedule_circuit(c, wrt_col, &p->prog, p->has_xy ? nullptr : &p->smask,
                                p->has_xy ? nullptr : &p->tcoeff, 0, 0, precision)) {
    delete p;
    return rc;
  }
  p->prog.precision = precision;
  p->prog.checks = env_int("VQC_CHECKS", 0) != 0;
  std::string err;
  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, p->device);
  const HostProgram& P = p->prog;
  if (e == cudaSuccess) e = p->tabs.upload_all(p->prog.segs, p->prog);
  if (e == cudaSuccess) e = upload(p->term_offs, &p->d_term_offs);
  if (e == cudaSuccess) e = upload(p->smask, &p->d_smask);
  if (e == cudaSuccess) e = upload(p->xmask, &p->d_xmask);
  if (e == cudaSuccess) e = upload(p->tphase, &p->d_tphase);
  if (e == cudaSuccess) e = upload(p->tcoeff, &p->d_tcoeff);
  if (e == cudaSuccess) e = upload(p->tobs, &p->d_tobs);
  if (e == cudaSuccess) e = upload(P.col_offs, &p->d_col_offs);
  if (e == cudaSuccess) e = upload(P.chain, &p->d_chain);
  if (e == cudaSuccess && P.checks) e = cudaMalloc(reinterpret_cast<void**>(&p->d_check), sizeof(unsigned));
  if (e != cudaSuccess) {
    vqc_plan_destroy(p);
    return cuda_fail(e, "plan upload");
  }
  fill_dev(p, P, p->tabs, p->D);
  p->state_budget = (size_t)env_int("VQC_STATE_BUDGET_MB", 16384) << 20;
  // JIT policy (VQC_JIT): unset = specialise HBM-pass plans (per-pass units
  // compile in parallel) and on-chip plans of n >= 8 qubits (shape-shared
  // segment code, one unit); 1 = every plan, 0 = interpreter only. Small
  // circuits are launch-bound and stay on the prebuilt interpreter.
  const int jit_mode = env_int("VQC_JIT", -1);
  // complex64 plans always specialise (the interpreter kernels are complex128)
  const bool want_jit = precision == 1 || P.checks || jit_mode > 0 || (jit_mode < 0 && (P.hbm || P.n >= 4));
  if (want_jit && (P.n_fwd_ops + P.n_bwd_ops > 0 || precision == 1 || P.checks)) {
    // HBM adjoint with both states per thread when its register slots allow
    // (VQC_ADJ_DUAL overrides: 0 = thread pairs)
    if ((P.hbm || (P.R <= 3 && smem_dual(P.n))) &&
        env_int("VQC_ADJ_DUAL", (P.R <= 3 || (P.hbm && precision == 1)) ? 1 : 0) != 0)
      p->prog.adj_dual = true;
    // HBM passes: ping-pong tile groups (VQC_PINGPONG=0 turns them off)
    // off by default: both modes measured slower than two free-running CTAs
    // per SM on cfg4 / cfg5
    const int pp_mode = std::max(0, std::min(2, env_int("VQC_PINGPONG", 0)));
    const int pingpong = (P.hbm && P.n - P.k >= 1 && 2 * pass_smem(p, P, true) <= (size_t)kMaxSmemBytes)
                             ? pp_mode : 0;
    p->prog.pingpong = pingpong;
    p->prog.warp_red = use_warp_red(p->prog);
    p->prog.direct_io = P.hbm && P.group_sync && pingpong == 0 && env_int("VQC_DIRECT_IO", 0) != 0;
    // separate forward schedule (VQC_FWD_TILE / VQC_FWD_REG) when it differs:
    // the main program then only needs its adjoint pass kernels and the
    // forward program its forward ones, and the two builds run side by side
    const int ft = env_int("VQC_FWD_TILE", P.k),
              fr = std::max(3, std::min(5, env_int("VQC_FWD_REG", P.n <= kPassFusedMaxQubits ? P.R : kHbmForwardRegs)));
    const bool sep = P.hbm && (ft != P.k || fr != P.R);
    p->prog.jit_kernels = sep ? 2 : 3;
    // Z-string observables become compile-time constants of the observing pass
    if (!p->has_xy && env_int("VQC_CONST_TERMS", 1) != 0) {
      p->prog.obs_mask = p->smask;
      p->prog.obs_coeff = p->tcoeff;
      p->prog.obs_offs = p->term_offs;
    }
    std::string main_err;
    std::thread main_build([&]() {
      cudaSetDevice(p->device);
      main_err = jit_build(P, use_split(P.n, P.R) && !P.adj_dual, &p->jit);
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() { if (t.joinable()) t.join(); }
    } joiner{main_build};
    p->use_jit = true;
    if (sep) {
      ProgDev* f = new ProgDev();
      p->fwd = f;
      std::vector<uint32_t> zm = p->smask;  // the same trailing gates are absorbed; masks already rewritten
      std::vector<double> zc = p->tcoeff;
      const bool z = !p->has_xy;
      if (int rc = schedule_circuit(c, wrt_col, &f->prog, z ? &zm : nullptr, z ? &zc : nullptr, ft, fr)) {
        vqc_plan_destroy(p);
        return rc;
      }
      f->prog.precision = precision;
      f->prog.checks = P.checks;
      f->prog.pingpong = (f->prog.n - f->prog.k >= 1 && 2 * pass_smem(p, f->prog, false) <= (size_t)kMaxSmemBytes)
                             ? pingpong : 0;
      f->prog.direct_io = f->prog.hbm && f->prog.group_sync && f->prog.pingpong == 0 && env_int("VQC_DIRECT_IO", 0) != 0;
      if (!f->prog.hbm || f->prog.NG != P.NG) {
        vqc_plan_destroy(p);
        return fail(VQC_E_UNSUPPORTED, "forward schedule disagrees with the adjoint schedule");
      }
      if ((e = f->tabs.upload_all(f->prog.segs, f->prog)) != cudaSuccess) {
        vqc_plan_destroy(p);
        return cuda_fail(e, "plan upload");
      }
      fill_dev(p, f->prog, f->tabs, f->D);
      f->prog.jit_kernels = 1;
      f->prog.obs_mask = p->prog.obs_mask;
      f->prog.obs_coeff = p->prog.obs_coeff;
      f->prog.obs_offs = p->prog.obs_offs;
      err = jit_build(f->prog, false, &f->jit);
      if (!err.empty()) {
        main_build.join();
        vqc_plan_destroy(p);
        return fail(VQC_E_CUDA, err);
      }
    }
    main_build.join();
    if (!main_err.empty()) {
      vqc_plan_destroy(p);
      return fail(VQC_E_CUDA, main_err);
    }
  }
  *out = p;
  return VQC_OK;
}

void vqc_plan_destroy(VqcPlan* p) {
  if (!p) return;
  p->tabs.free_all();
  if (p->fwd) {
    p->fwd->tabs.free_all();
    delete p->fwd;
  }
  cudaFree(p->d_term_offs);
  cudaFree(p->d_smask);
  cudaFree(p->d_xmask);
  cudaFree(p->d_tphase);
  cudaFree(p->d_tcoeff);
  cudaFree(p->d_tobs);
  cudaFree(p->d_col_offs);
  cudaFree(p->d_chain);
  cudaFree(p->d_check);
  if (p->h_dev) cudaFree(p->h_dev);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

int64_t vqc_plan_num_cols(const VqcPlan* p) { return p ? p->prog.n_cols : -1; }
int64_t vqc_plan_num_obs(const VqcPlan* p) { return p ? p->M : -1; }
int vqc_plan_mode(const VqcPlan* p) { return p ? (p->prog.hbm ? 1 : 0) : -1; }

int64_t vqc_plan_describe(const VqcPlan* p, char* buf, int64_t cap) {
  if (!p) return -1;
  const HostProgram& P = p->prog;
  int nseg = 0;
  for (const PassDesc& pd : P.passes) nseg += pd.seg_end - pd.seg_begin;
  char tmp[1024];
  const int len = snprintf(tmp, sizeof tmp,
                           "{\"n\": %d, \"mode\": \"%s\", \"tile_qubits\": %d, \"reg_slots\": %d, "
                           "\"passes\": %d, \"segments\": %d, \"rotations\": %d, \"grad_slots\": %d, "
                           "\"fwd_ops\": %d, \"bwd_ops\": %d, \"cols\": %d, \"obs\": %d, \"jit\": %s, "
                           "\"jit_compile_s\": %.3f, \"jit_cubin_bytes\": %zu, \"absorbed_gates\": %d, \"adjoint_dual\": %s, "
                           "\"fwd_tile_qubits\": %d, \"fwd_reg_slots\": %d, \"fwd_passes\": %d, \"precision\": \"%s\", \"pingpong\": %d, "
                           "\"circuit_qubits\": %d, \"thread_group_barriers\": %s, \"warp_reductions\": %s}",
                           P.n, P.hbm ? "hbm" : "smem", P.k, P.R, (int)P.passes.size(), nseg, P.n_rot,
                           P.NG, P.n_fwd_ops, P.n_bwd_ops, P.n_cols, p->M, p->use_jit ? "true" : "false",
                           p->jit.compile_s + (p->fwd ? p->fwd->jit.compile_s : 0.0),
                           p->jit.cubin_bytes + (p->fwd ? p->fwd->jit.cubin_bytes : 0), P.absorbed,
                           P.adj_dual ? "true" : "false", p->fwd ? p->fwd->prog.k : P.k,
                           p->fwd ? p->fwd->prog.R : P.R, (int)(p->fwd ? p->fwd->prog.passes.size() : P.passes.size()),
                           P.precision == 1 ? "complex64" : "complex128", P.pingpong, p->circuit_qubits,
                           P.group_sync ? "true" : "false", P.warp_red ? "true" : "false");
  if (buf && cap > 0) {
    const int64_t c = std::min<int64_t>(cap - 1, len);
    memcpy(buf, tmp, (size_t)c);
    buf[c] = 0;
  }
  return len;
}

size_t vqc_workspace_bytes(const VqcPlan* p, int64_t B, int mode) {
  if (!p || B < 0 || mode < 0 || mode > 2) return 0;
  return make_layout(p, B, mode).total;
}

int vqc_forward(VqcPlan* p, const double* d_in, const double* d_w, int64_t B, double* d_expect, void* ws,
                size_t ws_bytes, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_common(p, d_in, d_w, B);
  if (rc) return rc;
  if (B == 0 || p->M == 0) return VQC_OK;
  if (!d_expect) return fail(VQC_E_INVALID, "expect pointer is NULL");
  const Layout L = make_layout(p, B, VQC_MODE_FORWARD);
  if (ws_bytes < L.total || (!ws && L.total > 0)) return fail(VQC_E_WORKSPACE, "workspace too small");
  char* w = reinterpret_cast<char*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  return run_core(p, d_in, d_w, B, nullptr, d_expect, VQC_MODE_FORWARD, w, L, (cudaStream_t)stream);
}

int vqc_adjoint(VqcPlan* p, const double* d_in, const double* d_w, int64_t B, const double* d_up,
                double* d_expect, double* d_jac, double* d_rows, double* d_sum, void* ws, size_t ws_bytes,
                void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_common(p, d_in, d_w, B);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const HostProgram& P = p->prog;
  const int mode = d_up ? VQC_MODE_VJP : VQC_MODE_JACOBIAN;
  if (mode == VQC_MODE_JACOBIAN && !d_jac && P.n_cols > 0 && p->M > 0)
    return fail(VQC_E_INVALID, "Jacobian mode needs d_jac");
  // degenerate shapes (batch.py:464-468)
  if (B == 0) {
    if (d_sum && P.n_cols > 0) {
      cudaError_t e = cudaMemsetAsync(d_sum, 0, (size_t)P.n_cols * 8, st);
      if (e != cudaSuccess) return cuda_fail(e, "memset");
    }
    return VQC_OK;
  }
  if (p->M == 0 || P.n_cols == 0 || P.NG == 0) {
    cudaError_t e = cudaSuccess;
    if (d_jac && P.n_cols > 0 && p->M > 0) e = cudaMemsetAsync(d_jac, 0, (size_t)B * p->M * P.n_cols * 8, st);
    if (e == cudaSuccess && d_rows && P.n_cols > 0) e = cudaMemsetAsync(d_rows, 0, (size_t)B * P.n_cols * 8, st);
    if (e == cudaSuccess && d_sum && P.n_cols > 0) e = cudaMemsetAsync(d_sum, 0, (size_t)P.n_cols * 8, st);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
    if (p->M == 0 || !d_expect) return VQC_OK;
    const Layout L = make_layout(p, B, VQC_MODE_FORWARD);
    if (ws_bytes < L.total || !ws) return fail(VQC_E_WORKSPACE, "workspace too small");
    char* w = reinterpret_cast<char*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    return run_core(p, d_in, d_w, B, nullptr, d_expect, VQC_MODE_FORWARD, w, L, st);
  }
  const Layout L = make_layout(p, B, mode);
  if (ws_bytes < L.total || !ws) return fail(VQC_E_WORKSPACE, "workspace too small");
  char* w = reinterpret_cast<char*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((rc = run_core(p, d_in, d_w, B, d_up, d_expect, mode, w, L, st))) return rc;
  const double* ip = reinterpret_cast<const double*>(w + L.ip);
  if (mode == VQC_MODE_JACOBIAN) return run_chain(p, d_in, d_w, ip, B, L.K, d_jac, st);
  double* rows = d_rows ? d_rows : reinterpret_cast<double*>(w + L.rows);
  if ((rc = run_chain(p, d_in, d_w, ip, B, 1, rows, st))) return rc;
  if (d_sum) {
    const dim3 block(32, 32), grid((unsigned)((P.n_cols + 31) / 32));
    ProfScope ps("batch_sum", st);
    k_batch_sum<<<grid, block, 0, st>>>(rows, B, P.n_cols, d_sum);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "batch sum");
  }
  return VQC_OK;
}

int vqc_run_batch_host(VqcPlan* p, const double* h_in, const double* h_w, int64_t B, const double* h_up,
                       double* h_expect, double* h_jac, double* h_rows, double* h_sum) {
  g_err.clear();
  if (!p) return fail(VQC_E_INVALID, "plan is NULL");
  std::lock_guard<std::mutex> lk(p->mu);
  int rc = check_common(p, h_in, h_w, B);
  if (rc) return rc;
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  if (!p->stream && (e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail(e, "stream");
  const HostProgram& P = p->prog;
  const int M = p->M, C = P.n_cols;
  const bool fwd_only = !h_up && !h_jac;
  const int mode = fwd_only ? VQC_MODE_FORWARD : (h_up ? VQC_MODE_VJP : VQC_MODE_JACOBIAN);
  const size_t in_b = (size_t)B * p->enc_size * 8, w_b = (size_t)p->total_params * 8,
               up_b = h_up ? (size_t)B * M * 8 : 0, ex_b = (size_t)B * M * 8,
               jac_b = (mode == VQC_MODE_JACOBIAN) ? (size_t)B * M * C * 8 : 0,
               rows_b = (mode == VQC_MODE_VJP) ? (size_t)B * C * 8 : 0, sum_b = (size_t)C * 8;
  const size_t ws_b = vqc_workspace_bytes(p, B, mode);
  size_t off = 0;
  auto take = [&](size_t b) { const size_t o = off; off = align_up(off + b); return o; };
  const size_t o_in = take(in_b), o_w = take(w_b), o_up = take(up_b), o_ex = take(ex_b), o_jac = take(jac_b),
               o_rows = take(rows_b), o_sum = take(sum_b), o_ws = take(ws_b);
  if (off > p->h_dev_bytes) {
    if (p->h_dev) cudaFree(p->h_dev);
    p->h_dev = nullptr;
    p->h_dev_bytes = 0;
    if ((e = cudaMalloc(&p->h_dev, off)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    p->h_dev_bytes = off;
  }
  char* d = reinterpret_cast<char*>(p->h_dev);
  cudaStream_t st = p->stream;
  if (in_b && (e = cudaMemcpyAsync(d + o_in, h_in, in_b, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D inputs");
  if (w_b && (e = cudaMemcpyAsync(d + o_w, h_w, w_b, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D weights");
  if (up_b && (e = cudaMemcpyAsync(d + o_up, h_up, up_b, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D upstream");
  double* dex = reinterpret_cast<double*>(d + o_ex);
  if (fwd_only) {
    rc = vqc_forward(p, reinterpret_cast<double*>(d + o_in), reinterpret_cast<double*>(d + o_w), B, dex,
                     d + o_ws, ws_b, st);
  } else {
    rc = vqc_adjoint(p, reinterpret_cast<double*>(d + o_in), reinterpret_cast<double*>(d + o_w), B,
                     h_up ? reinterpret_cast<double*>(d + o_up) : nullptr, dex,
                     jac_b ? reinterpret_cast<double*>(d + o_jac) : nullptr,
                     rows_b ? reinterpret_cast<double*>(d + o_rows) : nullptr,
                     mode == VQC_MODE_VJP ? reinterpret_cast<double*>(d + o_sum) : nullptr, d + o_ws, ws_b, st);
  }
  if (rc) return rc;
  if (h_expect && ex_b && (e = cudaMemcpyAsync(h_expect, dex, ex_b, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H expect");
  if (h_jac && jac_b && (e = cudaMemcpyAsync(h_jac, d + o_jac, jac_b, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H jac");
  if (h_rows && rows_b && (e = cudaMemcpyAsync(h_rows, d + o_rows, rows_b, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H rows");
  if (h_sum && mode == VQC_MODE_VJP && sum_b &&
      (e = cudaMemcpyAsync(h_sum, d + o_sum, sum_b, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H sum");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "synchronize");
  return VQC_OK;
}

}  // extern "C"
