// Device program format: what the host scheduler (scheduler.cpp) emits and
// the sm_100a kernels (kernels.cu) interpret.
//
// A state of n qubits is processed in PASSES. A pass owns a set of k "local"
// qubits: one CTA stages a tile of 2^k amplitudes (all other index bits fixed)
// in shared memory. n <= kSmemMaxQubits runs as a single pass whose tile is the
// whole state, kept on chip for the entire forward + adjoint sweep. Larger n
// stream tiles between HBM and shared memory, one kernel launch per pass.
//
// Inside a tile, work is split into SEGMENTS: each thread holds 2^R amplitudes
// in registers (R "register slots" = R local qubits) and applies every gate of
// the segment to them; a segment boundary is a shared-memory transpose. Gates
// whose mixing qubit (rotation/H/X target, CNOT target) is a register slot run
// in registers; diagonal gates (RZ, CZ) and CNOT controls may sit on any qubit
// (their effect on non-register bits is a per-thread constant).
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (jit.cpp) has no system include path: the fixed-width types it needs
typedef unsigned int uint32_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef signed char int8_t;
typedef unsigned char uint8_t;
#else
#include <stdint.h>
#endif

#ifdef __CUDACC__
#define VQC_HD __host__ __device__
#else
#define VQC_HD
#endif

namespace vqc {

constexpr int kMaxR = 5;            // register slots per thread (max)
constexpr int kMaxQubits = 24;      // statevector.py:21
constexpr int kSmemMaxQubits = 12;  // on-chip (single pass) limit
constexpr int kMaxFactors = 4;      // factors per angle expression on this path
constexpr int kMaxTile = 16;        // tile-local positions a segment's address maps cover

// gate codes (_kernels.py:16-22, CZ new)
enum GateKind : int { G_RX = 0, G_RY = 1, G_RZ = 2, G_CNOT = 3, G_H = 4, G_X = 5, G_CZ = 6 };

// op codes of the device program
enum OpCode : uint32_t {
  OP_RX = 0, OP_RY = 1, OP_RZ = 2, OP_CNOT = 3, OP_H = 4, OP_X = 5, OP_CZ = 6,
  OP_IPX = 7, OP_IPY = 8, OP_IPZ = 9,
  OP_U2 = 10,     // fused run of 1q gates on a register slot: param = block id
  OP_IP3 = 11,    // Im<phi|X|psi>, Im<phi|Y|psi>, Im<phi|Z|psi> on a slot (3 red slots)
  OP_CZRUN = 12,  // fused run of CZ gates: param = diagonal-run id
  OP_U2SET = 13,  // fused blocks on several slots: param = set id; setids[kMaxR * id + slot]
                  // is the block id relative to the pass, -1 = none
  OP_IP3SET = 14, // IP3 on the slots in operand b's mask; 3 reduction slots each from op_ip
  OP_PUBLISH = 15, // split adjoint: write this thread's registers back to shared memory so
                   // the partner thread (other state) can read them for inner products
};

// operand field (6 bits): bit 5 set -> register slot (low 3 bits), else a
// global qubit number whose bit is constant per thread.
constexpr uint32_t kSlotFlag = 32u;

// w0: [0,5) opcode | [5,11) operand a | [11,17) operand b | [17,27) local
//     reduction slot | bit 31 adjoint (rotations: negate the angle; U2: U^dagger)
struct Op {
  uint32_t w0;
  uint32_t param;  // rotation id / block id / run id
};

// shared-memory swizzle of 16-byte tile element l: l ^ fold3(l >> 3); the
// bank group (p mod 8) is the XOR of l's bits grouped by position mod 3, and
// the map is GF(2)-linear (swz(a ^ b) = swz(a) ^ swz(b)).
VQC_HD inline uint32_t swz_index(uint32_t l) {
  const uint32_t x = l >> 3;
  const uint32_t f = x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12) ^ (x >> 15) ^ (x >> 18);
  return l ^ (f & 7u);
}

VQC_HD inline uint32_t op_code(uint32_t w0) { return w0 & 31u; }
VQC_HD inline uint32_t op_a(uint32_t w0) { return (w0 >> 5) & 63u; }
VQC_HD inline uint32_t op_b(uint32_t w0) { return (w0 >> 11) & 63u; }
VQC_HD inline uint32_t op_ip(uint32_t w0) { return (w0 >> 17) & 1023u; }
VQC_HD inline bool op_adj(uint32_t w0) { return (w0 >> 31) & 1u; }

// A gradient output of a segment: ip[gslot] = red[red] (direct IP op) or
// a . (red[red], red[red+1], red[red+2]) with a = the avec table entry
// (member of a fused block).
struct IpOut {
  int32_t gslot;
  int32_t red;
  int32_t avec;  // -1: direct
};

struct SegDesc {
  int32_t op_begin, op_end;
  int32_t ip_begin, ip_count;  // IpOut entries of this segment
  int32_t red_count;           // reduction slots used
  int32_t thr_off;             // this segment's rows in the per-thread table (ThrEntry)
  // Leading / trailing CNOT runs folded into the shared-memory address maps:
  // register index bit s is stored at / loaded from the tile position whose
  // register bits are col[s] (an R-bit mask over slots) translated by the
  // slots t with parity(J0 & k[t]) = 1 (CNOTs controlled by thread/tile bits).
  uint8_t ld_col[kMaxR], st_col[kMaxR];
  uint32_t ld_k[kMaxR], st_k[kMaxR];
  // precomputed swizzled tile addresses (swz_index): ps[s] of register bit s,
  // ldc/stc[s] of the folded load/store columns, tsw[i] of thread bit i
  uint16_t ps[kMaxR], ldc[kMaxR], stc[kMaxR];
  uint16_t tsw[kMaxQubits];
  int8_t nreg, nthr, pad0, pad1;
  int8_t reg_l[kMaxR];         // tile-local bit position of each register slot
  int8_t reg_g[kMaxR];         // global qubit of each register slot
  int8_t thr_l[kMaxQubits];    // tile-local bit position of thread-index bit i
  int8_t thr_g[kMaxQubits];    // global qubit of thread-index bit i
  // General form of the folded CNOT maps: output bit of tile-local position p
  // = parity(index & row[p]) over global bits (identity: 1 << local_q[p]).
  // The register columns ldc / stc are derived from these rows. Interpreter
  // plans only fold CNOTs whose target is a register slot (ld_col / ld_k
  // describe those maps completely, gen = 0); JIT HBM plans may also fold
  // CNOTs onto thread-bit targets (gen = 1), which the JIT emits from the
  // rows (thread bases and tile translations).
  uint32_t ld_row[kMaxTile], st_row[kMaxTile];
  int8_t gen;
  // Thread-group synchronisation (scheduler.cpp assign_thread_groups; JIT HBM
  // plans): the top sync_ld / sync_st thread-index bits sit on the same tile
  // positions as in the previous / next segment of the sweep and the folded
  // maps leave them alone, so that boundary only needs a barrier over
  // blockDim >> t threads; sync_self: top bits untouched by this segment's own
  // load and store maps (the barrier between its loads and stores).
  int8_t sync_ld, sync_st, sync_self;
};

// Per (segment, thread group) precomputed addressing: thread-bit part of
// the group's global index and its swizzled load / store base addresses
// (folded CNOT translations by thread bits applied; tile bits are added by
// the kernel). Filled at plan creation (engine.cu build_thr_table).
struct ThrEntry {
  uint32_t j0, lp0, sp0, pad;
};

struct PassDesc {
  int32_t seg_begin, seg_end;    // forward segments
  int32_t bseg_begin, bseg_end;  // adjoint segments (executed in order)
  int32_t rot_begin, rot_end;    // rotation ids used by this pass (contiguous)
  int32_t blk_begin, blk_end;    // fused blocks (contiguous)
  int32_t av_begin, av_end;      // block gradient vectors (contiguous)
  int32_t k;                     // local qubits (tile = 2^k amplitudes)
  uint32_t local_mask;           // global qubits local to the tile
  int8_t local_q[kMaxQubits];    // tile-local position -> global qubit
};

// angle_r = coeff * prod flat[fidx[0..nf)]   (_kernels.py:128-134)
struct RotDesc {
  double coeff;
  int32_t nf;
  int32_t fidx[kMaxFactors];
};

// Fused block: members [mem_begin, mem_end) in forward order. U = M_last..M_first.
struct BlockDesc {
  int32_t mem_begin, mem_end;
};
// kind: G_RX/G_RY/G_RZ/G_H/G_X; rot: rotation id (rotations); avec: gradient
// vector slot (rotations with a requested factor) or -1.
struct MemberDesc {
  int32_t kind, rot, avec;
};

// Fused CZ run as a quadratic form over the index bits, split for a thread
// whose non-register bits J0 are fixed and register pattern r varies:
//   Q(J0 ^ r) = Q(J0) ^ Q(r) ^ parity(r & m(J0)),
//   Q(r)      = bit r of qreg,
//   m(J0)_s   = parity(J0 & part[s]),
//   Q(J0)     = parity(sum_{c in J0} popc(J0 & upper[c])).
struct DiagRun {
  uint32_t qreg;
  uint32_t part[kMaxR];
  uint32_t upper[kMaxQubits];
};

// chain rule (_kernels.py:269-278): column col accumulates
//   ip[gslot] * coeff * prod_{u} flat[other[u]]
struct ChainEntry {
  int32_t gslot;
  int32_t nother;
  int32_t other[kMaxFactors - 1];
  double coeff;
};

}  // namespace vqc
