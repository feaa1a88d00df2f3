// librcv.so — sm_100a data plane of the ReCoVer gradient commit.
//
// One primitive does all floating-point work on the path: an ordered stack
// fold of n_in input buffers into n_out output buffers (rcv_fold, see
// include/rcv.h).  The reference's three data-movement sites are all folds:
//   * Communicator.ulfm_allreduce   comm.py:191-200   left fold over contributors,
//                                                     broadcast to every member
//   * execute_microbatch `+=`       trainer.py:212,225  acc + grad
//   * commit `flat / B`             trainer.py:446     fold of one input + divide
// and the B200-only canonical commit (dyadic tree over microbatch indices) is a
// post-order fold program.  The work is HBM/NVLink-bandwidth bound (one add
// per 4-8 bytes moved), so there are no tensor cores here: the kernels are
// built around keeping enough bytes in flight.
//
// Variants (chosen per call, RCV_VARIANT_*):
//   TMA    one producer warp streams every input's tile into a shared-memory
//          ring with cp.async.bulk (UBLKCP) + mbarrier complete_tx; four
//          consumer warps run the fold out of shared memory and store with
//          128-bit STG.  Bytes in flight are set by the ring depth, not by
//          registers, so it holds HBM/NVLink busy for any n_in.
//   DIRECT 128-bit LDG with one-input-ahead prefetch and U independent vectors
//          per thread, fold in registers.
//   SCALAR one element per thread; heads/tails and misaligned views.
//
// Fold order is exact: every add is __fadd_rn/__dadd_rn in program order,
// the final scale is __fdiv_rn/__ddiv_rn (IEEE true division, like numpy).

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rcv.h"

#define RCV_VERSION 1

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library

static int set_err(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return set_err(RCV_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,    \
                     cudaGetErrorString(e_));                                 \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers

// fp32 accumulation over bf16 inputs works on 8-element vectors so that a bf16
// input vector is one 16-byte load (8 elements) like every other access
struct __align__(16) float8 {
  float4 a, b;
};
struct F8 {};  // accumulator tag: fp32, 8 elements per vector

template <typename A> struct VecT;
template <> struct VecT<float> {
  using V = float4;
  static constexpr int E = 4;  // elements per 16-byte vector
  static constexpr int OUT = 16;
  __host__ __device__ static constexpr int in_bytes(bool bf16) { return bf16 ? 8 : 16; }
};
template <> struct VecT<double> {
  using V = double2;
  static constexpr int E = 2;
  static constexpr int OUT = 16;
  __host__ __device__ static constexpr int in_bytes(bool) { return 16; }
};
template <> struct VecT<F8> {
  using V = float8;
  static constexpr int E = 8;
  static constexpr int OUT = 32;
  __host__ __device__ static constexpr int in_bytes(bool bf16) { return bf16 ? 16 : 32; }
};

__device__ __forceinline__ float4 vadd(const float4 &a, const float4 &b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y),
                     __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 vadd(const double2 &a, const double2 &b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 vcanon(const float4 &a) {
  return vadd(make_float4(0.f, 0.f, 0.f, 0.f), a);
}
__device__ __forceinline__ double2 vcanon(const double2 &a) {
  return vadd(make_double2(0.0, 0.0), a);
}
__device__ __forceinline__ float4 vdiv(const float4 &a, double d) {
  const float f = (float)d;
  return make_float4(__fdiv_rn(a.x, f), __fdiv_rn(a.y, f), __fdiv_rn(a.z, f),
                     __fdiv_rn(a.w, f));
}
__device__ __forceinline__ double2 vdiv(const double2 &a, double d) {
  return make_double2(__ddiv_rn(a.x, d), __ddiv_rn(a.y, d));
}
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float vcanon(float a) { return __fadd_rn(0.f, a); }
__device__ __forceinline__ float8 vadd(const float8 &x, const float8 &y) {
  return float8{vadd(x.a, y.a), vadd(x.b, y.b)};
}
__device__ __forceinline__ float8 vcanon(const float8 &x) { return float8{vcanon(x.a), vcanon(x.b)}; }
__device__ __forceinline__ float8 vdiv(const float8 &x, double d) {
  return float8{vdiv(x.a, d), vdiv(x.b, d)};
}
template <typename V> __device__ __forceinline__ V vzero();
template <> __device__ __forceinline__ float4 vzero<float4>() {
  return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <> __device__ __forceinline__ double2 vzero<double2>() {
  return make_double2(0.0, 0.0);
}
template <> __device__ __forceinline__ float vzero<float>() { return 0.f; }
template <> __device__ __forceinline__ float8 vzero<float8>() {
  return float8{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
}

// 4 bf16 (8 bytes) -> float4, exact widening
__device__ __forceinline__ float4 bf16x4_to_f4(uint2 raw) {
  float4 r;
  r.x = __uint_as_float(raw.x << 16);
  r.y = __uint_as_float(raw.x & 0xffff0000u);
  r.z = __uint_as_float(raw.y << 16);
  r.w = __uint_as_float(raw.y & 0xffff0000u);
  return r;
}

// load one accumulator-vector of input i from a generic (global or peer) address
template <typename A>
__device__ __forceinline__ typename VecT<A>::V ld_vec(const char *p,
                                                      bool bf16) {
  if constexpr (std::is_same<A, F8>::value) {
    if (bf16) {  // 8 bf16 in one 16-byte load
      uint4 raw;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
                   : "l"(p));
      return float8{bf16x4_to_f4(make_uint2(raw.x, raw.y)), bf16x4_to_f4(make_uint2(raw.z, raw.w))};
    }
    float8 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w)
                 : "l"(p));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.b.x), "=f"(v.b.y), "=f"(v.b.z), "=f"(v.b.w)
                 : "l"(p + 16));
    return v;
  } else if constexpr (sizeof(A) == 4) {
    if (bf16) {
      uint2 raw;
      asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                   : "=r"(raw.x), "=r"(raw.y)
                   : "l"(p));
      return bf16x4_to_f4(raw);
    }
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
  } else {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
  }
}

template <typename A>
__device__ __forceinline__ typename VecT<A>::V lds_vec(const unsigned char *p,
                                                       bool bf16) {
  if constexpr (std::is_same<A, F8>::value) {
    if (bf16) {
      const uint4 raw = *reinterpret_cast<const uint4 *>(p);
      return float8{bf16x4_to_f4(make_uint2(raw.x, raw.y)), bf16x4_to_f4(make_uint2(raw.z, raw.w))};
    }
    return float8{*reinterpret_cast<const float4 *>(p), *reinterpret_cast<const float4 *>(p + 16)};
  } else if constexpr (sizeof(A) == 4) {
    if (bf16) return bf16x4_to_f4(*reinterpret_cast<const uint2 *>(p));
    return *reinterpret_cast<const float4 *>(p);
  } else {
    return *reinterpret_cast<const double2 *>(p);
  }
}

template <typename V> __device__ __forceinline__ void st_vec(char *p, const V &v) {
  *reinterpret_cast<V *>(p) = v;
}
__device__ __forceinline__ void st_vec(char *p, const float8 &v) {
  *reinterpret_cast<float4 *>(p) = v.a;
  *reinterpret_cast<float4 *>(p + 16) = v.b;
}

// Fixed-capacity register stack.  Indices are compared against the (warp-
// uniform) stack pointer with fully unrolled predicates, so the array stays in
// registers.
template <int MAXD, typename V> struct Stack {
  V s[MAXD];
  int sp;
  __device__ __forceinline__ Stack() : sp(0) {}
  __device__ __forceinline__ void push(const V &v) {
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d == sp) s[d] = v;
    ++sp;
  }
  __device__ __forceinline__ void merge() {
#pragma unroll
    for (int d = 0; d + 1 < MAXD; ++d)
      if (d + 2 == sp) s[d] = vadd(s[d], s[d + 1]);
    --sp;
  }
};

// ---------------------------------------------------------------------------
// kernel parameters

struct FoldParams {
  const char *in[RCV_MAX_IN];
  char *out[RCV_MAX_OUT];
  uint32_t smem_off[RCV_MAX_IN];  // TMA: byte offset of input i in a stage
  uint8_t op[RCV_MAX_IN];
  uint8_t bf16[RCV_MAX_IN];
  int n_in;
  int n_out;
  unsigned long long nvec;  // accumulator vectors in this launch
  double divisor;           // 0 => no scale
  uint32_t stage_bytes;     // TMA
  int stages;               // TMA
  int vpt;                  // TMA: vectors per consumer thread per input
  // real-kill mode: skip the whole launch when a live peer has timed out
  const unsigned int *guard;  // device status word (NULL: unguarded)
  unsigned int guard_mask;    // the peers this launch reads
  // forest (ProgForest): root f is a perfect tree of height root_L[f] over
  // inputs [root_first[f], root_first[f] + 2^root_L[f]), stored to out[f]
  int n_roots;
  uint8_t root_L[8];
  uint8_t root_first[8];
  // canonical tree (ProgTree): heap-indexed nodes, id = 2^(L-level)-1+idx
  int8_t node_in[2 * RCV_MAX_IN - 1];    // input feeding the node, or -1
  uint8_t present[2 * RCV_MAX_IN - 1];   // subtree holds at least one input
  // flag gate (multi-process runtime, gate_mask != 0): before its first read
  // every CTA waits until gate_flags[r] >= gate_value for each rank bit r
  // (the producers' "partials ready" sequence, raised from peer GPUs), and
  // the last CTA to finish releases done_value into every done_out[i] (the
  // consumers' "this call's pool set is read and its slices are stored")
  const unsigned long long *gate_flags;
  unsigned long long gate_value;
  unsigned int gate_mask;
  unsigned int *gate_status;  // timeout / dead-peer bits (barrier status word)
  unsigned long long gate_timeout_ns;
  unsigned int *done_counter;  // device-local CTA count, reset by the last CTA
  unsigned long long *done_out[32];
  int n_done;
  unsigned long long done_value;
  // launched as a programmatic dependent (PDL) of the previous kernel in its
  // stream: wait for that grid's completion and memory before any access
  int pdl;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread waits until flags[r] >= value for every rank bit r of mask,
// each wait bounded by %globaltimer.  A rank already marked in *status, or
// one that times out (then marked), is not waited for; with `strict` the
// call then returns false (the caller must not read that rank's memory).
__device__ __noinline__ bool flag_wait(const unsigned long long *flags, unsigned long long value,
                                       unsigned int mask, unsigned int *status,
                                       unsigned long long timeout_ns, bool strict) {
  bool ok = true;
  for (int r = 0; r < 32; ++r) {
    if (!((mask >> r) & 1u)) continue;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
      if (v >= value) break;
      if (*(volatile unsigned int *)status & (1u << r)) {  // known dead
        ok = !strict && ok;
        break;
      }
      if (globaltimer() - t0 > timeout_ns) {
        atomicOr(status, 1u << r);
        ok = !strict && ok;
        break;
      }
    }
  }
  return ok;
}

// Every thread of the CTA calls this before its first load of a gated launch:
// thread 0 acquires the producers' ready flags; false when one of them is
// dead or timed out (then nothing may be read, but gate_done still runs).
__device__ __noinline__ bool gate_enter(const FoldParams &p) {
  __shared__ int s_ok;
  if (threadIdx.x == 0)
    s_ok = !(p.guard && (*p.guard & p.guard_mask)) &&
           flag_wait(p.gate_flags, p.gate_value, p.gate_mask, p.gate_status, p.gate_timeout_ns, true);
  __syncthreads();
  return s_ok != 0;
}

// Every thread of the CTA calls this after its last store of a gated launch:
// the CTA's stores are made visible system-wide, counted, and the last CTA of
// the grid releases the done sequence to every consumer rank.
__device__ __noinline__ void gate_done(const FoldParams &p) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(p.done_counter, 1u);
    if (prev + 1 == gridDim.x) {
      atomicExch(p.done_counter, 0u);  // ready for the next gated launch
      __threadfence_system();
      for (int i = 0; i < p.n_done; ++i)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.done_out[i]), "l"(p.done_value)
                     : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// fold programs: evaluate one accumulator-vector from a loader ld(i) -> V.
// All control flow below depends only on kernel parameters, so it is uniform
// across the grid; no thread ever diverges.

// Generic: the stack program of include/rcv.h (push; merge top two).
template <int MAXD> struct ProgStack {
  template <typename V, typename Ld, typename P = FoldParams>
  __device__ __forceinline__ static V eval(const P &p, const Ld &ld) {
    Stack<MAXD, V> st;
    for (int i = 0; i < p.n_in; ++i) {
      V x = ld(i);
      const uint8_t op = p.op[i];
      st.push((op & RCV_OP_CANON) ? vcanon(x) : x);
      const int merges = op & RCV_OP_MERGES_MASK;
      for (int m = 0; m < merges; ++m) st.merge();
    }
    return st.s[0];
  }
};

// Left fold ((x0 + x1) + x2) + ...: the reference collective's order
// (comm.py:192-196) and the accumulation `flat += grad` (trainer.py:212).
struct ProgLeft {
  template <typename V, typename Ld, typename P = FoldParams>
  __device__ __forceinline__ static V eval(const P &p, const Ld &ld) {
    V acc = ld(0);
    if (p.op[0] & RCV_OP_CANON) acc = vcanon(acc);
    for (int i = 1; i < p.n_in; ++i) acc = vadd(acc, ld(i));
    return acc;
  }
};

// Canonical dyadic tree of height L, unrolled at compile time: a node is its
// input when one feeds it, else left + right when both subtrees hold
// something, else the non-empty side (empty leaves are skipped, not zeros).
template <int L> struct ProgTree {
  template <int LEVEL, int IDX, typename V, typename Ld, typename P>
  __device__ __forceinline__ static bool node(const P &p, const Ld &ld, V &out) {
    constexpr int id = (1 << (L - LEVEL)) - 1 + IDX;
    if (!p.present[id]) return false;
    const int in = p.node_in[id];
    if (in >= 0) {
      out = ld(in);
      return true;
    }
    if constexpr (LEVEL > 0) {
      V a = vzero<V>(), b = vzero<V>();
      const bool pa = node<LEVEL - 1, 2 * IDX>(p, ld, a);
      const bool pb = node<LEVEL - 1, 2 * IDX + 1>(p, ld, b);
      out = pa ? (pb ? vadd(a, b) : a) : b;
    }
    return true;
  }
  template <typename V, typename Ld, typename P = FoldParams>
  __device__ __forceinline__ static V eval(const P &p, const Ld &ld) {
    V r = vzero<V>();
    node<L, 0>(p, ld, r);
    return r;
  }
};

// Full canonical tree: input i is leaf i of a perfect tree of height L (the
// failure-free cover, and every canonical recompute cover). Branch-free and
// straight-line: 2^L loads, 2^L - 1 adds, all indices compile-time.
template <int L> struct ProgFull {
  template <int LEVEL, int IDX, typename V, typename Ld>
  __device__ __forceinline__ static V node(const Ld &ld) {
    if constexpr (LEVEL == 0) {
      return ld(IDX);
    } else {
      const V a = node<LEVEL - 1, 2 * IDX, V>(ld);
      const V b = node<LEVEL - 1, 2 * IDX + 1, V>(ld);
      return vadd(a, b);
    }
  }
  template <typename V, typename Ld, typename P = FoldParams>
  __device__ __forceinline__ static V eval(const P &, const Ld &ld) {
    return node<L, 0, V>(ld);
  }
};

// Several disjoint perfect subtrees in one pass (a rank's local cover after
// a failure, e.g. 8 + 4 + 2 + 1 leaves): each root is stored to its own
// output, without the divisor (pre-reduce partials).
struct ProgForest {
  static constexpr bool kMulti = true;
  template <typename V, typename Ld, typename St, typename P = FoldParams>
  __device__ __forceinline__ static void run(const P &p, const Ld &ld, const St &st) {
    for (int f = 0; f < p.n_roots; ++f) {
      const int base = p.root_first[f];
      auto sub = [&](int i) { return ld(base + i); };
      V r;
      switch (p.root_L[f]) {
        case 0: r = ProgFull<0>::template node<0, 0, V>(sub); break;
        case 1: r = ProgFull<1>::template node<1, 0, V>(sub); break;
        case 2: r = ProgFull<2>::template node<2, 0, V>(sub); break;
        case 3: r = ProgFull<3>::template node<3, 0, V>(sub); break;
        case 4: r = ProgFull<4>::template node<4, 0, V>(sub); break;
        case 5: r = ProgFull<5>::template node<5, 0, V>(sub); break;
        default: r = ProgFull<6>::template node<6, 0, V>(sub); break;
      }
      st(f, r);
    }
  }
};

template <typename Prog, typename = void> struct IsMulti { static constexpr bool value = false; };
template <typename Prog> struct IsMulti<Prog, decltype(void(Prog::kMulti))> {
  static constexpr bool value = Prog::kMulti;
};

// Evaluate and store one vector position: single-result programs write the
// (scaled) result to every output, multi-root programs one root per output.
template <typename Prog, typename V, typename Ld>
__device__ __forceinline__ void emit(const FoldParams &p, const Ld &ld, unsigned long long off) {
  if constexpr (IsMulti<Prog>::value) {
    Prog::template run<V>(p, ld, [&](int j, V r) { st_vec(p.out[j] + off, r); });
  } else {
    V r = Prog::template eval<V>(p, ld);
    if (p.divisor != 0.0) r = vdiv(r, p.divisor);
    for (int j = 0; j < p.n_out; ++j) st_vec(p.out[j] + off, r);
  }
}

// ---------------------------------------------------------------------------
// DIRECT variant: 128-bit LDG straight from (local or peer) global memory

template <typename A, typename Prog, bool kGate = false>
__global__ void __launch_bounds__(256)
    fold_direct_kernel(const __grid_constant__ FoldParams p) {
  using V = typename VecT<A>::V;
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if constexpr (kGate) {
    // the loads below are L1::no_allocate, so no line of a pool slot can be
    // cached on this SM before its producer's ready flag was acquired
    if (!gate_enter(p)) {
      gate_done(p);
      return;
    }
  } else if (p.guard && (*p.guard & p.guard_mask)) {
    return;
  }
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       v < p.nvec; v += (unsigned long long)gridDim.x * blockDim.x) {
    auto ld = [&](int i) {
      const bool b = p.bf16[i];
      return ld_vec<A>(p.in[i] + v * (unsigned long long)VecT<A>::in_bytes(b), b);
    };
    emit<Prog, V>(p, ld, v * (unsigned long long)VecT<A>::OUT);
  }
  if constexpr (kGate) gate_done(p);
}

// DIRECT, two vectors per thread per iteration, for small perfect trees
// (ProgFull<L>, L <= 3: the multi-GPU combine over one partial per rank):
// every input of both vectors is loaded before the first add or store, so a
// thread keeps 2 x 2^L 16-byte loads in flight across the NVLink round trip
// instead of 2^L (the loop body's stores otherwise fence the next loads).
template <typename P> struct FullTree { static constexpr int value = -1; };
template <int L> struct FullTree<ProgFull<L>> { static constexpr int value = L; };

template <typename Prog>
__global__ void __launch_bounds__(256)
    fold_direct_pair_kernel(const __grid_constant__ FoldParams p) {
  constexpr int L = FullTree<Prog>::value;
  constexpr int NIN = 1 << L;
  if (p.guard && (*p.guard & p.guard_mask)) return;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       v < p.nvec; v += 2 * stride) {
    const unsigned long long w = v + stride;
    const bool has_w = w < p.nvec;
    float4 x[2][NIN];
#pragma unroll
    for (int i = 0; i < NIN; ++i) {
      x[0][i] = ld_vec<float>(p.in[i] + v * 16ull, false);
      x[1][i] = has_w ? ld_vec<float>(p.in[i] + w * 16ull, false) : vzero<float4>();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && !has_w) break;
      float4 r = ProgFull<L>::template node<L, 0, float4>([&](int i) { return x[u][i]; });
      if (p.divisor != 0.0) r = vdiv(r, p.divisor);
      const unsigned long long off = (u ? w : v) * 16ull;
      for (int j = 0; j < p.n_out; ++j) st_vec(p.out[j] + off, r);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA variant: cp.async.bulk producer warp + 4 consumer warps

#define TMA_CONSUMERS 128
#define TMA_THREADS (32 + TMA_CONSUMERS)

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_addr(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src,
                                         uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

template <typename A, typename Prog, bool kGate = false>
__global__ void __launch_bounds__(TMA_THREADS)
    fold_tma_kernel(const __grid_constant__ FoldParams p) {
  using V = typename VecT<A>::V;
  // returns at once unless the grid was launched as a PDL dependent
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool guarded = p.guard && (*p.guard & p.guard_mask);
  if (!kGate && guarded) return;  // uniform: before any barrier
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t *empty = full + p.stages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TMA_CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // gated launch: this thread is also the TMA producer, so its acquire of
    // the producers' ready flags, followed by a generic->async proxy fence,
    // orders every bulk copy below after the peers' partial stores
    s_skip = 0;
    if constexpr (kGate) {
      s_skip = guarded || !flag_wait(p.gate_flags, p.gate_value, p.gate_mask, p.gate_status,
                                     p.gate_timeout_ns, true);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
  __syncthreads();

  const unsigned long long tv = (unsigned long long)TMA_CONSUMERS * p.vpt;
  const unsigned long long ntiles = s_skip ? 0 : (p.nvec + tv - 1) / tv;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t phase = 0;

      for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[s], phase ^ 1);
        const unsigned long long v0 = t * tv;
        const uint32_t nv = (uint32_t)min(tv, p.nvec - v0);
        uint32_t total = 0;
        for (int i = 0; i < p.n_in; ++i) total += nv * (uint32_t)VecT<A>::in_bytes(p.bf16[i]);
        mbar_expect_tx(&full[s], total);
        unsigned char *stage = smem + (size_t)s * p.stage_bytes;
        for (int i = 0; i < p.n_in; ++i) {
          const uint32_t vb = (uint32_t)VecT<A>::in_bytes(p.bf16[i]);
          bulk_g2s(stage + p.smem_off[i], p.in[i] + v0 * vb, nv * vb, &full[s]);
        }
        if (++s == p.stages) {
          s = 0;
          phase ^= 1;
        }
      }
    }
    if constexpr (kGate) gate_done(p);
    return;
  }

  const int ctid = threadIdx.x - 32;
  int s = 0;
  uint32_t phase = 0;
  for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], phase);
    const unsigned long long v0 = t * tv;
    const uint32_t nv = (uint32_t)min(tv, p.nvec - v0);
    const unsigned char *stage = smem + (size_t)s * p.stage_bytes;
    for (int u = 0; u < p.vpt; ++u) {
      const uint32_t vi = (uint32_t)u * TMA_CONSUMERS + ctid;
      if (vi >= nv) break;
      auto ld = [&](int i) {
        const bool b = p.bf16[i];
        return lds_vec<A>(stage + p.smem_off[i] + (size_t)vi * VecT<A>::in_bytes(b), b);
      };
      emit<Prog, V>(p, ld, (v0 + vi) * (unsigned long long)VecT<A>::OUT);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == p.stages) {
      s = 0;
      phase ^= 1;
    }
  }
  if constexpr (kGate) gate_done(p);
}

// ---------------------------------------------------------------------------
// SCALAR variant (any alignment; heads, tails, misaligned views)

struct ScalarParams {
  const char *in[RCV_MAX_IN];
  char *out[RCV_MAX_OUT];
  uint8_t op[RCV_MAX_IN];
  uint8_t bf16[RCV_MAX_IN];
  int n_in;
  int n_out;
  unsigned long long numel;
  double divisor;
  const unsigned int *guard;
  unsigned int guard_mask;
};

template <typename A>
__device__ __forceinline__ A ld_scalar(const char *base, unsigned long long e,
                                       bool bf16) {
  if constexpr (sizeof(A) == 4) {
    if (bf16) {
      const uint16_t raw = *reinterpret_cast<const uint16_t *>(base + e * 2);
      return __uint_as_float(((uint32_t)raw) << 16);
    }
    return *reinterpret_cast<const float *>(base + e * 4);
  } else {
    return *reinterpret_cast<const double *>(base + e * 8);
  }
}
__device__ __forceinline__ float sadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sdiv(float a, double d) { return __fdiv_rn(a, (float)d); }
__device__ __forceinline__ double sdiv(double a, double d) { return __ddiv_rn(a, d); }

template <typename A, int MAXD>
__global__ void __launch_bounds__(256)
    fold_scalar_kernel(const __grid_constant__ ScalarParams p) {
  if (p.guard && (*p.guard & p.guard_mask)) return;
  for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       e < p.numel; e += (unsigned long long)gridDim.x * blockDim.x) {
    A s[MAXD];
    int sp = 0;
    for (int i = 0; i < p.n_in; ++i) {
      A x = ld_scalar<A>(p.in[i], e, p.bf16[i]);
      if (p.op[i] & RCV_OP_CANON) x = sadd((A)0, x);
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d == sp) s[d] = x;
      ++sp;
      const int merges = p.op[i] & RCV_OP_MERGES_MASK;
      for (int m = 0; m < merges; ++m) {
#pragma unroll
        for (int d = 0; d + 1 < MAXD; ++d)
          if (d + 2 == sp) s[d] = sadd(s[d], s[d + 1]);
        --sp;
      }
    }
    A r = p.n_in ? s[0] : (A)0;
    if (p.divisor != 0.0) r = sdiv(r, p.divisor);
    for (int j = 0; j < p.n_out; ++j)
      *reinterpret_cast<A *>(p.out[j] + e * sizeof(A)) = r;
  }
}

// ---------------------------------------------------------------------------
// small utility kernels

__global__ void compare_kernel(const uint32_t *a, const uint32_t *b,
                               unsigned long long nwords,
                               const uint8_t *ta, const uint8_t *tb, int ntail,
                               unsigned long long *count) {
  unsigned long long local = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < nwords; i += (unsigned long long)gridDim.x * blockDim.x)
    local += (a[i] != b[i]);
  if (blockIdx.x == 0 && threadIdx.x < ntail) local += (ta[threadIdx.x] != tb[threadIdx.x]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

template <typename T>
__global__ void sgd_kernel(T *params, const T *flat, unsigned long long n,
                           double b, double lr) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 8) {
      params[i] = __dsub_rn(params[i], __dmul_rn(lr, __ddiv_rn(flat[i], b)));
    } else {
      params[i] = __fsub_rn(params[i],
                            __fmul_rn((float)lr, __fdiv_rn(flat[i], (float)b)));
    }
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void unit_lanes_kernel(double *out, uint64_t base,
                                  unsigned long long n, double scale,
                                  double shift, int floor7) {
  for (unsigned long long l = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       l < n; l += (unsigned long long)gridDim.x * blockDim.x) {
    const uint64_t z = mix64(base + (uint64_t)l * 0x9E3779B97F4A7C15ull);
    double u = __dmul_rn(__ull2double_rn(z >> 11), 0x1.0p-53);
    // numpy evaluates `u * scale + shift` as two roundings
    u = __dadd_rn(__dmul_rn(u, scale), shift);
    if (floor7) u = __dsub_rn(floor(__dmul_rn(u, 7.0)), 3.0);
    out[l] = u;
  }
}

// Fixed-order dot products over many blocks: block b owns a contiguous chunk,
// thread t folds the chunk's elements t, t+TOY_T, ... in order, the block
// folds its threads in a fixed tree, and one thread folds the block partials
// in block order.  Deterministic for a given dim; not numpy's ddot order, so
// the linear toy model is compared within tolerance (the constant model's
// integer data is exact either way).
#define TOY_T 256
#define TOY_MAXB 512
__global__ void toy_dot_partial_kernel(int linear, const double *params,
                                       const double *lanes, const double *wstar,
                                       unsigned long long dim, unsigned long long chunk,
                                       double *part) {
  __shared__ double sp_s[TOY_T], sw_s[TOY_T];
  const unsigned long long lo = blockIdx.x * chunk;
  const unsigned long long hi = min(dim, lo + chunk);
  double sp = 0.0, sw = 0.0;
  for (unsigned long long i = lo + threadIdx.x; i < hi; i += TOY_T) {
    sp = __dadd_rn(sp, __dmul_rn(params[i], lanes[i]));
    if (linear) sw = __dadd_rn(sw, __dmul_rn(wstar[i], lanes[i]));
  }
  sp_s[threadIdx.x] = sp;
  sw_s[threadIdx.x] = sw;
  __syncthreads();
  for (int w = TOY_T / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sp_s[threadIdx.x] = __dadd_rn(sp_s[threadIdx.x], sp_s[threadIdx.x + w]);
      sw_s[threadIdx.x] = __dadd_rn(sw_s[threadIdx.x], sw_s[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sp_s[0];
    part[2 * blockIdx.x + 1] = sw_s[0];
  }
}

__global__ void toy_finalize_kernel(int linear, const double *lanes, unsigned long long dim,
                                    const double *part, int nb, double *scal) {
  double tp = 0.0, tw = 0.0;
  for (int b = 0; b < nb; ++b) {
    tp = __dadd_rn(tp, part[2 * b]);
    tw = __dadd_rn(tw, part[2 * b + 1]);
  }
  if (linear) {
    const double y = __dadd_rn(tw, __dmul_rn(0.1, lanes[dim]));
    const double r = __dsub_rn(tp, y);
    scal[0] = r;               // residual
    scal[1] = __dmul_rn(r, r); // loss
  } else {
    scal[0] = 1.0;
    scal[1] = tp;
  }
}

__global__ void toy_grad_kernel(int linear, const double *lanes,
                                unsigned long long dim, const double *scal,
                                double *grad) {
  const double r = scal[0];
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < dim; i += (unsigned long long)gridDim.x * blockDim.x)
    grad[i] = linear ? __dmul_rn(r, lanes[i]) : lanes[i];
}

// ---------------------------------------------------------------------------
// cross-GPU flag barrier (multi-process mode)

struct BarrierParams {
  unsigned long long *peer[RCV_MAX_OUT];
  unsigned long long *local;
  unsigned int *status;
  unsigned long long live;
  unsigned long long value;
  unsigned long long timeout_ns;
  int n;
  int me;
  int fence;  // leading __threadfence_system (RCV_BAR_FENCE, default on)
};

__global__ void barrier_kernel(const __grid_constant__ BarrierParams p) {
  const int t = threadIdx.x;
  // a PDL-launched combine behind this barrier may start its CTAs now; they
  // block in griddepcontrol.wait until this grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // a peer that already timed out is dead: never signal or wait on it again
  const unsigned int dead = *(volatile const unsigned int *)p.status;
  const bool peer = t < p.n && t != p.me && ((p.live >> t) & 1ull) && !((dead >> t) & 1u);
  // everything this GPU wrote before this kernel (partials, remote stores)
  // is made visible system-wide before the flag store releases it
  if (p.fence) __threadfence_system();
  if (peer)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.peer[t] + p.me), "l"(p.value)
                 : "memory");
  if (peer) {
    const unsigned long long t0 = globaltimer();
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.local + t) : "memory");
      if (v >= p.value) break;
      if (globaltimer() - t0 > p.timeout_ns) {
        atomicOr(p.status, 1u << (t & 31));
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

// Flag signal / wait of the gated runtime (RCV_GATE): release `signal_value`
// into every signal[i] after a system fence (so everything this GPU wrote
// before the launch is visible to the peers that acquire it), then wait until
// wait_flags[r] >= wait_value for each rank bit of wait_mask.  Dead or
// timed-out ranks are skipped and marked in the status word.
struct GateParams {
  unsigned long long *signal[32];
  int n_signal;
  unsigned long long signal_value;
  const unsigned long long *wait_flags;
  unsigned long long wait_value;
  unsigned int wait_mask;
  unsigned int *status;
  unsigned long long timeout_ns;
};

__global__ void gate_kernel(const __grid_constant__ GateParams p) {
  const int t = threadIdx.x;
  if (p.n_signal) {
    __threadfence_system();
    if (t < p.n_signal)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.signal[t]), "l"(p.signal_value)
                   : "memory");
  }
  if (p.wait_mask && t == 0)
    flag_wait(p.wait_flags, p.wait_value, p.wait_mask, p.status, p.timeout_ns, false);
  __syncthreads();
}

// ---------------------------------------------------------------------------
// fused bucket kernel (multi-process): local pre-reduce and the owner-slice
// combine in ONE launch, synchronised per owner slice by release/acquire
// flags in peer memory instead of a barrier kernel between two launches.
//
//   CTAs [0, a_ctas)   phase A: the rank's cover nodes (a forest of perfect
//                      trees over its local leaves) into its pool slots,
//                      slice by slice in owner order; the last CTA to finish
//                      slice q releases `seq` into owner q's ready[me] flag.
//   CTAs [a_ctas, ..)  phase B: acquire ready[p] >= seq from every producer
//                      p (bounded by %globaltimer), then fold this rank's
//                      slice over every node's partial (peers' over NVLink),
//                      divide, and store it into every live rank's primary.
//
// Phase-A CTAs never wait and the grid never exceeds one CTA per SM, so all
// CTAs are co-resident and the kernel cannot deadlock on its own GPU; a
// producer that stops responding times out into the status word and the
// combine is skipped (real-kill mode).

#define FUSED_T 256
#define FUSED_MAX_SLICES 32

struct FusedParams {
  // phase A
  const char *leaf[RCV_MAX_IN];
  int n_leaf;
  int n_roots;
  uint8_t root_L[8];
  uint8_t root_first[8];
  char *pool_out[8];
  // phase B
  const char *node[RCV_MAX_IN];
  int n_node;
  int8_t node_in[2 * RCV_MAX_IN - 1];
  uint8_t present[2 * RCV_MAX_IN - 1];
  char *out[FUSED_MAX_SLICES];
  int n_out;
  double divisor;
  unsigned long long slice_lo[FUSED_MAX_SLICES + 1];  // in vectors
  int n_slices;
  int my_slice;
  unsigned long long *ready_out[FUSED_MAX_SLICES];     // owner q's ready array
  unsigned long long *ready_in;
  unsigned int producers;  // rank bits this rank's combine waits for
  unsigned int guard_mask;
  int me;
  unsigned long long seq;
  unsigned int *counter;   // device-local, one per slice
  unsigned int *status;
  unsigned long long timeout_ns;
  int a_ctas;
  int tail;  // n mod 4 trailing elements, handled by scalar code
};

// coherent 16-byte load (the pool slot was written during this kernel, on
// this or another GPU): bypass L1, no read-only path
__device__ __forceinline__ float4 ld_cg_f4(const char *p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

template <typename ProgB>
__global__ void __launch_bounds__(FUSED_T, 4)
    fused_bucket_kernel(const __grid_constant__ FusedParams p) {
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < p.a_ctas) {
    // ---- phase A: local partials, slice by slice in owner order ----
    const int a = blockIdx.x;
    for (int q = 0; q < p.n_slices; ++q) {
      for (unsigned long long v = p.slice_lo[q] + (unsigned long long)a * FUSED_T + tid;
           v < p.slice_lo[q + 1]; v += (unsigned long long)p.a_ctas * FUSED_T) {
        auto ld = [&](int i) { return ld_vec<float>(p.leaf[i] + v * 16ull, false); };
        ProgForest::run<float4>(p, ld, [&](int f, float4 r) { st_vec(p.pool_out[f] + v * 16ull, r); });
      }
      if (q == p.n_slices - 1 && a == 0 && tid < p.tail) {  // ragged end: scalar
        const unsigned long long e = p.slice_lo[p.n_slices] * 4ull + tid;
        auto ld = [&](int i) { return reinterpret_cast<const float *>(p.leaf[i])[e]; };
        ProgForest::run<float>(p, ld, [&](int f, float r) {
          reinterpret_cast<float *>(p.pool_out[f])[e] = r;
        });
      }
      __threadfence_system();  // this thread's partial stores, before the count
      __syncthreads();
      if (tid == 0) {
        const unsigned int done = atomicAdd(&p.counter[q], 1u) + 1u;
        if (done == (unsigned int)p.a_ctas) {  // the slice is complete here
          p.counter[q] = 0u;                   // ready for the next call
          __threadfence_system();
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.ready_out[q] + p.me),
                       "l"(p.seq)
                       : "memory");
        }
      }
    }
    return;
  }
  // ---- phase B: this rank's slice, once every producer's partial is in ----
  if (p.my_slice < 0) return;
  __shared__ int skip;
  if (tid == 0) {
    skip = 0;
    for (int r = 0; r < 32; ++r) {
      if (!((p.producers >> r) & 1u)) continue;
      const unsigned long long t0 = globaltimer();
      unsigned long long v;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.ready_in + r) : "memory");
        if (v >= p.seq) break;
        if (*(volatile unsigned int *)p.status & p.guard_mask & (1u << r)) {  // known dead
          skip = 1;
          break;
        }
        if (globaltimer() - t0 > p.timeout_ns) {
          atomicOr(p.status, 1u << r);
          skip = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  if (skip) return;
  const int b = blockIdx.x - p.a_ctas;
  const int nb = gridDim.x - p.a_ctas;
  const int q = p.my_slice;
  for (unsigned long long v = p.slice_lo[q] + (unsigned long long)b * FUSED_T + tid;
       v < p.slice_lo[q + 1]; v += (unsigned long long)nb * FUSED_T) {
    auto ld = [&](int i) { return ld_cg_f4(p.node[i] + v * 16ull); };
    float4 r = ProgB::template eval<float4>(p, ld);
    if (p.divisor != 0.0) r = vdiv(r, p.divisor);
    for (int j = 0; j < p.n_out; ++j) st_vec(p.out[j] + v * 16ull, r);
  }
  // the bucket's ragged end (n mod 4 elements) belongs to the last slice
  if (q == p.n_slices - 1 && b == 0 && tid < p.tail) {
    const unsigned long long e = p.slice_lo[p.n_slices] * 4ull + tid;
    auto ld = [&](int i) { return __ldcg(reinterpret_cast<const float *>(p.node[i]) + e); };
    float r = ProgB::template eval<float>(p, ld);
    if (p.divisor != 0.0) r = __fdiv_rn(r, (float)p.divisor);
    for (int j = 0; j < p.n_out; ++j) reinterpret_cast<float *>(p.out[j])[e] = r;
  }
}

// ---------------------------------------------------------------------------
// host side

namespace {

struct DevInfo {
  int sms = 0;
  bool tma_attr_set[3][4] = {};
};
std::mutex g_mu;
std::vector<DevInfo> g_dev;

int dev_sms(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
  if (!g_dev[dev].sms) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_dev[dev].sms = v;
  }
  return g_dev[dev].sms;
}

int esize(int dt) { return dt == RCV_F64 ? 8 : (dt == RCV_F32 ? 4 : 2); }

struct FoldReq {
  int n_in = 0;
  const char *in[RCV_MAX_IN];
  int in_dt[RCV_MAX_IN];
  uint8_t op[RCV_MAX_IN];
  int n_out = 0;
  char *out[RCV_MAX_OUT];
  int acc_dt = RCV_F32;
  double divisor = 0.0;
  int max_ctas = 0;  // > 0: cap on the grid, so concurrent kernels share SMs
  const unsigned int *guard = nullptr;
  unsigned int guard_mask = 0;
  int tree_L = -1;  // >= 0: canonical tree tables below are valid
  int full_L = -1;  // >= 0: inputs are the 2^full_L leaves of a perfect tree
  int n_roots = 0;  // > 0: a forest of perfect trees, one output per root
  uint8_t root_L[8] = {};
  uint8_t root_first[8] = {};
  int8_t node_in[2 * RCV_MAX_IN - 1];
  uint8_t present[2 * RCV_MAX_IN - 1];
  // fp32 inputs evaluated as 8-element vectors (two 16-byte loads per input):
  // halves the per-byte cost of a branchy evaluator's control flow
  bool wide32 = false;
  bool pdl = false;  // launch as a programmatic dependent (cudaLaunchKernelEx)
  bool pair = false;  // DIRECT: two vectors per thread (small perfect trees, fp32)
  // flag gate of a single vector launch (FoldParams::gate_*), runtime only
  const unsigned long long *gate_flags = nullptr;
  unsigned long long gate_value = 0;
  unsigned int gate_mask = 0;
  unsigned int *gate_status = nullptr;
  unsigned long long gate_timeout_ns = 0;
  unsigned int *done_counter = nullptr;
  unsigned long long *done_out[32];
  int n_done = 0;
  unsigned long long done_value = 0;
};

enum { PK_STACK = 0, PK_LEFT = 1, PK_TREE = 2 };

bool is_left_fold(const FoldReq &r) {
  if (r.n_in < 1 || (r.op[0] & RCV_OP_MERGES_MASK)) return false;
  for (int i = 1; i < r.n_in; ++i)
    if (r.op[i] != 1) return false;
  return true;
}

// simulate the program on the host: validates it and returns the max depth
int program_depth(const uint8_t *ops, int n, int *max_depth) {
  int sp = 0, mx = 0;
  for (int i = 0; i < n; ++i) {
    ++sp;
    mx = std::max(mx, sp);
    const int m = ops[i] & RCV_OP_MERGES_MASK;
    if (m > sp - 1) return set_err(RCV_EINVAL, "fold program: input %d merges %d with stack depth %d", i, m, sp);
    sp -= m;
  }
  if (n > 0 && sp != 1)
    return set_err(RCV_EINVAL, "fold program leaves %d values on the stack (want 1)", sp);
  *max_depth = mx;
  return RCV_OK;
}

template <typename A, int MAXD>
int launch_scalar_t(const FoldReq &r, unsigned long long e0, unsigned long long n,
                    cudaStream_t st, int sms) {
  ScalarParams p;
  memset(&p, 0, sizeof p);
  p.n_in = r.n_in;
  p.n_out = r.n_out;
  for (int i = 0; i < r.n_in; ++i) {
    p.in[i] = r.in[i] + e0 * esize(r.in_dt[i]);
    p.op[i] = r.op[i];
    p.bf16[i] = r.in_dt[i] == RCV_BF16;
  }
  for (int j = 0; j < r.n_out; ++j) p.out[j] = r.out[j] + e0 * sizeof(A);
  p.numel = n;
  p.divisor = r.divisor;
  p.guard = r.guard;
  p.guard_mask = r.guard_mask;
  const unsigned long long blocks = std::min<unsigned long long>((n + 255) / 256, (unsigned long long)sms * 8);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  fold_scalar_kernel<A, MAXD><<<(unsigned)std::max<unsigned long long>(blocks, 1), 256, 0, st>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}

template <typename A>
int launch_scalar(const FoldReq &r, int maxd, unsigned long long e0, unsigned long long n,
                  cudaStream_t st, int sms) {
  if (n == 0) return RCV_OK;
  if (maxd <= 2) return launch_scalar_t<A, 2>(r, e0, n, st, sms);
  if (maxd <= 4) return launch_scalar_t<A, 4>(r, e0, n, st, sms);
  if (maxd <= 8) return launch_scalar_t<A, 8>(r, e0, n, st, sms);
  return set_err(RCV_ERANGE, "fold program stack depth %d exceeds 8", maxd);
}

template <typename A>
void fill_vec_params(FoldParams &p, const FoldReq &r, unsigned long long e0,
                     unsigned long long nvec) {
  memset(&p, 0, sizeof p);
  p.n_in = r.n_in;
  p.n_out = r.n_out;
  for (int i = 0; i < r.n_in; ++i) {
    p.in[i] = r.in[i] + e0 * esize(r.in_dt[i]);
    p.op[i] = r.op[i];
    p.bf16[i] = r.in_dt[i] == RCV_BF16;
  }
  for (int j = 0; j < r.n_out; ++j) p.out[j] = r.out[j] + e0 * esize(r.acc_dt);
  p.nvec = nvec;
  p.divisor = r.divisor;
  p.guard = r.guard;
  p.guard_mask = r.guard_mask;
  p.n_roots = r.n_roots;
  p.pdl = r.pdl;
  p.gate_flags = r.gate_flags;
  p.gate_value = r.gate_value;
  p.gate_mask = r.gate_mask;
  p.gate_status = r.gate_status;
  p.gate_timeout_ns = r.gate_timeout_ns;
  p.done_counter = r.done_counter;
  for (int i = 0; i < r.n_done; ++i) p.done_out[i] = r.done_out[i];
  p.n_done = r.n_done;
  p.done_value = r.done_value;
  memcpy(p.root_L, r.root_L, sizeof p.root_L);
  memcpy(p.root_first, r.root_first, sizeof p.root_first);
  if (r.tree_L >= 0) {
    const int nodes = (2 << r.tree_L) - 1;
    memcpy(p.node_in, r.node_in, nodes);
    memcpy(p.present, r.present, nodes);
  }
}

// Launch as a programmatic dependent of the previous kernel in `st` (PDL):
// the grid may be scheduled while that kernel still runs and waits for it
// in griddepcontrol.wait (FoldParams::pdl).
cudaError_t launch_pdl(void (*kern)(FoldParams), unsigned blocks, unsigned threads, size_t smem,
                       cudaStream_t st, const FoldParams &p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

// gated instantiations exist only for the combine's programs over fp32
// pool slots (canonical trees of at most 64 leaves)
template <typename A, typename Prog> struct Gatable { static constexpr bool value = false; };
template <int L> struct Gatable<float, ProgTree<L>> { static constexpr bool value = true; };
template <int L> struct Gatable<float, ProgFull<L>> { static constexpr bool value = true; };

template <typename A, typename Prog>
int launch_direct_p(const FoldReq &r, unsigned long long e0, unsigned long long nvec,
                    cudaStream_t st, int sms) {
  FoldParams p;
  fill_vec_params<A>(p, r, e0, nvec);
  const unsigned long long want = (nvec + 255) / 256;
  unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)sms * 8));
  if (r.max_ctas > 0) blocks = std::min<unsigned long long>(blocks, (unsigned long long)r.max_ctas * 4);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if constexpr (Gatable<A, Prog>::value) {
    if (r.gate_mask) {
      fold_direct_kernel<A, Prog, true><<<(unsigned)blocks, 256, 0, st>>>(p);
      CK(cudaGetLastError());
      return RCV_OK;
    }
  }
  if (r.gate_mask) return set_err(RCV_EINVAL, "gated launch of a program without a gated kernel");
  if constexpr (std::is_same<A, float>::value && FullTree<Prog>::value >= 0 &&
                FullTree<Prog>::value <= 3) {
    if (r.pair && !r.pdl) {
      // the same (SM-share-capped) grid: twice the bytes in flight per SM
      fold_direct_pair_kernel<Prog><<<(unsigned)blocks, 256, 0, st>>>(p);
      CK(cudaGetLastError());
      return RCV_OK;
    }
  }
  if (r.pdl) {
    CK(launch_pdl(fold_direct_kernel<A, Prog>, (unsigned)blocks, 256, 0, st, p));
    return RCV_OK;
  }
  fold_direct_kernel<A, Prog><<<(unsigned)blocks, 256, 0, st>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}

// TMA geometry: vectors-per-thread, stages, CTAs per SM
struct TmaGeom {
  int vpt, stages, ctas_per_sm;
  uint32_t stage_bytes;
  size_t smem;
};

template <typename A>
bool tma_geom(const FoldReq &r, TmaGeom *g) {
  uint32_t bytes_per_vec = 0;  // sum over inputs of one vector
  for (int i = 0; i < r.n_in; ++i) bytes_per_vec += VecT<A>::in_bytes(r.in_dt[i] == RCV_BF16);
  const uint32_t per_vpt = bytes_per_vec * TMA_CONSUMERS;  // stage bytes at vpt=1
  int vpt = 1;
  while (vpt < 8 && per_vpt * (vpt * 2) <= 32768) vpt *= 2;
  const uint32_t stage = per_vpt * vpt;
  const size_t budget2 = 100 * 1024, budget1 = 200 * 1024;
  int ctas = 2, stages = (int)std::min<size_t>(8, budget2 / stage);
  if (stages < 3) {
    ctas = 1;
    stages = (int)std::min<size_t>(8, budget1 / stage);
  }
  if (stages < 2) return false;
  g->vpt = vpt;
  g->stages = stages;
  g->ctas_per_sm = ctas;
  g->stage_bytes = stage;
  g->smem = (size_t)stages * stage + 2 * stages * sizeof(uint64_t);
  return true;
}

template <typename A, typename Prog>
int launch_tma_p(const FoldReq &r, const TmaGeom &g, unsigned long long e0,
                 unsigned long long nvec, cudaStream_t st, int sms) {
  FoldParams p;
  fill_vec_params<A>(p, r, e0, nvec);
  uint32_t off = 0;
  for (int i = 0; i < r.n_in; ++i) {
    p.smem_off[i] = off;
    off += (uint32_t)TMA_CONSUMERS * g.vpt * (uint32_t)VecT<A>::in_bytes(p.bf16[i]);
  }
  p.stage_bytes = g.stage_bytes;
  p.stages = g.stages;
  p.vpt = g.vpt;
  auto kern = fold_tma_kernel<A, Prog>;
  if constexpr (Gatable<A, Prog>::value) {
    if (r.gate_mask) kern = fold_tma_kernel<A, Prog, true>;
  }
  if (r.gate_mask && kern == fold_tma_kernel<A, Prog>)
    return set_err(RCV_EINVAL, "gated launch of a program without a gated kernel");
  {
    // one attribute call per (kernel, device, size): it is not free
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void *, int>, size_t>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    bool have = false;
    for (auto &e : done)
      if (e.first.first == (const void *)kern && e.first.second == dev && e.second >= g.smem) have = true;
    if (!have) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024));
      done.push_back({{(const void *)kern, dev}, 200 * 1024 + 1024});
    }
  }
  const unsigned long long tv = (unsigned long long)TMA_CONSUMERS * g.vpt;
  const unsigned long long ntiles = (nvec + tv - 1) / tv;
  unsigned long long blocks = std::max<unsigned long long>(
      1, std::min<unsigned long long>(ntiles, (unsigned long long)sms * g.ctas_per_sm));
  if (r.max_ctas > 0) blocks = std::min<unsigned long long>(blocks, (unsigned long long)r.max_ctas);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (r.pdl) {
    CK(launch_pdl(kern, (unsigned)blocks, TMA_THREADS, g.smem, st, p));
    return RCV_OK;
  }
  kern<<<(unsigned)blocks, TMA_THREADS, g.smem, st>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}

// Launch `variant` (TMA / DIRECT) of the best program policy for r.
template <typename A>
int launch_vec(const FoldReq &r, bool tma, const TmaGeom &g, int maxd,
               unsigned long long e0, unsigned long long nvec, cudaStream_t st, int sms) {
#define RCV_LAUNCH(PROG) \
  return tma ? launch_tma_p<A, PROG>(r, g, e0, nvec, st, sms) : launch_direct_p<A, PROG>(r, e0, nvec, st, sms)
  if (r.n_roots > 0) RCV_LAUNCH(ProgForest);
  if (r.full_L >= 0 && r.full_L <= 6) {
    switch (r.full_L) {
      case 0: RCV_LAUNCH(ProgFull<0>);
      case 1: RCV_LAUNCH(ProgFull<1>);
      case 2: RCV_LAUNCH(ProgFull<2>);
      case 3: RCV_LAUNCH(ProgFull<3>);
      case 4: RCV_LAUNCH(ProgFull<4>);
      case 5: RCV_LAUNCH(ProgFull<5>);
      default: RCV_LAUNCH(ProgFull<6>);
    }
  }
  static const bool tree_as_stack = getenv("RCV_TREE_EVAL") && atoi(getenv("RCV_TREE_EVAL")) == 1;
  if (r.tree_L >= 0 && r.tree_L <= 6 && !(tree_as_stack && maxd <= 8)) {
    switch (r.tree_L) {
      case 0: RCV_LAUNCH(ProgTree<0>);
      case 1: RCV_LAUNCH(ProgTree<1>);
      case 2: RCV_LAUNCH(ProgTree<2>);
      case 3: RCV_LAUNCH(ProgTree<3>);
      case 4: RCV_LAUNCH(ProgTree<4>);
      case 5: RCV_LAUNCH(ProgTree<5>);
      default: RCV_LAUNCH(ProgTree<6>);
    }
  }
  if (is_left_fold(r)) RCV_LAUNCH(ProgLeft);
  if (maxd <= 2) RCV_LAUNCH(ProgStack<2>);
  if (maxd <= 4) RCV_LAUNCH(ProgStack<4>);
  if (maxd <= 8) RCV_LAUNCH(ProgStack<8>);
#undef RCV_LAUNCH
  return set_err(RCV_ERANGE, "fold program stack depth %d exceeds 8", maxd);
}

// head elements h (< 8) after which every pointer is 16-byte aligned, or -1
int common_head(const FoldReq &r) {
  for (int h = 0; h < 8; ++h) {
    bool ok = true;
    for (int i = 0; i < r.n_in && ok; ++i)
      ok = ((uintptr_t)(r.in[i] + (size_t)h * esize(r.in_dt[i])) & 15) == 0;
    for (int j = 0; j < r.n_out && ok; ++j)
      ok = ((uintptr_t)(r.out[j] + (size_t)h * esize(r.acc_dt)) & 15) == 0;
    if (ok) return h;
  }
  return -1;
}

int run_fold(const FoldReq &r, size_t numel, int variant, cudaStream_t st, int sms) {
  if (numel == 0 || r.n_out == 0) return RCV_OK;
  int maxd = 1;
  // a forest's inputs are its roots' leaves, not a stack program
  int rc = r.n_roots > 0 ? RCV_OK : program_depth(r.op, r.n_in, &maxd);
  if (rc) return rc;
  if (r.n_in == 0) {
    for (int j = 0; j < r.n_out; ++j) CK(cudaMemsetAsync(r.out[j], 0, numel * esize(r.acc_dt), st));
    return RCV_OK;
  }
  const bool f64 = r.acc_dt == RCV_F64;
  bool wide = r.wide32 && !f64;  // fp32 over bf16 inputs: 8-element vectors (float8)
  for (int i = 0; i < r.n_in && !f64; ++i) wide |= r.in_dt[i] == RCV_BF16;
  const int E = f64 ? 2 : (wide ? 8 : 4);
  int h = variant == RCV_VARIANT_SCALAR ? -1 : common_head(r);
  if (r.n_roots > 0 && (h != 0 || (numel % (2 * E)) != 0))
    return set_err(RCV_EINVAL, "forest fold needs 16-byte aligned, vector-multiple ranges");
  if (h < 0 || (size_t)h >= numel) {
    return f64 ? launch_scalar<double>(r, maxd, 0, numel, st, sms)
               : launch_scalar<float>(r, maxd, 0, numel, st, sms);
  }
  unsigned long long nvec = (numel - h) / E;
  nvec &= ~1ull;  // even: bf16 inputs then move whole 16-byte units
  const unsigned long long body_end = h + nvec * E;
  if (h) {
    rc = f64 ? launch_scalar<double>(r, maxd, 0, h, st, sms) : launch_scalar<float>(r, maxd, 0, h, st, sms);
    if (rc) return rc;
  }
  if (nvec) {
    TmaGeom g;
    // AUTO, from measurement (profiles/r1/variant_ab.txt): the straight-line
    // perfect-tree and forest evaluators run fastest from registers with
    // LDG.128 (93% of HBM at N=1 vs 87% through the TMA ring); evaluators
    // with warp-uniform branches (ProgTree, ProgStack, ProgLeft) keep the TMA
    // ring, which decouples their loads from the control flow.
    if (variant == RCV_VARIANT_AUTO && (r.full_L >= 0 || r.n_roots > 0)) variant = RCV_VARIANT_DIRECT;
    bool use_tma = variant == RCV_VARIANT_TMA || variant == RCV_VARIANT_AUTO;
    const bool geom_ok = f64 ? tma_geom<double>(r, &g) : (wide ? tma_geom<F8>(r, &g) : tma_geom<float>(r, &g));
    if (use_tma && !geom_ok) {
      if (variant == RCV_VARIANT_TMA)
        return set_err(RCV_EINVAL, "TMA variant: %d inputs do not fit a 2-stage ring", r.n_in);
      use_tma = false;
    }
    rc = f64 ? launch_vec<double>(r, use_tma, g, maxd, h, nvec, st, sms)
             : (wide ? launch_vec<F8>(r, use_tma, g, maxd, h, nvec, st, sms)
                     : launch_vec<float>(r, use_tma, g, maxd, h, nvec, st, sms));
    if (rc) return rc;
  }
  if (body_end < numel) {
    rc = f64 ? launch_scalar<double>(r, maxd, body_end, numel - body_end, st, sms)
             : launch_scalar<float>(r, maxd, body_end, numel - body_end, st, sms);
    if (rc) return rc;
  }
  return RCV_OK;
}

// Whether run_fold issues exactly one vector launch for r over numel
// elements (no scalar head or tail): the condition for a flag-gated launch.
bool single_vec_launch(const FoldReq &r, size_t numel) {
  if (numel == 0 || r.n_in == 0 || r.n_out == 0 || r.n_roots > 0) return false;
  if (r.acc_dt != RCV_F32 || r.tree_L < 0 || r.tree_L > 6 || r.wide32) return false;  // Gatable programs
  if (getenv("RCV_TREE_EVAL") && atoi(getenv("RCV_TREE_EVAL")) == 1) return false;
  for (int i = 0; i < r.n_in; ++i)
    if (r.in_dt[i] != RCV_F32) return false;
  return common_head(r) == 0 && numel % 8 == 0;
}

// run_fold issues exactly one vector launch (any program, any dtype)
bool single_vec_launch_any(const FoldReq &r, size_t numel) {
  if (numel == 0 || r.n_in == 0 || r.n_out == 0) return false;
  const bool f64 = r.acc_dt == RCV_F64;
  bool wide = r.wide32 && !f64;
  for (int i = 0; i < r.n_in && !f64; ++i) wide |= r.in_dt[i] == RCV_BF16;
  const size_t E = f64 ? 2 : (wide ? 8 : 4);
  return common_head(r) == 0 && numel % (2 * E) == 0;
}

int check_dtype(int acc_dt, int in_dt) {
  if (acc_dt != RCV_F32 && acc_dt != RCV_F64) return set_err(RCV_EINVAL, "acc dtype %d must be F32 or F64", acc_dt);
  if (in_dt == acc_dt) return RCV_OK;
  if (in_dt == RCV_BF16 && acc_dt == RCV_F32) return RCV_OK;
  return set_err(RCV_EINVAL, "input dtype %d cannot feed accumulator dtype %d", in_dt, acc_dt);
}

int current_device_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev_sms(dev);
}

// post-order emission of the canonical tree
struct TreeBuild {
  const uint32_t *lo, *level;
  int n, cur;
  uint8_t *ops;
  int depth, max_depth;
  int last_push;
  int err;
  bool emit(uint32_t lev, uint64_t idx) {
    const uint64_t a = idx << lev, b = a + (1ull << lev);
    if (cur >= n || lo[cur] >= b) return false;
    if (lo[cur] == a && level[cur] == lev) {
      ops[cur] = 0;
      last_push = cur++;
      if (++depth > max_depth) max_depth = depth;
      return true;
    }
    if (lev == 0) {
      err = 1;
      return false;
    }
    const bool l = emit(lev - 1, 2 * idx);
    const bool rr = emit(lev - 1, 2 * idx + 1);
    if (l && rr) {
      ops[last_push] += 1;
      --depth;
    }
    return l || rr;
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *rcv_last_error(void) { return g_err.c_str(); }
unsigned long long rcv_launch_count(void) { return g_launches.load(); }
int rcv_version(void) { return RCV_VERSION; }

int rcv_device_count(int *n) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *n = c;
  return RCV_OK;
}

int rcv_enable_peer_access(int n_dev, const int *devices) {
  int prev = 0;
  CK(cudaGetDevice(&prev));
  for (int a = 0; a < n_dev; ++a) {
    for (int b = 0; b < n_dev; ++b) {
      if (a == b) continue;
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, devices[a], devices[b]));
      if (!can) return set_err(RCV_EINVAL, "device %d cannot access peer %d", devices[a], devices[b]);
      CK(cudaSetDevice(devices[a]));
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return set_err(RCV_ECUDA, "enable peer %d->%d: %s", devices[a], devices[b], cudaGetErrorString(e));
      }
    }
  }
  CK(cudaSetDevice(prev));
  return RCV_OK;
}

int rcv_fold(int n_in, const void *const *in, const uint8_t *ops,
             const int *in_dtypes, int n_out, void *const *out, int acc_dtype,
             size_t numel, double divisor, int variant, void *stream) {
  if (n_in < 0 || n_in > RCV_MAX_IN || n_out < 0 || n_out > RCV_MAX_OUT)
    return set_err(RCV_ERANGE, "n_in %d / n_out %d out of range", n_in, n_out);
  FoldReq r;
  r.n_in = n_in;
  r.n_out = n_out;
  r.acc_dt = acc_dtype;
  r.divisor = divisor;
  for (int i = 0; i < n_in; ++i) {
    int rc = check_dtype(acc_dtype, in_dtypes[i]);
    if (rc) return rc;
    r.in[i] = (const char *)in[i];
    r.in_dt[i] = in_dtypes[i];
    r.op[i] = ops[i];
  }
  if (acc_dtype != RCV_F32 && acc_dtype != RCV_F64) return check_dtype(acc_dtype, acc_dtype);
  for (int j = 0; j < n_out; ++j) r.out[j] = (char *)out[j];
  return run_fold(r, numel, variant, (cudaStream_t)stream, current_device_sms());
}

static int build_allreduce(FoldReq &r, void *const *views, int n, uint64_t contrib_mask,
                           int dtype, double divisor) {
  if (n < 1 || n > RCV_MAX_OUT) return set_err(RCV_ERANGE, "member count %d out of range", n);
  if (n < 64 && (contrib_mask >> n)) return set_err(RCV_EINVAL, "contributor mask names non-members");
  int rc = check_dtype(dtype, dtype);
  if (rc) return rc;
  r.acc_dt = dtype;
  r.divisor = divisor;
  r.n_in = 0;
  for (int i = 0; i < n; ++i) {
    if (!((contrib_mask >> i) & 1)) continue;
    r.in[r.n_in] = (const char *)views[i];
    r.in_dt[r.n_in] = dtype;
    r.op[r.n_in] = r.n_in ? 1 : 0;  // first contributor is copied, later ones added
    ++r.n_in;
  }
  r.n_out = n;
  for (int i = 0; i < n; ++i) r.out[i] = (char *)views[i];
  return RCV_OK;
}

int rcv_masked_allreduce(void *const *views, int n, uint64_t contrib_mask,
                         int dtype, size_t numel, double divisor,
                         void *stream) {
  FoldReq r;
  int rc = build_allreduce(r, views, n, contrib_mask, dtype, divisor);
  if (rc) return rc;
  return run_fold(r, numel, RCV_VARIANT_AUTO, (cudaStream_t)stream, current_device_sms());
}

int rcv_masked_allreduce_multidev(void *const *views, int n,
                                  uint64_t contrib_mask, int dtype,
                                  size_t numel, double divisor, int n_dev,
                                  const int *devices, void *const *streams) {
  if (n_dev < 1 || n_dev > 64) return set_err(RCV_ERANGE, "device count %d out of range", n_dev);
  FoldReq r;
  int rc = build_allreduce(r, views, n, contrib_mask, dtype, divisor);
  if (rc) return rc;
  if (numel == 0) return RCV_OK;
  int prev = 0;
  CK(cudaGetDevice(&prev));
  // entry: every device's stream waits for every other stream's prior work
  // (the contributors' accumulation), exit: likewise for the peers' stores.
  std::vector<cudaEvent_t> ev(n_dev);
  auto cross_order = [&]() -> int {
    for (int d = 0; d < n_dev; ++d) {
      CK(cudaSetDevice(devices[d]));
      CK(cudaEventCreateWithFlags(&ev[d], cudaEventDisableTiming));
      CK(cudaEventRecord(ev[d], (cudaStream_t)streams[d]));
    }
    for (int d = 0; d < n_dev; ++d) {
      CK(cudaSetDevice(devices[d]));
      for (int o = 0; o < n_dev; ++o)
        if (o != d) CK(cudaStreamWaitEvent((cudaStream_t)streams[d], ev[o], 0));
    }
    for (int d = 0; d < n_dev; ++d) CK(cudaEventDestroy(ev[d]));
    return RCV_OK;
  };
  rc = cross_order();
  if (rc) return rc;
  // owner slices, multiples of 8 elements (16-byte units for f32/f64 and bf16)
  const size_t unit = 8;
  const size_t units = (numel + unit - 1) / unit;
  for (int d = 0; d < n_dev; ++d) {
    const size_t a = std::min(numel, units * d / n_dev * unit);
    const size_t b = std::min(numel, units * (d + 1) / n_dev * unit);
    if (b <= a) continue;
    CK(cudaSetDevice(devices[d]));
    FoldReq s = r;
    const int es = esize(dtype);
    for (int i = 0; i < s.n_in; ++i) s.in[i] += a * es;
    for (int j = 0; j < s.n_out; ++j) s.out[j] += a * es;
    rc = run_fold(s, b - a, RCV_VARIANT_AUTO, (cudaStream_t)streams[d], dev_sms(devices[d]));
    if (rc) return rc;
  }
  rc = cross_order();
  if (rc) return rc;
  CK(cudaSetDevice(prev));
  return RCV_OK;
}

int rcv_accumulate(void *acc, const void *grad, int acc_dtype, int grad_dtype,
                   size_t numel, int first, void *stream) {
  int rc = check_dtype(acc_dtype, grad_dtype);
  if (rc) return rc;
  FoldReq r;
  r.acc_dt = acc_dtype;
  if (first) {
    r.n_in = 1;
    r.in[0] = (const char *)grad;
    r.in_dt[0] = grad_dtype;
    r.op[0] = RCV_OP_CANON;
  } else {
    r.n_in = 2;
    r.in[0] = (const char *)acc;
    r.in_dt[0] = acc_dtype;
    r.op[0] = 0;
    r.in[1] = (const char *)grad;
    r.in_dt[1] = grad_dtype;
    r.op[1] = 1;
  }
  r.n_out = 1;
  r.out[0] = (char *)acc;
  return run_fold(r, numel, RCV_VARIANT_AUTO, (cudaStream_t)stream, current_device_sms());
}

int rcv_tree_program(const uint32_t *lo, const uint32_t *level, int n_blocks,
                     uint32_t n_leaves, uint8_t *ops_out, int *max_depth) {
  if (n_blocks < 0 || n_blocks > RCV_MAX_IN) return set_err(RCV_ERANGE, "block count %d out of range", n_blocks);
  if (n_leaves < 1) return set_err(RCV_EINVAL, "n_leaves must be >= 1");
  uint32_t L = 0;
  while ((1ull << L) < n_leaves) ++L;
  for (int i = 0; i < n_blocks; ++i) {
    if (level[i] > L) return set_err(RCV_EINVAL, "block %d level %u above tree height %u", i, level[i], L);
    const uint64_t sz = 1ull << level[i];
    if (lo[i] % sz) return set_err(RCV_EINVAL, "block %d (lo %u, level %u) is not aligned", i, lo[i], level[i]);
    if ((uint64_t)lo[i] + sz > (1ull << L)) return set_err(RCV_EINVAL, "block %d exceeds the tree", i);
    if (i && (uint64_t)lo[i - 1] + (1ull << level[i - 1]) > lo[i])
      return set_err(RCV_EINVAL, "blocks %d and %d overlap or are unsorted", i - 1, i);
  }
  TreeBuild tb{lo, level, n_blocks, 0, ops_out, 0, 0, -1, 0};
  if (n_blocks) tb.emit(L, 0);
  if (tb.err || tb.cur != n_blocks) return set_err(RCV_EINVAL, "blocks do not form a canonical tree cover");
  *max_depth = tb.max_depth;
  return RCV_OK;
}

int rcv_tree_commit(const rcv_block *blocks, int n_blocks, uint32_t n_leaves,
                    int n_out, void *const *out, int acc_dtype, size_t numel,
                    double divisor, int variant, void *stream) {
  return rcv_tree_commit_at(blocks, n_blocks, n_leaves, n_out, out, acc_dtype, 0, 0,
                            numel, divisor, variant, stream);
}

}  // extern "C"

namespace {
// Validate a canonical-tree cover once and fill everything rcv_fold needs
// (stack program, heap tables, perfect-tree shortcut); pointers unshifted.
int prepare_tree(const rcv_block *blocks, int n_blocks, uint32_t n_leaves, int n_out,
                 void *const *out, int acc_dtype, double divisor, FoldReq &r);

void shift(FoldReq &r, size_t in_offset, size_t out_offset) {
  for (int i = 0; i < r.n_in; ++i) r.in[i] += in_offset * esize(r.in_dt[i]);
  for (int j = 0; j < r.n_out; ++j) r.out[j] += out_offset * esize(r.acc_dt);
}
}  // namespace

extern "C" int rcv_tree_commit_at(const rcv_block *blocks, int n_blocks, uint32_t n_leaves,
                                  int n_out, void *const *out, int acc_dtype, size_t in_offset,
                                  size_t out_offset, size_t numel, double divisor, int variant,
                                  void *stream) {
  FoldReq r;
  int rc = prepare_tree(blocks, n_blocks, n_leaves, n_out, out, acc_dtype, divisor, r);
  if (rc) return rc;
  shift(r, in_offset, out_offset);
  return run_fold(r, numel, variant, (cudaStream_t)stream, current_device_sms());
}

namespace {
int prepare_tree(const rcv_block *blocks, int n_blocks, uint32_t n_leaves, int n_out,
                 void *const *out, int acc_dtype, double divisor, FoldReq &r) {
  if (n_blocks < 0 || n_blocks > RCV_MAX_IN || n_out < 0 || n_out > RCV_MAX_OUT)
    return set_err(RCV_ERANGE, "block/output count out of range");
  uint32_t lo[RCV_MAX_IN], lev[RCV_MAX_IN];
  for (int i = 0; i < n_blocks; ++i) {
    lo[i] = blocks[i].lo;
    lev[i] = blocks[i].level;
  }
  r = FoldReq();
  int depth = 0;
  int rc = rcv_tree_program(lo, lev, n_blocks, n_leaves, r.op, &depth);
  if (rc) return rc;
  r.n_in = n_blocks;
  r.acc_dt = acc_dtype;
  r.divisor = divisor;
  for (int i = 0; i < n_blocks; ++i) {
    rc = check_dtype(acc_dtype, blocks[i].dtype);
    if (rc) return rc;
    r.in[i] = (const char *)blocks[i].ptr;
    r.in_dt[i] = blocks[i].dtype;
  }
  r.n_out = n_out;
  for (int j = 0; j < n_out; ++j) r.out[j] = (char *)out[j];
  uint32_t L = 0;
  while ((1ull << L) < n_leaves) ++L;
  if (L <= 6) {  // compile-time tree kernels cover up to 64 leaves
    const int nodes = (2 << L) - 1;
    memset(r.node_in, -1, sizeof r.node_in);
    memset(r.present, 0, sizeof r.present);
    for (int i = 0; i < n_blocks; ++i) {
      const int id = (1 << (L - lev[i])) - 1 + (int)(lo[i] >> lev[i]);
      r.node_in[id] = (int8_t)i;
      r.present[id] = 1;
    }
    // a node is present when it or any descendant is fed; ids of children of
    // node id are 2id+1, 2id+2, so sweep from the leaves upward
    for (int id = nodes - 1; id > 0; --id)
      if (r.present[id]) r.present[(id - 1) / 2] = 1;
    r.tree_L = (int)L;
    // all blocks at one level, all present, in order: a perfect tree of
    // height L - level over the inputs themselves
    bool full = n_blocks > 0 && (n_blocks & (n_blocks - 1)) == 0;
    for (int i = 0; i < n_blocks && full; ++i)
      full = lev[i] == lev[0] && lo[i] == ((uint32_t)i << lev[0]);
    if (full && ((uint32_t)n_blocks << lev[0]) == (1u << L)) {
      int fl = 0;
      while ((1 << fl) < n_blocks) ++fl;
      r.full_L = fl;
    }
  }
  return RCV_OK;
}
}  // namespace

extern "C" {

int rcv_ipc_export(const void *ptr, void *handle_out, size_t *offset_out) {
  void *base = nullptr;
  size_t size = 0;
  CUdeviceptr b = 0;
  // the allocation holding ptr (torch's caching allocator sub-allocates);
  // the driver symbol is resolved at run time so the library loads on hosts
  // without libcuda (the CPU build box)
  typedef CUresult (*range_fn)(CUdeviceptr *, size_t *, CUdeviceptr);
  static range_fn get_range = nullptr;
  if (!get_range) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn)
      return set_err(RCV_ECUDA, "cuMemGetAddressRange unavailable");
    get_range = (range_fn)fn;
  }
  if (get_range(&b, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return set_err(RCV_EINVAL, "ipc export: %p is not a device allocation", ptr);
  base = (void *)b;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, base));
  memcpy(handle_out, &h, sizeof h);
  *offset_out = (size_t)((const char *)ptr - (const char *)base);
  return RCV_OK;
}

// ---- cuMem VMM shareable allocations (real-kill mode) ----------------------
// Physical memory exported as a POSIX file descriptor is reference counted by
// every importer, so a peer's buffers stay mapped after the peer dies.

namespace {
struct Vmm {
  CUresult (*create)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
  CUresult (*reserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
  CUresult (*exportfd)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*importfd)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
  CUresult (*granularity)(size_t *, const CUmemAllocationProp *, CUmemAllocationGranularity_flags);
  CUresult (*release)(CUmemGenericAllocationHandle);
  bool ok = false;
};

int vmm(Vmm **out) {
  static Vmm v;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!v.ok) {
    struct { const char *name; void **fn; } t[] = {
        {"cuMemCreate", (void **)&v.create},          {"cuMemAddressReserve", (void **)&v.reserve},
        {"cuMemMap", (void **)&v.map},                {"cuMemSetAccess", (void **)&v.access},
        {"cuMemExportToShareableHandle", (void **)&v.exportfd},
        {"cuMemImportFromShareableHandle", (void **)&v.importfd},
        {"cuMemGetAllocationGranularity", (void **)&v.granularity},
        {"cuMemRelease", (void **)&v.release}};
    for (auto &e : t) {
      cudaDriverEntryPointQueryResult q;
      CK(cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !*e.fn) return set_err(RCV_ECUDA, "%s unavailable", e.name);
    }
    v.ok = true;
  }
  *out = &v;
  return RCV_OK;
}

int vmm_map(Vmm *v, CUmemGenericAllocationHandle h, size_t size, int dev, void **ptr) {
  CUdeviceptr va = 0;
  if (v->reserve(&va, size, 0, 0, 0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemAddressReserve");
  if (v->map(va, size, 0, h, 0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemMap");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  std::vector<CUmemAccessDesc> acc;
  for (int d = 0; d < n; ++d) {
    int can = d == dev;
    if (!can) cudaDeviceCanAccessPeer(&can, d, dev);
    if (!can) continue;
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = d;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc.push_back(a);
  }
  if (v->access(va, size, acc.data(), acc.size()) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemSetAccess");
  *ptr = (void *)va;
  return RCV_OK;
}
}  // namespace

int rcv_vmm_alloc(size_t bytes, void **ptr_out, size_t *size_out, int *fd_out) {
  Vmm *v = nullptr;
  int rc = vmm(&v);
  if (rc) return rc;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  if (v->granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemGetAllocationGranularity");
  const size_t size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  if (v->create(&h, size, &prop, 0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemCreate %zu", size);
  rc = vmm_map(v, h, size, dev, ptr_out);
  if (rc) return rc;
  int fd = -1;
  if (v->exportfd(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemExportToShareableHandle");
  v->release(h);  // the mapping keeps the physical memory alive
  *size_out = size;
  *fd_out = fd;
  return RCV_OK;
}

int rcv_vmm_import(int fd, size_t size, int owner_device, void **ptr_out) {
  Vmm *v = nullptr;
  int rc = vmm(&v);
  if (rc) return rc;
  CUmemGenericAllocationHandle h;
  if (v->importfd(&h, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemImportFromShareableHandle(fd %d)", fd);
  rc = vmm_map(v, h, size, owner_device, ptr_out);
  v->release(h);
  return rc;
}

int rcv_ipc_import(const void *handle, size_t offset, void **ptr_out) {
  static std::mutex mu;
  static std::vector<std::pair<std::string, void *>> opened;
  std::lock_guard<std::mutex> lk(mu);
  const std::string key((const char *)handle, sizeof(cudaIpcMemHandle_t));
  for (auto &e : opened)
    if (e.first == key) {
      *ptr_out = (char *)e.second + offset;
      return RCV_OK;
    }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void *base = nullptr;
  CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  opened.emplace_back(key, base);
  *ptr_out = (char *)base + offset;
  return RCV_OK;
}

int rcv_barrier(uint64_t *local_flags, void *const *peer_flags, int n, int me,
                uint64_t live_mask, uint64_t value, uint64_t timeout_ns,
                uint32_t *status, void *stream) {
  if (n < 1 || n > 32 || me < 0 || me >= n) return set_err(RCV_ERANGE, "barrier: n %d me %d", n, me);
  BarrierParams p;
  memset(&p, 0, sizeof p);
  for (int r = 0; r < n; ++r) p.peer[r] = (unsigned long long *)peer_flags[r];
  p.local = (unsigned long long *)local_flags;
  p.status = status;
  p.live = live_mask;
  p.value = value;
  p.timeout_ns = timeout_ns;
  p.n = n;
  p.me = me;
  p.fence = 1;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}

int rcv_copy(void *dst, const void *src, size_t bytes, void *stream) {
  if (!bytes || dst == src) return RCV_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return RCV_OK;
}

int rcv_zero(void *dst, size_t bytes, void *stream) {
  if (!bytes) return RCV_OK;
  CK(cudaMemsetAsync(dst, 0, bytes, (cudaStream_t)stream));
  return RCV_OK;
}

int rcv_compare(const void *a, const void *b, size_t bytes,
                unsigned long long *d_count, void *stream) {
  if (!bytes) return RCV_OK;
  const unsigned long long nw = bytes / 4;
  const int tail = (int)(bytes % 4);
  const int sms = current_device_sms();
  const unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>((nw + 255) / 256, (unsigned long long)sms * 8));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  compare_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t *)a, (const uint32_t *)b, nw, (const uint8_t *)a + nw * 4,
      (const uint8_t *)b + nw * 4, tail, d_count);
  CK(cudaGetLastError());
  return RCV_OK;
}

int rcv_sgd_commit(void *params, const void *flat, int dtype, size_t numel,
                   double b, double lr, void *stream) {
  if (!numel) return RCV_OK;
  const int sms = current_device_sms();
  const unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>((numel + 255) / 256, (unsigned long long)sms * 8));
  if (dtype != RCV_F64 && dtype != RCV_F32) return set_err(RCV_EINVAL, "sgd dtype %d", dtype);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (dtype == RCV_F64)
    sgd_kernel<double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((double *)params, (const double *)flat, numel, b, lr);
  else
    sgd_kernel<float><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((float *)params, (const float *)flat, numel, b, lr);
  CK(cudaGetLastError());
  return RCV_OK;
}

int rcv_unit_lanes(double *out, uint64_t base, size_t n, double scale,
                   double shift, int floor7, void *stream) {
  if (!n) return RCV_OK;
  const int sms = current_device_sms();
  const unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>((n + 255) / 256, (unsigned long long)sms * 8));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  unit_lanes_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, base, n, scale, shift, floor7);
  CK(cudaGetLastError());
  return RCV_OK;
}

int rcv_toy_grad(int kind_linear, const double *params, const double *lanes,
                 const double *wstar, size_t dim, double *grad, double *scal,
                 void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // block partials live in scal[2..]: the caller's scratch holds 2 + 2*TOY_MAXB doubles
  const unsigned long long nb = std::max<unsigned long long>(
      1, std::min<unsigned long long>(TOY_MAXB, (dim + 4095) / 4096));
  const unsigned long long chunk = (dim + nb - 1) / nb;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  toy_dot_partial_kernel<<<(unsigned)nb, TOY_T, 0, st>>>(kind_linear, params, lanes, wstar, dim,
                                                          chunk, scal + 2);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  toy_finalize_kernel<<<1, 1, 0, st>>>(kind_linear, lanes, dim, scal + 2, (int)nb, scal);
  CK(cudaGetLastError());
  if (dim && grad) {  // grad == NULL: loss only (the constant stream's x is g0)
    const int sms = current_device_sms();
    const unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>((dim + 255) / 256, (unsigned long long)sms * 8));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    toy_grad_kernel<<<(unsigned)blocks, 256, 0, st>>>(kind_linear, lanes, dim, scal, grad);
    CK(cudaGetLastError());
  }
  return RCV_OK;
}


// ---------------------------------------------------------------------------
// native per-bucket runtime (multi-process commit)

}  // extern "C"

struct TimingRec {
  int kind;
  double bytes, nin, nout;
  cudaEvent_t a, b;
};

struct rcv_ctx {
  int n_ranks = 0, me = 0, device = 0, sms = 148;
  BarrierParams bar;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_ready = nullptr, ev_arrived[3] = {nullptr, nullptr, nullptr};
  bool in_step = false;
  unsigned long long calls = 0, seq = 0;
  struct Pending {
    FoldReq req;
    size_t lo, n;
    int variant;
    unsigned long long call;  // bucket call index that combined it
    bool fused = false;       // combined by the fused kernel: complete only after a barrier
    // copy-engine all-gather (RCV_CE_GATHER): pull each peer's finished
    // slice of this bucket from its primary into ours before broadcasting
    std::vector<std::pair<const char *, std::pair<size_t, size_t>>> gather;  // src base, [a, z)
    char *dst = nullptr;
    int es = 4;
  };
  std::vector<Pending> pending;  // combined buckets awaiting the local broadcast
  // gated runtime (RCV_GATE, default on): per-call ready / done sequences in
  // the flag arrays instead of a barrier kernel between pre-reduce and combine
  bool gate = false;
  // local broadcasts on their own stream, right behind each barrier
  // (RCV_BCAST_STREAM), instead of between pre-reduces on the side stream
  bool pdl = false;  // combine launched as a PDL dependent of its barrier (RCV_PDL=1)
  cudaStream_t bstream = nullptr;
  cudaEvent_t ev_bcast = nullptr;  // bstream's tail, for a side-stream flush after it
  bool bstream_dirty = false;      // bstream holds broadcasts the side has not waited for
  unsigned int *d_gate_counter = nullptr;  // CTAs of the running gated combine
  unsigned int *d_counter = nullptr;  // fused kernel: phase-A CTAs done per slice
  unsigned long long fseq = 0;        // fused kernel: ready-flag sequence
  bool fused_in_step = false;
  bool timing = false;
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> spare_events;
  cudaEvent_t ev() {
    if (!spare_events.empty()) {
      cudaEvent_t e = spare_events.back();
      spare_events.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

struct rcv_plan {
  rcv_ctx *ctx = nullptr;
  std::vector<FoldReq> pre;
  std::vector<int> pre_count;
  bool has_forest = false;  // all pre nodes fused into one launch
  FoldReq forest;
  int forest_count = 0;
  size_t set_stride = 0;
  bool has_comb = false;
  FoldReq comb;
  int slice_q = 0, slice_nr = 1;
  std::vector<uint64_t> cum_w;  // cumulative owner-slice weights (empty: equal)
  // first element of owner slice q of a bucket of `units` 64-element units
  size_t slice_at(size_t units, int q) const {
    if (cum_w.empty()) return units * q / slice_nr * 64;
    return (size_t)((unsigned __int128)units * cum_w[q] / cum_w[slice_nr]) * 64;
  }
  bool has_bcast = false;
  FoldReq bcast;
  bool fused = false;                 // one fused kernel per bucket (RCV_FUSED)
  FusedParams ftmpl;
  void (*fkern)(FusedParams) = nullptr;
  int fgrid = 0;
  bool ce_gather = false;             // all-gather by copy engine instead of STG
  std::vector<const char *> peer_primary;  // per live rank (slice order)
  char *my_primary = nullptr;
  int variant = 0, comb_variant = 0;
  uint64_t live_mask = 0;
  bool participate = false;
  bool perfect = false;  // one cover node per live rank (the failure-free layout)
  int remote_in = 0, remote_out = 0;
};

namespace {

template <typename F>
int timed(rcv_ctx *c, cudaStream_t st, int kind, double bytes, double nin, double nout, F &&launch) {
  if (!c->timing) return launch();
  TimingRec r{kind, bytes, nin, nout, c->ev(), c->ev()};
  CK(cudaEventRecord(r.a, st));
  int rc = launch();
  CK(cudaEventRecord(r.b, st));
  c->recs.push_back(r);
  return rc;
}

int ctx_barrier(rcv_ctx *c, uint64_t live, bool participate, cudaStream_t st) {
  if (!participate || __builtin_popcountll(live) < 2) return RCV_OK;
  c->bar.live = live;
  c->bar.value = ++c->seq;
  return timed(c, st, 1, 0, 0, 0, [&]() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    barrier_kernel<<<1, 32, 0, st>>>(c->bar);
    CK(cudaGetLastError());
    return RCV_OK;
  });
}

// Broadcast the pending buckets combined at call index <= upto (all of them
// when upto < 0) from this rank's primary replica to its other replicas.
int ctx_flush(rcv_ctx *c, cudaStream_t st, long long upto) {
  while (!c->pending.empty() && (upto < 0 || (long long)c->pending.front().call <= upto)) {
    // buckets committed by the fused kernel have no per-bucket barrier: only
    // the step's closing barrier (upto < 0) proves their slices landed
    if (upto >= 0 && c->pending.front().fused) break;
    rcv_ctx::Pending e = c->pending.front();
    c->pending.erase(c->pending.begin());
    for (auto &g : e.gather) {
      const size_t a = g.second.first, z = g.second.second;
      if (z > a)
        CK(cudaMemcpyAsync(e.dst + (e.lo + a) * e.es, g.first + (e.lo + a) * e.es,
                           (z - a) * e.es, cudaMemcpyDeviceToDevice, st));
    }
    if (e.req.n_out == 0) continue;  // gather only: no other local replica
    shift(e.req, e.lo, e.lo);
    const double bytes = (double)(e.req.n_in + e.req.n_out) * e.n * esize(e.req.acc_dt);
    int rc = timed(c, st, 2, bytes, 0, 0,
                   [&]() { return run_fold(e.req, e.n, e.variant, st, c->sms); });
    if (rc) return rc;
  }
  return RCV_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// Load every kernel of this library's module on the current device.  Under
// CUDA lazy loading (the default) the first launch of a kernel may need a
// context synchronisation; if a flag-gated combine is already spinning for a
// signal that kernel is to produce, that is a deadlock (broken only by the
// wait's timeout).  So the runtime loads all of its kernels up front, once
// per device, before any gated launch.
int preload_module_kernels() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return RCV_OK;
  typedef CUresult (*GetModule)(CUmodule *, CUfunction);
  typedef CUresult (*Count)(unsigned int *, CUmodule);
  typedef CUresult (*Enum)(CUfunction *, unsigned int, CUmodule);
  typedef CUresult (*Load)(CUfunction);
  typedef CUresult (*SetAttr)(CUfunction, CUfunction_attribute, int);
  GetModule get_module = nullptr;
  SetAttr set_attr = nullptr;
  Count count = nullptr;
  Enum enumerate = nullptr;
  Load load = nullptr;
  struct {
    const char *name;
    void **fn;
  } eps[] = {{"cuFuncGetModule", (void **)&get_module},
             {"cuModuleGetFunctionCount", (void **)&count},
             {"cuModuleEnumerateFunctions", (void **)&enumerate},
             {"cuFuncLoad", (void **)&load},
             {"cuFuncSetAttribute", (void **)&set_attr}};
  for (auto &e : eps) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !*e.fn) return set_err(RCV_ECUDA, "%s unavailable", e.name);
  }
  cudaFunction_t f0 = nullptr;
  CK(cudaGetFuncBySymbol(&f0, (const void *)gate_kernel));
  CUmodule mod = nullptr;
  if (get_module(&mod, (CUfunction)f0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuFuncGetModule");
  unsigned int n = 0;
  if (count(&n, mod) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuModuleGetFunctionCount");
  std::vector<CUfunction> fs(n);
  if (n && enumerate(fs.data(), n, mod) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuModuleEnumerateFunctions");
  // Optional shared-memory carveout for every kernel (RCV_CARVEOUT=0..100).
  // Hypothesis tested: DIRECT CTAs (no smem) keep SMs in a large-L1 split
  // that blocks concurrent TMA CTAs.  Max-shared measured slower (pre-reduce
  // 44 -> 50 us, profiles/r1f/schedule_ab.txt 2.), so the default (-1)
  // leaves the driver's choice.
  const char *cv = getenv("RCV_CARVEOUT");
  const int carveout = cv ? atoi(cv) : -1;
  for (CUfunction f : fs) {
    if (load(f) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuFuncLoad");
    if (carveout >= 0 &&
        set_attr(f, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, carveout) != CUDA_SUCCESS)
      return set_err(RCV_ECUDA, "cuFuncSetAttribute(carveout)");
  }
  done.push_back(dev);
  return RCV_OK;
}

}  // namespace

extern "C" {

int rcv_ctx_create(int n_ranks, int me, uint64_t *local_flags, void *const *peer_flags,
                   uint32_t *status, uint64_t timeout_ns, rcv_ctx **out) {
  if (n_ranks < 1 || n_ranks > 32 || me < 0 || me >= n_ranks)
    return set_err(RCV_ERANGE, "ctx: n_ranks %d me %d", n_ranks, me);
  {
    const int rc = preload_module_kernels();
    if (rc) return rc;
  }
  rcv_ctx *c = new rcv_ctx();
  c->n_ranks = n_ranks;
  c->me = me;
  CK(cudaGetDevice(&c->device));
  c->sms = dev_sms(c->device);
  memset(&c->bar, 0, sizeof c->bar);
  for (int r = 0; r < n_ranks; ++r) c->bar.peer[r] = (unsigned long long *)peer_flags[r];
  c->bar.local = (unsigned long long *)local_flags;
  c->bar.status = status;
  c->bar.timeout_ns = timeout_ns;
  c->bar.n = n_ranks;
  c->bar.me = me;
  {
    const char *bf = getenv("RCV_BAR_FENCE");
    c->bar.fence = bf ? atoi(bf) : 1;
  }
  // the side stream carries the HBM-bound critical path (pre-reduce and
  // local broadcast); RCV_SIDE_PRIORITY=1 schedules its CTAs ahead of the
  // NVLink-bound combine on the caller's stream
  int lo_pri = 0, hi_pri = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  const char *sp = getenv("RCV_SIDE_PRIORITY");
  CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking,
                                  (sp && atoi(sp)) ? hi_pri : lo_pri));
  CK(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  for (int i = 0; i < 3; ++i) CK(cudaEventCreateWithFlags(&c->ev_arrived[i], cudaEventDisableTiming));
  CK(cudaMalloc(&c->d_counter, FUSED_MAX_SLICES * sizeof(unsigned int)));
  CK(cudaMemset(c->d_counter, 0, FUSED_MAX_SLICES * sizeof(unsigned int)));
  CK(cudaMalloc(&c->d_gate_counter, sizeof(unsigned int)));
  CK(cudaMemset(c->d_gate_counter, 0, sizeof(unsigned int)));
  {
    const char *g = getenv("RCV_GATE");
    const char *fz = getenv("RCV_FUSED");
    const char *ce = getenv("RCV_CE_GATHER");
    c->gate = (g ? atoi(g) != 0 : false) && !(fz && atoi(fz)) && !(ce && atoi(ce));
    const char *pd = getenv("RCV_PDL");
    c->pdl = pd ? atoi(pd) != 0 : false;  // measured neutral (schedule_ab.txt 8.)
    const char *bs = getenv("RCV_BCAST_STREAM");
    // not with the gate: gate + broadcast stream measured slower (N=4
    // failure-free 1.75 vs 1.66 ms) and hung the multi-GPU tests
    if ((bs ? atoi(bs) != 0 : true) && !c->gate && !(ce && atoi(ce)))
    {
      CK(cudaStreamCreateWithPriority(&c->bstream, cudaStreamNonBlocking, lo_pri));
      CK(cudaEventCreateWithFlags(&c->ev_bcast, cudaEventDisableTiming));
    }
  }
  *out = c;
  return RCV_OK;
}

int rcv_ctx_destroy(rcv_ctx *c) {
  if (!c) return RCV_OK;
  cudaStreamSynchronize(c->side);
  for (auto &r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->spare_events) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_main);
  cudaEventDestroy(c->ev_ready);
  for (int i = 0; i < 3; ++i) cudaEventDestroy(c->ev_arrived[i]);
  cudaFree(c->d_counter);
  cudaFree(c->d_gate_counter);
  if (c->bstream) {
    cudaStreamSynchronize(c->bstream);
    cudaStreamDestroy(c->bstream);
    cudaEventDestroy(c->ev_bcast);
  }
  cudaStreamDestroy(c->side);
  delete c;
  return RCV_OK;
}

int rcv_ctx_set_timing(rcv_ctx *c, int on) {
  c->timing = on != 0;
  return RCV_OK;
}

int rcv_ctx_timing(rcv_ctx *c, int max, int *kind, float *ms, double *bytes, double *nvl_in,
                   double *nvl_out, int *count) {
  int n = 0;
  for (auto &r : c->recs) {
    if (n < max) {
      kind[n] = r.kind;
      CK(cudaEventElapsedTime(&ms[n], r.a, r.b));
      bytes[n] = r.bytes;
      nvl_in[n] = r.nin;
      nvl_out[n] = r.nout;
      ++n;
    }
    c->spare_events.push_back(r.a);
    c->spare_events.push_back(r.b);
  }
  c->recs.clear();
  *count = n;
  return RCV_OK;
}

int rcv_ctx_finish(rcv_ctx *c, uint64_t live_mask, int participate, void *main_stream) {
  cudaStream_t st = (cudaStream_t)main_stream;
  if (c->in_step) {
    // the side stream's tail (broadcasts) joins the caller's stream
    CK(cudaEventRecord(c->ev_ready, c->side));
    CK(cudaStreamWaitEvent(st, c->ev_ready, 0));
    if (c->bstream_dirty) {
      CK(cudaEventRecord(c->ev_ready, c->bstream));
      CK(cudaStreamWaitEvent(st, c->ev_ready, 0));
      c->bstream_dirty = false;
    }
  }
  int rc = ctx_barrier(c, live_mask, participate != 0, st);
  if (rc) return rc;
  rc = ctx_flush(c, st, -1);
  if (rc) return rc;
  c->in_step = false;
  c->fused_in_step = false;
  return RCV_OK;
}

static int env_ctas(const char *name, int sms, double dflt_frac) {
  const char *v = getenv(name);
  const double f = v ? atof(v) : dflt_frac;
  if (f <= 0) return 0;                    // 0: uncapped
  if (f > 2.0) return (int)f;              // an absolute CTA count
  return std::max(1, (int)(f * sms));      // a fraction of the SMs
}

// SM shares of the two concurrent streams (profiles/r1/caps_sweep.txt): the
// NVLink-bound combine saturates the links with about a third of the SMs,
// and a full-occupancy grid of either kernel would keep the other off the
// GPU until its last wave drains.  Measured at N=4 on configs[1]: 2.95 ->
// 2.60 ms/step (failure-free 2.27 -> 1.91, degraded 3.59 -> 3.28); N=2
// neutral.  RCV_COMB_CTAS / RCV_PRE_CTAS override (0: uncapped).
constexpr double kCombShare = 0.35, kPreShare = 0.65;
// A perfect cover (one node per live rank, the failure-free layout) moves
// the fewest NVLink bytes per HBM byte of pre-reduce, so the pre-reduce sets
// the cadence and gets the larger share: 0.25 / 0.75 (N=2 failure-free
// 2.31 -> 2.21 ms; N=4 1.64-1.66 ms at 0.25-0.35, within noise;
// profiles/r1f/schedule_ab.txt).  RCV_PERFECT_SHARE sets the combine share
// of perfect covers (0: the fragmented split).
double comb_share(const rcv_plan_desc *d) {
  const bool perfect = d->n_comb > 0 && d->n_comb == d->slice_nr;
  const char *v = getenv("RCV_PERFECT_SHARE");
  const double f = v ? atof(v) : 0.25;
  if (perfect && f > 0) return f;
  const char *fr = getenv("RCV_FRAG_SHARE");  // fragmented covers (experiments)
  return fr && atof(fr) > 0 ? atof(fr) : kCombShare;
}

int rcv_plan_create(rcv_ctx *ctx, const rcv_plan_desc *d, rcv_plan **out) {
  rcv_plan *p = new rcv_plan();
  p->ctx = ctx;
  p->set_stride = d->set_stride;
  p->variant = d->variant;
  p->comb_variant = d->comb_variant;
  if (const char *cv = getenv("RCV_COMB_VARIANT")) p->comb_variant = atoi(cv);  // experiments
  p->live_mask = d->live_mask;
  p->participate = d->participate != 0;
  p->perfect = d->n_comb > 0 && d->n_comb == d->slice_nr;
  p->remote_in = d->remote_in;
  p->remote_out = d->remote_out;
  int off = 0;
  for (int i = 0; i < d->n_pre; ++i) {
    FoldReq r;
    void *dst = d->pre_out[i];
    int rc = prepare_tree(d->pre_blocks + off, d->pre_counts[i], d->pre_leaves[i], 1, &dst,
                          d->acc_dtype, 0.0, r);
    if (rc) {
      delete p;
      return rc;
    }
    r.max_ctas = env_ctas("RCV_PRE_CTAS", ctx->sms, 1.0 - comb_share(d));
    p->pre.push_back(r);
    p->pre_count.push_back(d->pre_counts[i]);
    off += d->pre_counts[i];
  }
  // several full pre-reduce nodes (each 2^level leaves, all present) fuse
  // into one forest launch; plain nodes stay separate requests
  if (d->n_pre > 1 && d->n_pre <= 8 && getenv("RCV_NO_FOREST") == nullptr) {
    bool ok = true;
    int total = 0;
    for (int i = 0; i < d->n_pre && ok; ++i) {
      ok = d->pre_counts[i] == (int)d->pre_leaves[i];
      total += d->pre_counts[i];
    }
    ok = ok && total <= RCV_MAX_IN;
    if (ok) {
      FoldReq &r = p->forest;
      int k = 0;
      for (int i = 0; i < d->n_pre; ++i) {
        int L = 0;
        while ((1 << L) < d->pre_counts[i]) ++L;
        r.root_L[i] = (uint8_t)L;
        r.root_first[i] = (uint8_t)k;
        for (int j = 0; j < d->pre_counts[i]; ++j, ++k) {
          const rcv_block &b = d->pre_blocks[k];
          int rc = check_dtype(d->acc_dtype, b.dtype);
          if (rc) {
            delete p;
            return rc;
          }
          r.in[k] = (const char *)b.ptr;
          r.in_dt[k] = b.dtype;
          r.op[k] = 0;  // unused by the forest evaluator
        }
        r.out[i] = (char *)d->pre_out[i];
      }
      r.n_in = k;
      r.n_out = d->n_pre;
      r.n_roots = d->n_pre;
      r.acc_dt = d->acc_dtype;
      r.max_ctas = env_ctas("RCV_PRE_CTAS", ctx->sms, 1.0 - comb_share(d));
      p->has_forest = true;
      p->forest_count = k;
    }
  }
  if (getenv("RCV_DEBUG")) {
    fprintf(stderr, "[rcv] rank %d plan: n_pre %d forest %d counts", ctx->me, d->n_pre, (int)p->has_forest);
    for (int i = 0; i < d->n_pre; ++i) fprintf(stderr, " %d/%u", d->pre_counts[i], d->pre_leaves[i]);
    fprintf(stderr, " | n_comb %d tree_L %d full_L %d\n", d->n_comb, p->has_comb ? p->comb.tree_L : -9,
            p->has_comb ? p->comb.full_L : -9);
  }
  p->ce_gather = getenv("RCV_CE_GATHER") && atoi(getenv("RCV_CE_GATHER")) && d->participate &&
                 d->n_comb_out > 1;
  if (p->ce_gather) {
    for (int q = 0; q < d->n_comb_out; ++q) p->peer_primary.push_back((const char *)d->comb_out[q]);
    p->my_primary = (char *)d->comb_out[d->slice_q];
  }
  if (d->n_comb > 0 && d->participate) {
    // with the copy-engine gather the combine stores only this rank's slice
    // into this rank's primary; peers pull it after the next barrier
    void *const *outs = p->ce_gather ? &d->comb_out[d->slice_q] : d->comb_out;
    const int n_outs = p->ce_gather ? 1 : d->n_comb_out;
    int rc = prepare_tree(d->comb_blocks, d->n_comb, d->n_leaves, n_outs, outs,
                          d->acc_dtype, d->divisor, p->comb);
    if (rc) {
      delete p;
      return rc;
    }
    p->comb.max_ctas = env_ctas("RCV_COMB_CTAS", ctx->sms, comb_share(d));
    {
      // RCV_WIDE_COMB: 0 off, 1 branchy trees (ProgTree: fragmented covers),
      // 2 every combine
      const char *w = getenv("RCV_WIDE_COMB");
      const int wide = w ? atoi(w) : 1;
      p->comb.wide32 = wide >= 2 || (wide == 1 && p->comb.full_L < 0);
      // RCV_PAIR: two vectors per thread for the DIRECT perfect-tree combine
      const char *pr = getenv("RCV_PAIR");
      p->comb.pair = pr ? atoi(pr) != 0 : true;
    }
    if (d->guarded) {
      // the combine reads live peers' partials: skip it once one timed out
      p->comb.guard = (const unsigned int *)ctx->bar.status;
      p->comb.guard_mask = (unsigned int)(d->live_mask & ~(1ull << ctx->me));
    }
    p->has_comb = true;
    p->slice_q = d->slice_q;
    p->slice_nr = d->slice_nr;
    if (d->slice_w) {
      uint64_t acc = 0;
      p->cum_w.push_back(0);
      for (int q = 0; q < d->slice_nr; ++q) p->cum_w.push_back(acc += d->slice_w[q]);
      if (acc == 0) {
        delete p;
        return set_err(RCV_EINVAL, "rcv_plan_create: owner-slice weights sum to 0");
      }
      // the combine's SM share follows this rank's slice (its loads and
      // stores scale with the slice; the pre-reduce keeps the rest)
      const char *ss = getenv("RCV_SLICE_SHARE");
      const double f = (ss && !atoi(ss)) ? 1.0 : (double)d->slice_w[d->slice_q] / (double)acc * d->slice_nr;
      const double share = std::min(0.7, std::max(0.1, comb_share(d) * f));
      p->comb.max_ctas = getenv("RCV_COMB_CTAS") ? p->comb.max_ctas : std::max(1, (int)(share * ctx->sms));
      const int pre_ctas = getenv("RCV_PRE_CTAS") ? -1 : std::max(1, (int)((1.0 - share) * ctx->sms));
      if (pre_ctas > 0) {
        for (auto &r : p->pre) r.max_ctas = pre_ctas;
        p->forest.max_ctas = pre_ctas;
      }
    }
  }
  // fused kernel: every local node a full perfect subtree (a forest of at
  // most 8 roots over fp32 leaves), the combine a tree of at most 64 leaves
  {
    // the caller decides from the global cover (every live rank must agree:
    // the ready flags pair launches across ranks); a rank that cannot
    // honour it fails loudly rather than desynchronising the sequence
    bool ok = d->participate && p->has_comb && d->slice_nr <= FUSED_MAX_SLICES &&
              d->n_pre <= 8 && d->acc_dtype == RCV_F32 &&
              (p->comb.full_L >= 0 || (p->comb.tree_L >= 0 && p->comb.tree_L <= 6));
    int total = 0;
    for (int i = 0; i < d->n_pre && ok; ++i) {
      ok = d->pre_counts[i] == (int)d->pre_leaves[i];
      total += d->pre_counts[i];
    }
    for (int k = 0; k < total && ok; ++k) ok = d->pre_blocks[k].dtype == RCV_F32;
    ok = ok && total <= RCV_MAX_IN;
    if (d->fused && !ok) {
      delete p;
      return set_err(RCV_EINVAL, "rcv_plan_create: fused plan requested but this rank's cover is not eligible");
    }
    if (d->fused) {
      FusedParams &f = p->ftmpl;
      memset(&f, 0, sizeof f);
      int k = 0;
      for (int i = 0; i < d->n_pre; ++i) {
        int L = 0;
        while ((1 << L) < d->pre_counts[i]) ++L;
        f.root_L[i] = (uint8_t)L;
        f.root_first[i] = (uint8_t)k;
        for (int j = 0; j < d->pre_counts[i]; ++j, ++k) f.leaf[k] = (const char *)d->pre_blocks[k].ptr;
        f.pool_out[i] = (char *)d->pre_out[i];
      }
      f.n_leaf = k;
      f.n_roots = d->n_pre;
      f.n_node = p->comb.n_in;
      for (int i = 0; i < f.n_node; ++i) f.node[i] = p->comb.in[i];
      memcpy(f.node_in, p->comb.node_in, sizeof f.node_in);
      memcpy(f.present, p->comb.present, sizeof f.present);
      f.n_out = p->comb.n_out;
      for (int j = 0; j < f.n_out; ++j) f.out[j] = p->comb.out[j];
      f.divisor = d->divisor;
      f.n_slices = d->slice_nr;
      f.my_slice = d->slice_q;
      int q = 0;
      for (int r = 0; r < 64 && q < d->slice_nr; ++r)
        if ((d->live_mask >> r) & 1ull) f.ready_out[q++] = ctx->bar.peer[r] + 64;
      f.ready_in = ctx->bar.local + 64;
      // wait for every live rank, not only those holding cover nodes: a
      // rank's ready flag also proves it finished reading this pool set
      // three calls ago, before phase A overwrites it
      f.producers = (unsigned int)d->live_mask;
      f.guard_mask = (unsigned int)d->live_mask;
      f.me = ctx->me;
      f.counter = ctx->d_counter;
      f.status = ctx->bar.status;
      f.timeout_ns = ctx->bar.timeout_ns;
      const char *fa = getenv("RCV_FUSED_A");
      const double frac = fa ? atof(fa) : 0.75;
      const int L = p->comb.full_L >= 0 ? p->comb.full_L : p->comb.tree_L;
      const bool full = p->comb.full_L >= 0;
      void (*tab_full[7])(FusedParams) = {
          fused_bucket_kernel<ProgFull<0>>, fused_bucket_kernel<ProgFull<1>>,
          fused_bucket_kernel<ProgFull<2>>, fused_bucket_kernel<ProgFull<3>>,
          fused_bucket_kernel<ProgFull<4>>, fused_bucket_kernel<ProgFull<5>>,
          fused_bucket_kernel<ProgFull<6>>};
      void (*tab_tree[7])(FusedParams) = {
          fused_bucket_kernel<ProgTree<0>>, fused_bucket_kernel<ProgTree<1>>,
          fused_bucket_kernel<ProgTree<2>>, fused_bucket_kernel<ProgTree<3>>,
          fused_bucket_kernel<ProgTree<4>>, fused_bucket_kernel<ProgTree<5>>,
          fused_bucket_kernel<ProgTree<6>>};
      p->fkern = full ? tab_full[L] : tab_tree[L];
      // every CTA co-resident (phase-B CTAs spin on flags phase-A CTAs raise)
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p->fkern, FUSED_T, 0));
      const char *fo = getenv("RCV_FUSED_OCC");
      if (fo) occ = std::min(occ, std::max(1, atoi(fo)));
      p->fgrid = ctx->sms * std::max(1, occ);
      f.a_ctas = std::max(1, std::min(p->fgrid - 1, (int)(frac * p->fgrid)));
      p->fused = true;
    }
  }
  if (d->n_bcast > 0) {
    FoldReq &r = p->bcast;
    r.n_in = 1;
    r.in[0] = (const char *)d->bcast_src;
    r.in_dt[0] = d->acc_dtype;
    r.op[0] = 0;
    r.n_out = d->n_bcast;
    for (int j = 0; j < d->n_bcast; ++j) r.out[j] = (char *)d->bcast_out[j];
    r.acc_dt = d->acc_dtype;
    r.max_ctas = env_ctas("RCV_BCAST_CTAS", ctx->sms, 0.0);
    p->has_bcast = true;
  }
  *out = p;
  return RCV_OK;
}

}  // extern "C"

namespace {

constexpr int kReadyBase = 128, kDoneBase = 160;  // flag slots (dist.FLAG_SLOTS >= 192)

int launch_gate(rcv_ctx *c, cudaStream_t st, const GateParams &g) {
  return timed(c, st, 1, 0, 0, 0, [&]() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    gate_kernel<<<1, 32, 0, st>>>(g);
    CK(cudaGetLastError());
    return RCV_OK;
  });
}

// Gated per-bucket schedule of call j (no barrier kernel, no cross-stream
// events inside the step):
//   side: broadcasts of calls <= j-3 -> pre-reduce(j) into pool set j%3 ->
//         gate: release ready = j+1 to every live rank, then acquire every
//         live rank's done >= j-1 (their combine of call j-2 has read pool
//         set (j+1)%3 and stored its slices), so the side stream runs at most
//         two calls ahead of the slowest combine
//   main: combine(j), whose CTAs acquire ready >= j+1 from every live rank
//         before the first load and whose last CTA releases done = j+1.
// A combine that cannot run as one vector launch (ragged slice) or a timed
// pass takes the explicit form: gate(wait ready) -> combine -> gate(done).
int plan_bucket_gated(rcv_plan *p, size_t lo, size_t n, cudaStream_t main, cudaStream_t side) {
  rcv_ctx *c = p->ctx;
  if (!c->in_step) {
    // leaves were produced on the caller's stream
    c->in_step = true;
    c->fused_in_step = false;
    CK(cudaEventRecord(c->ev_main, main));
    CK(cudaStreamWaitEvent(c->side, c->ev_main, 0));
  }
  const unsigned long long j = c->calls++;
  const size_t set_off = (j % 3) * p->set_stride;
  const int es = esize(p->has_comb ? p->comb.acc_dt : RCV_F32);
  int rc = RCV_OK;
  // perfect covers broadcast on their own stream behind a done-flag wait
  // (as in the barrier runtime); fragmented ones on the side stream
  const bool bstream = c->bstream && !c->timing && p->perfect;
  if (j >= 3 && !bstream) {
    if (c->bstream_dirty) {
      CK(cudaEventRecord(c->ev_bcast, c->bstream));
      CK(cudaStreamWaitEvent(side, c->ev_bcast, 0));
      c->bstream_dirty = false;
    }
    if ((rc = ctx_flush(c, side, (long long)j - 3))) return rc;
  }
  if (!p->participate) return RCV_OK;
  bool forest_done = false;
  if (p->has_forest && n % 64 == 0) {
    FoldReq r = p->forest;
    shift(r, lo, set_off);
    if (common_head(r) == 0) {
      const double bytes = (double)(p->forest_count + r.n_out) * n * esize(r.acc_dt);
      if ((rc = timed(c, side, 0, bytes, 0, 0, [&]() { return run_fold(r, n, p->variant, side, c->sms); })))
        return rc;
      forest_done = true;
    }
  }
  for (size_t i = 0; i < p->pre.size() && !forest_done; ++i) {
    FoldReq r = p->pre[i];
    shift(r, lo, set_off);
    const double bytes = (double)(p->pre_count[i] + 1) * n * esize(r.acc_dt);
    if ((rc = timed(c, side, 0, bytes, 0, 0, [&]() { return run_fold(r, n, p->variant, side, c->sms); })))
      return rc;
  }
  const unsigned int live = (unsigned int)p->live_mask;
  GateParams ready;
  memset(&ready, 0, sizeof ready);
  for (int r = 0; r < c->n_ranks; ++r)
    if ((live >> r) & 1u) ready.signal[ready.n_signal++] = c->bar.peer[r] + kReadyBase + c->me;
  ready.signal_value = j + 1;
  if (j >= 2) {
    ready.wait_flags = c->bar.local + kDoneBase;
    ready.wait_value = j - 1;
    ready.wait_mask = live;
  }
  ready.status = c->bar.status;
  ready.timeout_ns = c->bar.timeout_ns;
  if ((rc = launch_gate(c, side, ready))) return rc;

  GateParams done;
  memset(&done, 0, sizeof done);
  for (int r = 0; r < c->n_ranks; ++r)
    if ((live >> r) & 1u) done.signal[done.n_signal++] = c->bar.peer[r] + kDoneBase + c->me;
  done.signal_value = j + 1;
  done.status = c->bar.status;
  done.timeout_ns = c->bar.timeout_ns;
  size_t a = 0, z = 0;
  if (p->has_comb) {
    const size_t units = (n + 63) / 64;
    a = std::min(n, p->slice_at(units, p->slice_q));
    z = std::min(n, p->slice_at(units, p->slice_q + 1));
  }
  if (z > a) {
    FoldReq r = p->comb;
    shift(r, set_off + a, lo + a);
    const double sl = (double)(z - a) * es;
    const double local = (double)(r.n_in - p->remote_in + r.n_out - p->remote_out) * sl;
    if (!c->timing && single_vec_launch(r, z - a)) {
      r.gate_flags = c->bar.local + kReadyBase;
      r.gate_value = j + 1;
      r.gate_mask = live;
      r.gate_status = c->bar.status;
      r.gate_timeout_ns = c->bar.timeout_ns;
      r.done_counter = c->d_gate_counter;
      for (int i = 0; i < done.n_signal; ++i) r.done_out[i] = done.signal[i];
      r.n_done = done.n_signal;
      r.done_value = j + 1;
      // waiting CTAs hold their SMs: leave at least half of the GPU to the
      // pre-reduce they wait for
      const int cap = std::max(1, c->sms / 2);
      if (r.max_ctas <= 0 || r.max_ctas > cap) r.max_ctas = cap;
      rc = timed(c, main, 3, local, p->remote_in * sl, p->remote_out * sl,
                 [&]() { return run_fold(r, z - a, p->comb_variant, main, c->sms); });
      if (rc) return rc;
    } else {
      GateParams w;
      memset(&w, 0, sizeof w);
      w.wait_flags = c->bar.local + kReadyBase;
      w.wait_value = j + 1;
      w.wait_mask = live;
      w.status = c->bar.status;
      w.timeout_ns = c->bar.timeout_ns;
      if ((rc = launch_gate(c, main, w))) return rc;
      rc = timed(c, main, 3, local, p->remote_in * sl, p->remote_out * sl,
                 [&]() { return run_fold(r, z - a, p->comb_variant, main, c->sms); });
      if (rc) return rc;
      if ((rc = launch_gate(c, main, done))) return rc;
    }
  } else if ((rc = launch_gate(c, main, done))) {
    return rc;
  }
  if (bstream && j >= 1 && !c->pending.empty()) {
    // every live rank's combine of call j-1 is done: the buckets combined
    // at calls <= j-1 are complete in this rank's primary
    GateParams w;
    memset(&w, 0, sizeof w);
    w.wait_flags = c->bar.local + kDoneBase;
    w.wait_value = j;
    w.wait_mask = live;
    w.status = c->bar.status;
    w.timeout_ns = c->bar.timeout_ns;
    if ((rc = launch_gate(c, c->bstream, w))) return rc;
    if ((rc = ctx_flush(c, c->bstream, (long long)j - 1))) return rc;
    c->bstream_dirty = true;
  }
  if (p->has_bcast) {
    rcv_ctx::Pending e;
    e.req = p->bcast;
    e.lo = lo;
    e.n = n;
    e.variant = p->variant;
    e.call = j;
    c->pending.push_back(e);
  }
  return RCV_OK;
}

}  // namespace

extern "C" {

int rcv_plan_destroy(rcv_plan *p) {
  delete p;
  return RCV_OK;
}

int rcv_plan_bucket(rcv_plan *p, size_t lo, size_t n, void *main_stream) {
  if (n == 0) return RCV_OK;
  rcv_ctx *c = p->ctx;
  cudaStream_t main = (cudaStream_t)main_stream;
  // while timing launch by launch everything runs on the caller's stream, so
  // each kernel's duration is its own (no cross-stream overlap stretching it)
  cudaStream_t side = c->timing ? main : c->side;
  const int es = esize(p->has_comb ? p->comb.acc_dt : RCV_F32);
  if (p->fused) {
    // one launch: local partials and this rank's slice of the combine,
    // synchronised per owner slice by ready flags in peer memory
    c->in_step = true;
    c->fused_in_step = true;
    const unsigned long long j = c->calls++;
    const size_t set_off = (j % 3) * p->set_stride;
    FusedParams f = p->ftmpl;
    uintptr_t mis = 0;
    for (int i = 0; i < f.n_leaf; ++i) mis |= (uintptr_t)(f.leaf[i] += lo * 4);
    for (int i = 0; i < f.n_roots; ++i) mis |= (uintptr_t)(f.pool_out[i] += set_off * 4);
    for (int i = 0; i < f.n_node; ++i) mis |= (uintptr_t)(f.node[i] += set_off * 4);
    for (int i = 0; i < f.n_out; ++i) mis |= (uintptr_t)(f.out[i] += lo * 4);
    if (mis & 15)
      return set_err(RCV_EINVAL, "fused bucket: every leaf, pool slot and output must be 16-byte aligned");
    const size_t nvec = n / 4, units = (n + 63) / 64;
    for (int q = 0; q < f.n_slices; ++q) f.slice_lo[q] = std::min(n, p->slice_at(units, q)) / 4;
    f.slice_lo[f.n_slices] = nvec;
    f.tail = (int)(n % 4);
    f.seq = ++c->fseq;
    const double local = (double)(f.n_leaf + f.n_roots) * n * 4;
    int rc = timed(c, main, 4, local, p->remote_in * (double)n * 4 / f.n_slices,
                   p->remote_out * (double)n * 4 / f.n_slices, [&]() {
                     g_launches.fetch_add(1, std::memory_order_relaxed);
                     p->fkern<<<p->fgrid, FUSED_T, 0, main>>>(f);
                     CK(cudaGetLastError());
                     return RCV_OK;
                   });
    if (rc) return rc;
    if (p->has_bcast) {
      rcv_ctx::Pending e;
      e.req = p->bcast;
      e.lo = lo;
      e.n = n;
      e.variant = p->variant;
      e.call = j;
      e.fused = true;
      c->pending.push_back(e);
    }
    return RCV_OK;
  }
  if (c->gate) return plan_bucket_gated(p, lo, n, main, side);
  if (!c->in_step || c->fused_in_step) {
    // leaves were produced on the caller's stream (and, after fused
    // buckets, the pool sets they used are released only in stream order)
    c->in_step = true;
    c->fused_in_step = false;
    CK(cudaEventRecord(c->ev_main, main));
    CK(cudaStreamWaitEvent(c->side, c->ev_main, 0));
  }
  // Three pool sets: call j's pre-reduce overwrites the set last read by the
  // combine of call j-3, which every peer finished before its barrier of
  // call j-2.  So the side stream only waits for that barrier and can run
  // up to two buckets ahead of the combines; the buckets combined at calls
  // <= j-3 are then also complete in this rank's primary, and their local
  // broadcasts go here, off the main stream.
  const unsigned long long j = c->calls++;
  const size_t set_off = (j % 3) * p->set_stride;
  // perfect covers (pre-reduce-bound) broadcast on their own stream right
  // behind each barrier; fragmented ones (combine-bound) keep them on the
  // side stream, off the SMs the NVLink-bound combine needs
  // (profiles/r1f/schedule_ab.txt)
  const bool bstream = c->bstream && !c->timing && p->perfect;
  if (j >= 2) {
    CK(cudaStreamWaitEvent(side, c->ev_arrived[(j - 2) % 3], 0));
    if (j >= 3 && !bstream) {
      if (c->bstream_dirty) {
        // an earlier broadcast of the same bucket may still be on bstream
        CK(cudaEventRecord(c->ev_bcast, c->bstream));
        CK(cudaStreamWaitEvent(side, c->ev_bcast, 0));
        c->bstream_dirty = false;
      }
      int rc = ctx_flush(c, side, (long long)j - 3);
      if (rc) return rc;
    }
  }
  bool forest_done = false;
  if (p->has_forest && n % 64 == 0) {
    FoldReq r = p->forest;
    shift(r, lo, set_off);
    // the forest evaluator needs 16-byte aligned whole vectors; misaligned
    // leaves (a caller's odd tensor offsets) take the per-node launches
    if (common_head(r) == 0) {
      const double bytes = (double)(p->forest_count + r.n_out) * n * esize(r.acc_dt);
      int rc = timed(c, side, 0, bytes, 0, 0,
                     [&]() { return run_fold(r, n, p->variant, side, c->sms); });
      if (rc) return rc;
      forest_done = true;
    }
  }
  for (size_t i = 0; i < p->pre.size() && !forest_done; ++i) {
    FoldReq r = p->pre[i];
    shift(r, lo, set_off);
    const double bytes = (double)(p->pre_count[i] + 1) * n * esize(r.acc_dt);
    int rc = timed(c, side, 0, bytes, 0, 0,
                   [&]() { return run_fold(r, n, p->variant, side, c->sms); });
    if (rc) return rc;
  }
  CK(cudaEventRecord(c->ev_ready, side));
  CK(cudaStreamWaitEvent(main, c->ev_ready, 0));
  int rc = ctx_barrier(c, p->live_mask, p->participate, main);
  if (rc) return rc;
  CK(cudaEventRecord(c->ev_arrived[j % 3], main));
  if (bstream && j >= 1) {
    // passing barrier j proves every peer finished combine j-1: the buckets
    // combined at calls <= j-1 are complete in this rank's primary
    CK(cudaStreamWaitEvent(c->bstream, c->ev_arrived[j % 3], 0));
    rc = ctx_flush(c, c->bstream, (long long)j - 1);
    if (rc) return rc;
    c->bstream_dirty = true;
  }
  if (p->has_comb) {
    const size_t units = (n + 63) / 64;
    const size_t a = std::min(n, p->slice_at(units, p->slice_q));
    const size_t z = std::min(n, p->slice_at(units, p->slice_q + 1));
    if (z > a) {
      FoldReq r = p->comb;
      shift(r, set_off + a, lo + a);
      // PDL behind the barrier (RCV_PDL=1, opt-in), one vector launch
      // only: a scalar head would sit between the barrier and the body
      r.pdl = c->pdl && !c->timing && p->participate &&
              __builtin_popcountll(p->live_mask) >= 2 && single_vec_launch_any(r, z - a);
      const double sl = (double)(z - a) * es;
      const double local = (double)(r.n_in - p->remote_in + r.n_out - p->remote_out) * sl;
      rc = timed(c, main, 3, local, p->remote_in * sl, p->remote_out * sl,
                 [&]() { return run_fold(r, z - a, p->comb_variant, main, c->sms); });
      if (rc) return rc;
    }
  }
  if (p->ce_gather) {
    rcv_ctx::Pending e;
    if (p->has_bcast) e.req = p->bcast;  // else n_out stays 0: gather only
    e.lo = lo;
    e.n = n;
    e.variant = p->variant;
    e.call = j;
    e.dst = p->my_primary;
    e.es = es;
    const size_t units = (n + 63) / 64;
    for (int q = 0; q < p->slice_nr; ++q) {
      if (q == p->slice_q) continue;
      const size_t a = std::min(n, p->slice_at(units, q));
      const size_t z = std::min(n, p->slice_at(units, q + 1));
      e.gather.push_back({p->peer_primary[q], {a, z}});
    }
    c->pending.push_back(e);
  } else if (p->has_bcast) {
    rcv_ctx::Pending e;
    e.req = p->bcast;
    e.lo = lo;
    e.n = n;
    e.variant = p->variant;
    e.call = j;
    c->pending.push_back(e);
  }
  return RCV_OK;
}

}  // extern "C"
