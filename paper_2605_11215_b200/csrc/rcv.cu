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

#define RCV_VERSION 2

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library

extern "C" int rcv_set_error(int code, const char *msg) {
  g_err = msg;
  return code;
}

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
// fp32, 8 elements per vector moved as ONE 32-byte access (sm_100
// LDG.E.256 / STG.E.256): every pointer 32-byte aligned, fp32 inputs only.
// F8WS stores with .cs (evict-first streaming).  The straight-line DIRECT
// programs of the HBM-bound folds (the N=1 commit, the pre-reduce forests)
// run on it: tools/hbm_probe.cu measured 6.16 -> 6.7+ TB/s on the 32:8 mix.
struct F8W {};
struct F8WS {};
template <typename A> struct IsW256 { static constexpr bool value = false; };
template <> struct IsW256<F8W> { static constexpr bool value = true; };
template <> struct IsW256<F8WS> { static constexpr bool value = true; };

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
template <> struct VecT<F8W> : VecT<F8> {};
template <> struct VecT<F8WS> : VecT<F8> {};

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
  if constexpr (IsW256<A>::value) {
    float8 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y),
                   "=f"(v.b.z), "=f"(v.b.w)
                 : "l"(p));
    return v;
  } else if constexpr (std::is_same<A, F8>::value) {
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

// one 32-byte store (F8W) or one streaming 32-byte store (F8WS)
template <typename A>
__device__ __forceinline__ void st_w256(char *p, const float8 &v) {
  if constexpr (std::is_same<A, F8WS>::value) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.a.x),
                 "f"(v.a.y), "f"(v.a.z), "f"(v.a.w), "f"(v.b.x), "f"(v.b.y), "f"(v.b.z), "f"(v.b.w)
                 : "memory");
  } else {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.a.x),
                 "f"(v.a.y), "f"(v.a.z), "f"(v.a.w), "f"(v.b.x), "f"(v.b.y), "f"(v.b.z), "f"(v.b.w)
                 : "memory");
  }
}

// Stores through an NVLink SHARP multicast address (a cuMulticast object
// mapped into this context, rcv_mc_*): the switch writes the vector into the
// bound buffer of every GPU of the team, so one egress replaces n-1 peer
// stores.  PTX has no f64 vector form: double2 is two scalar stores.
__device__ __forceinline__ void st_mc(char *p, const float4 &v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_mc(char *p, const float8 &v) {
  st_mc(p, v.a);
  st_mc(p + 16, v.b);
}
__device__ __forceinline__ void st_mc(char *p, const double2 &v) {
  asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p), "d"(v.x) : "memory");
  asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p + 8), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_mc(char *p, const float &v) {
  asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
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
  uint32_t mc_mask;         // bit j: out[j] is a multicast address (st_mc)
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
};

template <typename V>
__device__ __forceinline__ void st_out(const FoldParams &p, int j, unsigned long long off, const V &v) {
  if ((p.mc_mask >> j) & 1u)
    st_mc(p.out[j] + off, v);
  else
    st_vec(p.out[j] + off, v);
}

// multicast stores alias the peers' unicast mappings of the same memory: order
// them before the stream's next barrier releases the buffers to their readers
__device__ __forceinline__ void mc_fence(const FoldParams &p) {
  if (p.mc_mask) asm volatile("fence.proxy.alias;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

// A fixed canonical-tree program known at compile time (a degraded cover of
// the multi-process combine, tools/cover_shapes.py -> shapes.inc): input i is
// pushed, then the top two stack entries merge OPS[i] times (3 bits per
// input).  Every stack index is a template constant, so the evaluation is
// straight-line code over registers, like ProgFull, instead of ProgTree's
// parameter-driven walk over 2^(L+1)-1 heap nodes.
template <int N, unsigned long long OPS> struct ProgFixed {
  template <int SP, int M, typename V>
  __device__ __forceinline__ static void merge(V (&s)[N]) {
    if constexpr (M > 0) {
      s[SP - 2] = vadd(s[SP - 2], s[SP - 1]);
      merge<SP - 1, M - 1>(s);
    }
  }
  template <int I, int SP, typename V, typename Ld>
  __device__ __forceinline__ static void push(V (&s)[N], const Ld &ld) {
    if constexpr (I < N) {
      constexpr int M = (int)((OPS >> (3 * I)) & 7ull);
      static_assert(M <= SP, "fixed program merges below the stack");
      s[SP] = ld(I);
      merge<SP + 1, M>(s);
      push<I + 1, SP + 1 - M>(s, ld);
    }
  }
  template <typename V, typename Ld, typename P = FoldParams>
  __device__ __forceinline__ static V eval(const P &, const Ld &ld) {
    V s[N];
    push<0, 0>(s, ld);
    return s[0];
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
template <typename A, typename Prog, typename V, typename Ld>
__device__ __forceinline__ void emit(const FoldParams &p, const Ld &ld, unsigned long long off) {
  if constexpr (IsW256<A>::value) {
    // 256-bit path: straight-line programs, plain (never multicast) outputs
    if constexpr (IsMulti<Prog>::value) {
      Prog::template run<V>(p, ld, [&](int j, V r) { st_w256<A>(p.out[j] + off, r); });
    } else {
      V r = Prog::template eval<V>(p, ld);
      if (p.divisor != 0.0) r = vdiv(r, p.divisor);
      for (int j = 0; j < p.n_out; ++j) st_w256<A>(p.out[j] + off, r);
    }
  } else if constexpr (IsMulti<Prog>::value) {
    Prog::template run<V>(p, ld, [&](int j, V r) { st_out(p, j, off, r); });
  } else {
    V r = Prog::template eval<V>(p, ld);
    if (p.divisor != 0.0) r = vdiv(r, p.divisor);
    // the multicast case is its own loop: the plain one keeps its registers
    if (p.mc_mask) {
      for (int j = 0; j < p.n_out; ++j) st_out(p, j, off, r);
    } else {
      for (int j = 0; j < p.n_out; ++j) st_vec(p.out[j] + off, r);
    }
  }
}

// ---------------------------------------------------------------------------
// DIRECT variant: 128-bit LDG straight from (local or peer) global memory

// programs a multicast combine may run DIRECT: the fixed degraded-cover
// programs and perfect trees over <= 8 nodes (run_fold sends any other
// multicast fold through the TMA kernel)
template <typename P> struct McDirect { static constexpr bool value = false; };
template <int L> struct McDirect<ProgFull<L>> { static constexpr bool value = L <= 3; };
template <int N, unsigned long long OPS> struct McDirect<ProgFixed<N, OPS>> {
  static constexpr bool value = true;
};

template <typename A, typename Prog>
__global__ void __launch_bounds__(256)
    fold_direct_kernel(const __grid_constant__ FoldParams p) {
  using V = typename VecT<A>::V;
  if (p.guard && (*p.guard & p.guard_mask)) return;
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       v < p.nvec; v += (unsigned long long)gridDim.x * blockDim.x) {
    auto ld = [&](int i) {
      const bool b = p.bf16[i];
      return ld_vec<A>(p.in[i] + v * (unsigned long long)VecT<A>::in_bytes(b), b);
    };
    emit<A, Prog, V>(p, ld, v * (unsigned long long)VecT<A>::OUT);
  }
  // only the programs a multicast combine runs DIRECT carry the fence: in the
  // N=1 commit's ProgFull<5> it costs 18 registers (46 -> 64)
  if constexpr (McDirect<Prog>::value) mc_fence(p);
}

// DIRECT, two vectors per thread per iteration, for small perfect trees
// (ProgFull<L>, L <= 3: the multi-GPU combine over one partial per rank):
// every input of both vectors is loaded before the first add or store, so a
// thread keeps 2 x 2^L 16-byte loads in flight across the NVLink round trip
// instead of 2^L (the loop body's stores otherwise fence the next loads).
template <typename P> struct FullTree { static constexpr int value = -1; };
template <int L> struct FullTree<ProgFull<L>> { static constexpr int value = L; };
// inputs of a straight-line program (0: not straight-line)
template <typename P> struct StraightIn { static constexpr int value = 0; };
template <int L> struct StraightIn<ProgFull<L>> { static constexpr int value = 1 << L; };
template <int N, unsigned long long OPS> struct StraightIn<ProgFixed<N, OPS>> {
  static constexpr int value = N;
};

template <typename Prog>
__global__ void __launch_bounds__(256)
    fold_direct_pair_kernel(const __grid_constant__ FoldParams p) {
  constexpr int NIN = StraightIn<Prog>::value;
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
      float4 r = Prog::template eval<float4>(p, [&](int i) { return x[u][i]; });
      if (p.divisor != 0.0) r = vdiv(r, p.divisor);
      const unsigned long long off = (u ? w : v) * 16ull;
      for (int j = 0; j < p.n_out; ++j) st_out(p, j, off, r);
    }
  }
  mc_fence(p);
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

template <typename A, typename Prog>
__global__ void __launch_bounds__(TMA_THREADS)
    fold_tma_kernel(const __grid_constant__ FoldParams p) {
  using V = typename VecT<A>::V;
  if (p.guard && (*p.guard & p.guard_mask)) return;  // uniform: before any barrier
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t *empty = full + p.stages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TMA_CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  const unsigned long long tv = (unsigned long long)TMA_CONSUMERS * p.vpt;
  const unsigned long long ntiles = (p.nvec + tv - 1) / tv;

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
      emit<A, Prog, V>(p, ld, (v0 + vi) * (unsigned long long)VecT<A>::OUT);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == p.stages) {
      s = 0;
      phase ^= 1;
    }
  }
  mc_fence(p);
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
  uint32_t mc_mask;  // bit j: out[j] is a multicast address
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
    for (int j = 0; j < p.n_out; ++j) {
      if ((p.mc_mask >> j) & 1u) {
        if constexpr (sizeof(A) == 4)
          st_mc(p.out[j] + e * sizeof(A), r);
        else
          asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(p.out[j] + e * sizeof(A)), "d"(r) : "memory");
      } else {
        *reinterpret_cast<A *>(p.out[j] + e * sizeof(A)) = r;
      }
    }
  }
  if (p.mc_mask) asm volatile("fence.proxy.alias;" ::: "memory");
}

// ---------------------------------------------------------------------------
// K-ACC: one carry-chain push of the canonical dyadic accumulator

#define KACC_MAX_SEGS 256
#define KACC_MAX_DEPTH 8

struct KaccParams {
  const char *src[KACC_MAX_SEGS];
  unsigned long long off[KACC_MAX_SEGS + 1];  // flat element offsets, off[n_seg] = numel
  const float *stack[KACC_MAX_DEPTH];         // [0] deepest merged node .. [c-1] top
  float *out;
  unsigned long long nvec;  // 4-element vectors
  int n_seg;
  int c;
  int bf16;
};

__global__ void __launch_bounds__(256) kacc_kernel(const __grid_constant__ KaccParams p) {
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       v < p.nvec; v += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long e = v * 4ull;
    // segment holding e (warp-uniform almost everywhere: a warp covers 128
    // contiguous elements and segments are whole parameter tensors)
    int lo = 0, hi = p.n_seg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const unsigned long long r = e - p.off[lo];
    float4 x = p.bf16 ? ld_vec<float>(p.src[lo] + r * 2ull, true)
                      : ld_vec<float>(p.src[lo] + r * 4ull, false);
    // canonical order: the new leaf is the right child of every node it
    // completes, so it is added on the right, innermost (top) first
    for (int i = p.c - 1; i >= 0; --i)
      // coherent load: out may alias stack[0] (the merge is in place)
      x = vadd(__ldcg(reinterpret_cast<const float4 *>(p.stack[i] + e)), x);
    // c == 0: the leaf node itself, bit for bit (a -0.0 gradient stays -0.0,
    // as in the fused commit's tree)
    *reinterpret_cast<float4 *>(p.out + e) = x;
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
  // pool-set integrity stamps (multi-process runtime): after the wait, the
  // stamps the next combine will read must equal now_value (bit 0 of *err
  // otherwise: a partial is not ready), and the stamps the previous combine
  // read must still equal prev_value (bit 1: a producer invalidated them,
  // i.e. started overwriting a partial, before that combine had finished)
  const unsigned long long *chk_now[32];
  const unsigned long long *chk_prev[32];
  unsigned long long prev_value[32];  // per entry: earlier combines read different calls' sets
  int n_now, n_prev;
  unsigned long long now_value;
  unsigned int *err;
  // this rank's own pool-set stamps (multi-process runtime): `ready` (the set
  // the pre-reduce of this call wrote) gets ready_value before the signal;
  // `inval` (the set the next overwrite targets, free once every live peer
  // passed this barrier) gets 0 after the wait.  NULL: none.
  unsigned long long *ready;
  unsigned long long ready_value;
  unsigned long long *inval;
  // real-kill mode: the node's liveness dead word (mapped host memory,
  // rcv_liveness); a peer whose bit is set is not waited for
  const volatile unsigned int *host_dead;
};

__global__ void barrier_kernel(const __grid_constant__ BarrierParams p) {
  const int t = threadIdx.x;
  // the combines listed in chk_prev have finished (the host ordered this
  // launch behind them): their producers' stamps must still be those calls'.
  // Checked before this rank signals: no producer may rewrite such a pool
  // set before it has seen this rank arrive here, so a changed stamp means a
  // real overwrite race.
  if (t < p.n_prev) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.chk_prev[t]) : "memory");
    if (v != p.prev_value[t]) atomicOr(p.err, 2u);
  }
  // a peer that already timed out is dead: never signal or wait on it again
  const unsigned int dead = *(volatile const unsigned int *)p.status | (p.host_dead ? *p.host_dead : 0u);
  const bool peer = t < p.n && t != p.me && ((p.live >> t) & 1ull) && !((dead >> t) & 1u);
  // this call's partials are complete (the host ordered this launch behind
  // the pre-reduce): stamp their set before any peer is released to read it
  if (t == 0 && p.ready) *(volatile unsigned long long *)p.ready = p.ready_value;
  __syncthreads();
  // everything this GPU wrote before this kernel (partials, remote and
  // multicast stores) is made visible system-wide before the flag store
  // releases it
  // (fence cost is not on the critical path: release/acquire-only and
  // relaxed flag accesses measured the same, gpurun_out/r2s)
  asm volatile("fence.proxy.alias;" ::: "memory");
  __threadfence_system();
  if (peer)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.peer[t] + p.me), "l"(p.value)
                 : "memory");
  if (peer) {
    const unsigned long long t0 = globaltimer();
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.local + t) : "memory");
      if (v >= p.value) break;
      if (globaltimer() - t0 > p.timeout_ns || (p.host_dead && ((*p.host_dead >> t) & 1u))) {
        atomicOr(p.status, 1u << (t & 31));
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
  asm volatile("fence.proxy.alias;" ::: "memory");
  // every live peer has arrived, so every producer finished this call's
  // partials: the stamps the combine behind this barrier reads must be set
  if (t < p.n_now) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.chk_now[t]) : "memory");
    if (v != p.now_value) atomicOr(p.err, 1u);
  }
  // every live peer finished the combine that last read the set `inval`
  // names: mark it invalid before the pre-reduce behind this barrier
  // overwrites it (a late reader's re-check then sees the change)
  if (t == 0 && p.inval) *(volatile unsigned long long *)p.inval = 0ull;
}

// ---------------------------------------------------------------------------
// drop-in multi-device collective in one launch per device (single process,
// one view per replica on several GPUs): entry flag barrier, this device's
// owner slice of the ascending masked fold (ref:comm.py:191-200), exit flag
// barrier, fused so a small bucket costs one launch per device instead of
// three.  Flags are the device group's (MdGroup): slot `me` of every peer's
// array receives this device's sequence numbers.

constexpr int kMdMaxIn = 8;  // contributors evaluated from registers

struct MdParams {
  const char *in[kMdMaxIn];
  char *out[RCV_MAX_OUT];
  int n_in, n_out;
  unsigned long long nvec;  // whole vectors of the owner slice
  unsigned long long tail;  // trailing scalars (ragged last slice)
  double divisor;           // 0: no scale
  unsigned long long *peer[32];
  unsigned long long *local;
  unsigned int *status;
  unsigned int *count;  // blocks done (reset by the last one)
  unsigned long long v_in, v_out, timeout_ns;
  int n_dev, me;
};

__device__ __forceinline__ void md_wait(const MdParams &p, int t, unsigned long long v) {
  if (t < p.n_dev && t != p.me) {
    const unsigned long long t0 = globaltimer();
    unsigned long long x;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p.local + t) : "memory");
      if (x >= v) break;
      if (globaltimer() - t0 > p.timeout_ns) {
        atomicOr(p.status, 1u << (t & 31));
        break;
      }
    }
  }
}

__device__ __forceinline__ void md_signal(const MdParams &p, int t, unsigned long long v) {
  if (t < p.n_dev && t != p.me)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.peer[t] + p.me), "l"(v) : "memory");
}

template <typename T> struct MdVec;
template <> struct MdVec<float> { typedef float4 V; };
template <> struct MdVec<double> { typedef double2 V; };

// coherent 16-byte load (the peers' views were written before their entry
// signal, which this thread's block acquired)
__device__ __forceinline__ float4 md_ld(const char *a, float4 *) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ double2 md_ld(const char *a, double2 *) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a) : "memory");
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) md_allreduce_kernel(const __grid_constant__ MdParams p) {
  typedef typename MdVec<T>::V V;
  const int t = threadIdx.x;
  __shared__ int last;
  if (blockIdx.x == 0) {
    // this device's earlier stream work (the contributors' accumulation) is
    // complete: release it to the peers
    __threadfence_system();
    md_signal(p, t, p.v_in);
  }
  md_wait(p, t, p.v_in);
  __syncthreads();
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + t; i < p.nvec; i += stride) {
    const unsigned long long off = i * sizeof(V);
    V x[kMdMaxIn];
#pragma unroll
    for (int k = 0; k < kMdMaxIn; ++k)
      if (k < p.n_in) x[k] = md_ld(p.in[k] + off, (V *)nullptr);
    V acc = x[0];
#pragma unroll
    for (int k = 1; k < kMdMaxIn; ++k)
      if (k < p.n_in) acc = vadd(acc, x[k]);
    if (p.divisor != 0.0) acc = vdiv(acc, p.divisor);
    for (int j = 0; j < p.n_out; ++j) *reinterpret_cast<V *>(p.out[j] + off) = acc;
  }
  if (blockIdx.x == 0 && t < (int)p.tail) {
    const unsigned long long off = p.nvec * sizeof(V) + (unsigned long long)t * sizeof(T);
    T acc = *reinterpret_cast<const volatile T *>(p.in[0] + off);
    for (int k = 1; k < p.n_in; ++k) acc = sadd(acc, *reinterpret_cast<const volatile T *>(p.in[k] + off));
    if (p.divisor != 0.0) acc = sdiv(acc, p.divisor);
    for (int j = 0; j < p.n_out; ++j) *reinterpret_cast<T *>(p.out[j] + off) = acc;
  }
  // exit: the last block to finish tells the peers that every store of this
  // device's slice has landed, then waits until theirs have (this launch
  // completes only when every remote store into this device's views is done)
  __threadfence_system();
  __syncthreads();
  if (t == 0) {
    const unsigned int done = atomicAdd(p.count, 1u);
    last = done == gridDim.x - 1;
    if (last) *p.count = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence_system();
  md_signal(p, t, p.v_out);
  md_wait(p, t, p.v_out);
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
  bool pair = false;  // DIRECT: two vectors per thread (small perfect trees, fp32)
  int shape = -1;     // >= 0: index of a compile-time program (shapes.inc)
  uint32_t mc_mask = 0;  // bit j: out[j] is a multicast address (fp32 vector paths only)
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
  p.mc_mask = r.mc_mask;
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
  p.mc_mask = r.mc_mask;
  p.nvec = nvec;
  p.divisor = r.divisor;
  p.guard = r.guard;
  p.guard_mask = r.guard_mask;
  p.n_roots = r.n_roots;
  memcpy(p.root_L, r.root_L, sizeof p.root_L);
  memcpy(p.root_first, r.root_first, sizeof p.root_first);
  if (r.tree_L >= 0) {
    const int nodes = (2 << r.tree_L) - 1;
    memcpy(p.node_in, r.node_in, nodes);
    memcpy(p.present, r.present, nodes);
  }
}

template <typename A, typename Prog>
int launch_direct_p(const FoldReq &r, unsigned long long e0, unsigned long long nvec,
                    cudaStream_t st, int sms) {
  FoldParams p;
  fill_vec_params<A>(p, r, e0, nvec);
  const unsigned long long want = (nvec + 255) / 256;
  unsigned long long blocks = std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)sms * 8));
  if (r.max_ctas > 0) blocks = std::min<unsigned long long>(blocks, (unsigned long long)r.max_ctas * 4);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if constexpr (std::is_same<A, float>::value && StraightIn<Prog>::value >= 1 &&
                StraightIn<Prog>::value <= 16) {
    if (r.pair) {
      // the same (SM-share-capped) grid: twice the bytes in flight per SM
      fold_direct_pair_kernel<Prog><<<(unsigned)blocks, 256, 0, st>>>(p);
      CK(cudaGetLastError());
      return RCV_OK;
    }
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
  kern<<<(unsigned)blocks, TMA_THREADS, g.smem, st>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}

// Straight-line evaluators of the degraded covers (shapes.inc), DIRECT only.
template <typename A>
int launch_shape(const FoldReq &r, unsigned long long e0, unsigned long long nvec,
                 cudaStream_t st, int sms) {
  if constexpr (std::is_same<A, double>::value) {
    return set_err(RCV_EINVAL, "fixed tree programs are fp32 only");
  } else {
    switch (r.shape) {
#define RCV_SHAPE(I, N, OPS) \
  case I:                    \
    return launch_direct_p<A, ProgFixed<N, OPS>>(r, e0, nvec, st, sms);
#include "shapes.inc"
#undef RCV_SHAPE
      default:
        return set_err(RCV_EINVAL, "unknown fixed tree program %d", r.shape);
    }
  }
}

// Launch `variant` (TMA / DIRECT) of the best program policy for r.
template <typename A>
int launch_vec(const FoldReq &r, bool tma, const TmaGeom &g, int maxd,
               unsigned long long e0, unsigned long long nvec, cudaStream_t st, int sms) {
#define RCV_LAUNCH(PROG) \
  return tma ? launch_tma_p<A, PROG>(r, g, e0, nvec, st, sms) : launch_direct_p<A, PROG>(r, e0, nvec, st, sms)
  if (r.n_roots > 0) RCV_LAUNCH(ProgForest);
  if (r.shape >= 0 && !tma && !std::is_same<A, double>::value)
    return launch_shape<A>(r, e0, nvec, st, sms);
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
  if (r.tree_L >= 0 && r.tree_L <= 6) {
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

// head elements h (< 8) after which every pointer is 32-byte aligned, or -1
int common_head32(const FoldReq &r) {
  for (int h = 0; h < 8; ++h) {
    bool ok = true;
    for (int i = 0; i < r.n_in && ok; ++i)
      ok = ((uintptr_t)(r.in[i] + (size_t)h * esize(r.in_dt[i])) & 31) == 0;
    for (int j = 0; j < r.n_out && ok; ++j)
      ok = ((uintptr_t)(r.out[j] + (size_t)h * esize(r.acc_dt)) & 31) == 0;
    if (ok) return h;
  }
  return -1;
}

// The 256-bit DIRECT launch of a straight-line program (A = F8W / F8WS).
template <typename A>
int launch_w256(const FoldReq &r, unsigned long long e0, unsigned long long nvec, cudaStream_t st,
                int sms) {
  if (r.n_roots > 0) return launch_direct_p<A, ProgForest>(r, e0, nvec, st, sms);
  switch (r.full_L) {
    case 0: return launch_direct_p<A, ProgFull<0>>(r, e0, nvec, st, sms);
    case 1: return launch_direct_p<A, ProgFull<1>>(r, e0, nvec, st, sms);
    case 2: return launch_direct_p<A, ProgFull<2>>(r, e0, nvec, st, sms);
    case 3: return launch_direct_p<A, ProgFull<3>>(r, e0, nvec, st, sms);
    case 4: return launch_direct_p<A, ProgFull<4>>(r, e0, nvec, st, sms);
    case 5: return launch_direct_p<A, ProgFull<5>>(r, e0, nvec, st, sms);
    case 6: return launch_direct_p<A, ProgFull<6>>(r, e0, nvec, st, sms);
    default: return set_err(RCV_ERANGE, "256-bit path: perfect tree height %d", r.full_L);
  }
}

// RCV_W256: 0 off, 1 32-byte loads and stores, 2 the same with streaming
// (.cs) stores
int w256_mode() {
  static const int mode = [] {
    const char *v = getenv("RCV_W256");
    return v ? atoi(v) : 2;
  }();
  return mode;
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
    if (r.mc_mask) return set_err(RCV_EINVAL, "multicast output of an empty fold");
    for (int j = 0; j < r.n_out; ++j) CK(cudaMemsetAsync(r.out[j], 0, numel * esize(r.acc_dt), st));
    return RCV_OK;
  }
  const bool f64 = r.acc_dt == RCV_F64;
  bool wide = r.wide32 && !f64;  // fp32 over bf16 inputs: 8-element vectors (float8)
  bool any_bf16 = false;
  for (int i = 0; i < r.n_in && !f64; ++i) any_bf16 |= r.in_dt[i] == RCV_BF16;
  wide |= any_bf16;
  // HBM-bound straight-line folds over fp32 (the N=1 commit's perfect tree,
  // the pre-reduce forests): 32-byte vectors, one LDG/STG.256 per input and
  // output (not the NVLink combines, which keep the two-vector pair kernel)
  static const bool w256_comb = getenv("RCV_W256_COMB") && atoi(getenv("RCV_W256_COMB"));
  if (w256_mode() && !f64 && !any_bf16 && !r.mc_mask && (!r.pair || w256_comb) &&
      (variant == RCV_VARIANT_AUTO || variant == RCV_VARIANT_DIRECT) &&
      ((r.full_L >= 0 && r.full_L <= 6) || r.n_roots > 0)) {
    const int h32 = common_head32(r);
    if (h32 >= 0 && (size_t)h32 < numel && (r.n_roots == 0 || (h32 == 0 && numel % 8 == 0))) {
      const unsigned long long nv = (numel - h32) / 8;
      const unsigned long long end = h32 + nv * 8;
      if (h32) {
        rc = launch_scalar<float>(r, maxd, 0, h32, st, sms);
        if (rc) return rc;
      }
      if (nv) {
        rc = w256_mode() == 2 ? launch_w256<F8WS>(r, h32, nv, st, sms) : launch_w256<F8W>(r, h32, nv, st, sms);
        if (rc) return rc;
      }
      if (end < numel) rc = launch_scalar<float>(r, maxd, end, numel - end, st, sms);
      return rc;
    }
  }
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
    if (variant == RCV_VARIANT_AUTO && (r.full_L >= 0 || r.n_roots > 0 || r.shape >= 0))
      variant = RCV_VARIANT_DIRECT;
    if (r.mc_mask && variant == RCV_VARIANT_DIRECT && !(r.shape >= 0 || (r.full_L >= 0 && r.full_L <= 3)))
      variant = RCV_VARIANT_TMA;  // the DIRECT kernel fences multicast stores only for McDirect programs
    bool use_tma = variant == RCV_VARIANT_TMA || variant == RCV_VARIANT_AUTO;
    const bool geom_ok = f64 ? tma_geom<double>(r, &g) : (wide ? tma_geom<F8>(r, &g) : tma_geom<float>(r, &g));
    if (use_tma && !geom_ok) {
      if (variant == RCV_VARIANT_TMA || r.mc_mask)
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

}  // extern "C"

namespace {
// Flag arrays of one single-process device set (the drop-in multi-device
// collective): 64 u64 barrier slots and a status word per device, allocated
// once, read and written by peers over NVLink.
struct MdGroup {
  std::vector<int> devs;
  std::vector<unsigned long long *> flags;
  std::vector<unsigned int *> status;
  std::vector<unsigned int *> count;  // md_allreduce_kernel's finished-block counter
  unsigned long long seq = 0;
};
std::mutex g_md_mu;
std::vector<MdGroup *> g_md;

int md_group(const int *devices, int n, MdGroup **out) {
  std::lock_guard<std::mutex> lk(g_md_mu);
  for (MdGroup *g : g_md)
    if ((int)g->devs.size() == n && std::equal(g->devs.begin(), g->devs.end(), devices)) {
      *out = g;
      return RCV_OK;
    }
  MdGroup *g = new MdGroup();
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(devices[d]));
    unsigned long long *f = nullptr;
    unsigned int *s = nullptr;
    CK(cudaMalloc(&f, 64 * sizeof(unsigned long long)));
    CK(cudaMemset(f, 0, 64 * sizeof(unsigned long long)));
    CK(cudaMalloc(&s, 2 * sizeof(unsigned int)));
    CK(cudaMemset(s, 0, 2 * sizeof(unsigned int)));
    g->devs.push_back(devices[d]);
    g->flags.push_back(f);
    g->status.push_back(s);
    g->count.push_back(s + 1);
  }
  CK(cudaDeviceSynchronize());
  g_md.push_back(g);
  *out = g;
  return RCV_OK;
}

int md_barrier(MdGroup *g, int d, cudaStream_t st, unsigned long long value) {
  BarrierParams p;
  memset(&p, 0, sizeof p);
  const int n = (int)g->devs.size();
  for (int r = 0; r < n; ++r) p.peer[r] = g->flags[r];
  p.local = g->flags[d];
  p.status = g->status[d];
  p.live = n >= 64 ? ~0ull : ((1ull << n) - 1);
  p.value = value;
  p.timeout_ns = 10ull * 1000000000ull;
  p.n = n;
  p.me = d;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  barrier_kernel<<<1, 32, 0, st>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
}
// The fused one-launch path: fp32/fp64 views, at most kMdMaxIn
// contributors, 16-byte aligned views (RCV_MD_SPLIT=1: the three-launch
// path, a measurement A/B).
bool md_fused_ok(const FoldReq &r, void *const *views, int n) {
  static const bool split = getenv("RCV_MD_SPLIT") && atoi(getenv("RCV_MD_SPLIT"));
  if (split || r.n_in < 1 || r.n_in > kMdMaxIn || (r.acc_dt != RCV_F32 && r.acc_dt != RCV_F64))
    return false;
  for (int i = 0; i < n; ++i)
    if ((uintptr_t)views[i] % 16) return false;
  return true;
}

int md_fused(const FoldReq &r, MdGroup *g, size_t numel, const int *devices, int n_dev,
             void *const *streams, unsigned long long v_in, unsigned long long v_out) {
  const int es = esize(r.acc_dt);
  const size_t w = 16 / es;  // elements per vector
  const size_t unit = 8;
  const size_t units = (numel + unit - 1) / unit;
  MdParams p;
  memset(&p, 0, sizeof p);
  p.n_in = r.n_in;
  p.n_out = r.n_out;
  p.divisor = r.divisor;
  p.timeout_ns = 10ull * 1000000000ull;
  p.n_dev = n_dev;
  p.v_in = v_in;
  p.v_out = v_out;
  for (int k = 0; k < n_dev; ++k) p.peer[k] = g->flags[k];
  // every device launches, an empty slice included: its peers wait on its flags
  for (int d = 0; d < n_dev; ++d) {
    const size_t a = std::min(numel, units * d / n_dev * unit);
    const size_t b = std::min(numel, units * (d + 1) / n_dev * unit);
    for (int i = 0; i < r.n_in; ++i) p.in[i] = r.in[i] + a * es;
    for (int j = 0; j < r.n_out; ++j) p.out[j] = r.out[j] + a * es;
    p.nvec = (b - a) / w;
    p.tail = (b - a) % w;
    p.local = g->flags[d];
    p.status = g->status[d];
    p.count = g->count[d];
    p.me = d;
    CK(cudaSetDevice(devices[d]));
    const unsigned long long want = (p.nvec + 255) / 256;
    const unsigned int blocks = (unsigned int)std::max<unsigned long long>(
        1, std::min<unsigned long long>(want, 4ull * dev_sms(devices[d])));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (r.acc_dt == RCV_F32)
      md_allreduce_kernel<float><<<blocks, 256, 0, (cudaStream_t)streams[d]>>>(p);
    else
      md_allreduce_kernel<double><<<blocks, 256, 0, (cudaStream_t)streams[d]>>>(p);
    CK(cudaGetLastError());
  }
  return RCV_OK;
}
}  // namespace

extern "C" {

// One owner slice per device, fenced on both sides by a device-side flag
// barrier among the devices (no host round trip, no per-call events): the
// entry barrier proves every device's prior stream work (the contributors'
// accumulation into their views) is done before any peer reads it, the exit
// barrier that every remote store into this device's views has landed
// before its stream moves on.  fp32/fp64 with <= 8 contributors: all three
// in one launch per device (md_allreduce_kernel); otherwise barrier, fold
// kernel, barrier.
int rcv_masked_allreduce_multidev(void *const *views, int n,
                                  uint64_t contrib_mask, int dtype,
                                  size_t numel, double divisor, int n_dev,
                                  const int *devices, void *const *streams) {
  if (n_dev < 1 || n_dev > 32) return set_err(RCV_ERANGE, "device count %d out of range", n_dev);
  FoldReq r;
  int rc = build_allreduce(r, views, n, contrib_mask, dtype, divisor);
  if (rc) return rc;
  if (numel == 0) return RCV_OK;
  int prev = 0;
  CK(cudaGetDevice(&prev));
  MdGroup *g = nullptr;
  if ((rc = md_group(devices, n_dev, &g))) return rc;
  const unsigned long long v_in = ++g->seq, v_out = ++g->seq;
  if (md_fused_ok(r, views, n)) {
    rc = md_fused(r, g, numel, devices, n_dev, streams, v_in, v_out);
    cudaSetDevice(prev);
    return rc;
  }
  for (int d = 0; d < n_dev; ++d) {
    CK(cudaSetDevice(devices[d]));
    if ((rc = md_barrier(g, d, (cudaStream_t)streams[d], v_in))) return rc;
  }
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
  for (int d = 0; d < n_dev; ++d) {
    CK(cudaSetDevice(devices[d]));
    if ((rc = md_barrier(g, d, (cudaStream_t)streams[d], v_out))) return rc;
  }
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

int rcv_kacc_push(const void *const *seg_ptr, const uint64_t *seg_off, const uint64_t *seg_len,
                  int n_seg, int grad_dtype, const float *const *stack, int c, float *out,
                  size_t numel, void *stream) {
  if (n_seg < 1 || n_seg > KACC_MAX_SEGS) return set_err(RCV_ERANGE, "kacc: %d segments (1..%d)", n_seg, KACC_MAX_SEGS);
  if (c < 0 || c > KACC_MAX_DEPTH) return set_err(RCV_ERANGE, "kacc: carry chain %d (0..%d)", c, KACC_MAX_DEPTH);
  if (grad_dtype != RCV_F32 && grad_dtype != RCV_BF16) return set_err(RCV_EINVAL, "kacc: gradient dtype %d", grad_dtype);
  if (!out || ((uintptr_t)out & 15)) return set_err(RCV_EINVAL, "kacc: output must be 16-byte aligned");
  KaccParams p;
  memset(&p, 0, sizeof p);
  unsigned long long pos = 0;
  const unsigned align = grad_dtype == RCV_BF16 ? 8u : 16u;
  for (int i = 0; i < n_seg; ++i) {
    if (seg_off[i] != pos) return set_err(RCV_EINVAL, "kacc: segment %d starts at %llu, want %llu", i,
                                          (unsigned long long)seg_off[i], pos);
    if (seg_len[i] % 4 || ((uintptr_t)seg_ptr[i] & (align - 1)))
      return set_err(RCV_EINVAL, "kacc: segment %d (%llu elements at %p) is not a whole, aligned "
                     "number of 4-element vectors", i, (unsigned long long)seg_len[i], seg_ptr[i]);
    p.src[i] = (const char *)seg_ptr[i];
    p.off[i] = pos;
    pos += seg_len[i];
  }
  if (pos != numel) return set_err(RCV_EINVAL, "kacc: segments hold %llu elements, want %zu", pos, numel);
  p.off[n_seg] = pos;
  for (int i = 0; i < c; ++i) {
    if (!stack[i] || ((uintptr_t)stack[i] & 15)) return set_err(RCV_EINVAL, "kacc: stack entry %d must be 16-byte aligned", i);
    p.stack[i] = stack[i];
  }
  p.out = out;
  p.nvec = numel / 4;
  p.n_seg = n_seg;
  p.c = c;
  p.bf16 = grad_dtype == RCV_BF16;
  if (!p.nvec) return RCV_OK;
  const int sms = current_device_sms();
  const unsigned long long blocks = std::max<unsigned long long>(
      1, std::min<unsigned long long>((p.nvec + 255) / 256, (unsigned long long)sms * 8));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  kacc_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p);
  CK(cudaGetLastError());
  return RCV_OK;
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
  if (r.full_L < 0 && acc_dtype == RCV_F32 && n_blocks <= 21 && !getenv("RCV_NO_FIXED")) {
    // a compile-time program for this cover (the degraded combines)?
    static const struct {
      int n;
      unsigned long long ops;
    } kShapes[] = {
#define RCV_SHAPE(I, N, OPS) {N, OPS},
#include "shapes.inc"
#undef RCV_SHAPE
    };
    unsigned long long packed = 0;
    bool fits = true;
    for (int i = 0; i < n_blocks; ++i) {
      fits &= (r.op[i] & RCV_OP_MERGES_MASK) <= 7;
      packed |= (unsigned long long)(r.op[i] & 7) << (3 * i);
    }
    for (int s = 0; fits && s < (int)(sizeof kShapes / sizeof kShapes[0]); ++s)
      if (kShapes[s].n == n_blocks && kShapes[s].ops == packed) r.shape = s;
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

// ---- NVLink SHARP multicast objects ----------------------------------------

namespace {
struct McApi {
  CUresult (*create)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
  CUresult (*gran)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
  CUresult (*add)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*bind)(CUmemGenericAllocationHandle, size_t, CUdeviceptr, size_t, unsigned long long);
  CUresult (*unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*device)(CUdevice *, int);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*free_va)(CUdeviceptr, size_t);
  bool ok = false;
};

int mc_api(McApi **out) {
  static McApi a;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!a.ok) {
    struct { const char *name; void **fn; } t[] = {
        {"cuMulticastCreate", (void **)&a.create},
        {"cuMulticastGetGranularity", (void **)&a.gran},
        {"cuMulticastAddDevice", (void **)&a.add},
        {"cuMulticastBindAddr", (void **)&a.bind},
        {"cuMulticastUnbind", (void **)&a.unbind},
        {"cuDeviceGet", (void **)&a.device},
        {"cuMemUnmap", (void **)&a.unmap},
        {"cuMemAddressFree", (void **)&a.free_va}};
    for (auto &e : t) {
      cudaDriverEntryPointQueryResult q;
      CK(cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !*e.fn) return set_err(RCV_ECUDA, "%s unavailable", e.name);
    }
    a.ok = true;
  }
  *out = &a;
  return RCV_OK;
}

CUmulticastObjectProp mc_prop(size_t bytes, int n_dev) {
  CUmulticastObjectProp prop = {};
  prop.numDevices = (unsigned int)n_dev;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = bytes;
  return prop;
}

int mc_current_device(McApi *a, CUdevice *dev) {
  int d = 0;
  CK(cudaGetDevice(&d));
  if (a->device(dev, d) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuDeviceGet(%d)", d);
  return RCV_OK;
}
}  // namespace

int rcv_mc_supported(int *ok) {
  int d = 0;
  CK(cudaGetDevice(&d));
  *ok = 0;
  CK(cudaDeviceGetAttribute(ok, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  return RCV_OK;
}

int rcv_mc_granularity(int n_dev, size_t *gran) {
  McApi *a = nullptr;
  int rc = mc_api(&a);
  if (rc) return rc;
  CUmulticastObjectProp prop = mc_prop(1 << 21, n_dev);
  if (a->gran(gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMulticastGetGranularity");
  return RCV_OK;
}

int rcv_mc_create(size_t bytes, int n_dev, uint64_t *handle, size_t *size_out, int *fd_out) {
  McApi *a = nullptr;
  Vmm *v = nullptr;
  int rc = mc_api(&a);
  if (rc || (rc = vmm(&v))) return rc;
  size_t gran = 0;
  if ((rc = rcv_mc_granularity(n_dev, &gran))) return rc;
  const size_t size = (bytes + gran - 1) / gran * gran;
  CUmulticastObjectProp prop = mc_prop(size, n_dev);
  CUmemGenericAllocationHandle h;
  CUresult e = a->create(&h, &prop);
  if (e != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMulticastCreate(%zu bytes, %d GPUs): %d", size, n_dev, (int)e);
  int fd = -1;
  if (v->exportfd(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemExportToShareableHandle(multicast)");
  *handle = (uint64_t)h;
  *size_out = size;
  *fd_out = fd;
  return RCV_OK;
}

int rcv_mc_import(int fd, uint64_t *handle) {
  Vmm *v = nullptr;
  int rc = vmm(&v);
  if (rc) return rc;
  CUmemGenericAllocationHandle h;
  if (v->importfd(&h, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemImportFromShareableHandle(multicast fd %d)", fd);
  *handle = (uint64_t)h;
  return RCV_OK;
}

int rcv_mc_add_device(uint64_t handle) {
  McApi *a = nullptr;
  int rc = mc_api(&a);
  if (rc) return rc;
  CUdevice dev;
  if ((rc = mc_current_device(a, &dev))) return rc;
  CUresult e = a->add((CUmemGenericAllocationHandle)handle, dev);
  if (e != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMulticastAddDevice: %d", (int)e);
  return RCV_OK;
}

int rcv_mc_bind(uint64_t handle, void *local_ptr, size_t bytes) {
  McApi *a = nullptr;
  int rc = mc_api(&a);
  if (rc) return rc;
  CUresult e = a->bind((CUmemGenericAllocationHandle)handle, 0, (CUdeviceptr)local_ptr, bytes, 0);
  if (e != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMulticastBindAddr(%zu bytes): %d", bytes, (int)e);
  return RCV_OK;
}

int rcv_mc_map(uint64_t handle, size_t size, void **mc_ptr) {
  Vmm *v = nullptr;
  int rc = vmm(&v);
  if (rc) return rc;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  size_t gran = 0;
  CUdeviceptr va = 0;
  if ((rc = rcv_mc_granularity(1, &gran))) return rc;
  if (v->reserve(&va, size, gran, 0, 0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemAddressReserve(multicast)");
  if (v->map(va, size, 0, (CUmemGenericAllocationHandle)handle, 0) != CUDA_SUCCESS)
    return set_err(RCV_ECUDA, "cuMemMap(multicast)");
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (v->access(va, size, &acc, 1) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuMemSetAccess(multicast)");
  *mc_ptr = (void *)va;
  return RCV_OK;
}

int rcv_mc_release(uint64_t handle, void *mc_ptr, size_t size) {
  McApi *a = nullptr;
  Vmm *v = nullptr;
  int rc = mc_api(&a);
  if (rc || (rc = vmm(&v))) return rc;
  if (mc_ptr) {
    a->unmap((CUdeviceptr)mc_ptr, size);
    a->free_va((CUdeviceptr)mc_ptr, size);
  }
  CUdevice dev;
  if (mc_current_device(a, &dev) == RCV_OK) a->unbind((CUmemGenericAllocationHandle)handle, dev, 0, size);
  v->release((CUmemGenericAllocationHandle)handle);
  return RCV_OK;
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

}  // extern "C"

// ---------------------------------------------------------------------------
// native per-bucket runtime (multi-process commit)

namespace {

// pool-set integrity stamps live in the rank's flag array after the barrier
// slots: word kStampBase + s belongs to pool set s (rcv_pool_sets() sets)
constexpr int kStampBase = 64;
constexpr int kMaxSets = 8;


}  // namespace

struct TimingRec {
  int kind;
  double bytes, nin, nout;
  cudaEvent_t a, b;
};

struct rcv_ctx {
  int n_ranks = 0, me = 0, device = 0, sms = 148;
  BarrierParams bar;
  unsigned int *err = nullptr;  // status word 1: stamp mismatches seen by this rank's combines
  cudaStream_t side = nullptr;     // pre-reduces (and fragmented covers' broadcasts)
  cudaStream_t bstream = nullptr;  // perfect covers' broadcasts, right behind each barrier
  cudaStream_t bar_st = nullptr;   // every flag barrier, in call order
  cudaEvent_t ev_main = nullptr, ev_ready = nullptr, ev_trans = nullptr, ev_bcast = nullptr;
  cudaEvent_t ev_join = nullptr;
  cudaEvent_t ev_arrived[kMaxSets] = {};  // barrier of call j passed
  cudaEvent_t ev_comb[kMaxSets] = {};     // combine of call j finished
  int sets = 4;                           // pool sets rotated through (rcv_pool_sets)
  // barrier lag L (RCV_BARRIER_LAG, 1 or 2): the barrier of call j runs on
  // its own stream behind this rank's combine j-L, so with L = 2 it overlaps
  // combine j-1 and the combines run back to back on the main stream.
  // Passing barrier j proves every live peer finished its pre-reduce j and
  // its combine j-L; every other wait in the schedule follows from that.
  int lag = 2;
  bool in_step = false;
  bool bstream_dirty = false;  // bstream holds broadcasts the side stream has not waited for
  unsigned long long calls = 0, seq = 0;
  // live mask of the previous bucket call in this step (0: none since the
  // last rcv_ctx_finish).  A call whose mask drops ranks first joins one
  // barrier over this mask, departing ranks included: their last combine
  // read this rank's pool sets and stored into its primary.
  uint64_t last_live = 0;
  bool no_stamps = false;  // RCV_NO_STAMPS=1: measurement A/B only
  // the stamps each combine not yet re-checked read, in call order; a
  // barrier re-checks those of the combines it is ordered behind
  struct Check {
    unsigned long long call, value;
    std::vector<const unsigned long long *> stamps;
  };
  std::vector<Check> hist;
  struct Pending {
    FoldReq req;
    size_t lo, n;
    int variant;
    unsigned long long call;  // bucket call index that combined it
  };
  std::vector<Pending> pending;  // combined buckets awaiting the local broadcast
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
  unsigned long long *stamp_of(int rank, int set) const { return bar.peer[rank] + kStampBase + set; }
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
  std::vector<int> producers;  // distinct ranks whose pool slots the combine reads
  bool has_bcast = false;
  FoldReq bcast;
  int variant = 0, comb_variant = 0;
  uint64_t live_mask = 0;
  bool participate = false;
  bool perfect = false;  // one cover node per live rank (the failure-free layout)
  int remote_in = 0, remote_out = 0;
  // first element of owner slice q of a bucket of `units` 64-element units
  size_t slice_at(size_t units, int q) const { return units * q / slice_nr * 64; }
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

// Barriers run on the bar stream (the caller's stream while timing launch
// by launch).  `upto`: the last call whose combine this barrier is ordered
// behind (-1: all of them; the caller made the bar stream wait for main's
// tail); those combines' stamps are re-checked before the signal.  `now`:
// the stamps the combine of this call reads, checked == now_value after the
// wait.  `ready` / `inval`: this rank's own stamps the kernel writes
// (BarrierParams).
int ctx_barrier(rcv_ctx *c, uint64_t live, bool participate, cudaStream_t st, long long upto,
                unsigned long long call = 0,
                const std::vector<const unsigned long long *> *now = nullptr,
                unsigned long long now_value = 0, unsigned long long *ready = nullptr,
                unsigned long long *inval = nullptr) {
  if (!participate || __builtin_popcountll(live) < 2) {
    c->hist.clear();  // no peer: nothing can race this rank's combines
    return RCV_OK;
  }
  c->bar.live = live;
  c->bar.value = ++c->seq;
  c->bar.err = c->err;
  int np = 0;
  size_t done = 0;
  for (; done < c->hist.size(); ++done) {
    const rcv_ctx::Check &h = c->hist[done];
    if (upto >= 0 && (long long)h.call > upto) break;
    for (const unsigned long long *a : h.stamps) {
      if (np == 32) break;
      c->bar.chk_prev[np] = a;
      c->bar.prev_value[np++] = h.value;
    }
  }
  c->hist.erase(c->hist.begin(), c->hist.begin() + done);
  c->bar.n_prev = np;
  c->bar.n_now = now ? (int)now->size() : 0;
  for (int i = 0; i < c->bar.n_now; ++i) c->bar.chk_now[i] = (*now)[i];
  c->bar.now_value = now_value;
  c->bar.ready = ready;
  c->bar.ready_value = now_value;
  c->bar.inval = inval;
  if (now) c->hist.push_back({call, now_value, *now});
  return timed(c, st, 1, 0, 0, 0, [&]() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    barrier_kernel<<<1, 32, 0, st>>>(c->bar);
    CK(cudaGetLastError());
    return RCV_OK;
  });
}

cudaStream_t bar_stream(rcv_ctx *c, cudaStream_t main) { return c->timing ? main : c->bar_st; }

// `to` waits for everything enqueued on `from` so far
int join(rcv_ctx *c, cudaStream_t from, cudaStream_t to) {
  if (from == to) return RCV_OK;
  CK(cudaEventRecord(c->ev_join, from));
  CK(cudaStreamWaitEvent(to, c->ev_join, 0));
  return RCV_OK;
}

// A barrier behind all of this rank's work on `main` (closing, poll and
// transition barriers), then `main`, side and bstream wait for it.
int full_barrier(rcv_ctx *c, uint64_t live, bool participate, cudaStream_t main) {
  cudaStream_t b = bar_stream(c, main);
  int rc = join(c, main, b);
  if (rc) return rc;
  if ((rc = ctx_barrier(c, live, participate, b, -1))) return rc;
  CK(cudaEventRecord(c->ev_trans, b));
  CK(cudaStreamWaitEvent(main, c->ev_trans, 0));
  CK(cudaStreamWaitEvent(c->side, c->ev_trans, 0));
  if (c->bstream) CK(cudaStreamWaitEvent(c->bstream, c->ev_trans, 0));
  return RCV_OK;
}

// Membership shrank since the previous call of this step: every rank of the
// previous mask joins one barrier over it, after its last combine.  Passing
// it proves that the departing ranks' combines, which read this rank's pool
// sets and stored into its primary replica, are complete, so no pool set is
// rewritten and no bucket broadcast before they land.
int ctx_transition(rcv_ctx *c, uint64_t live, cudaStream_t main) {
  const uint64_t prev = c->last_live;
  c->last_live = live;
  if (!prev || !(prev & ~live)) return RCV_OK;
  return full_barrier(c, prev, (prev >> c->me) & 1ull, main);
}

// Broadcast the pending buckets combined at call index <= upto (all of them
// when upto < 0) from this rank's primary replica to its other replicas.
int ctx_flush(rcv_ctx *c, cudaStream_t st, long long upto) {
  while (!c->pending.empty() && (upto < 0 || (long long)c->pending.front().call <= upto)) {
    rcv_ctx::Pending e = c->pending.front();
    c->pending.erase(c->pending.begin());
    shift(e.req, e.lo, e.lo);
    const double bytes = (double)(e.req.n_in + e.req.n_out) * e.n * esize(e.req.acc_dt);
    int rc = timed(c, st, 2, bytes, 0, 0,
                   [&]() { return run_fold(e.req, e.n, e.variant, st, c->sms); });
    if (rc) return rc;
  }
  return RCV_OK;
}

// Load every kernel of this library's module on the current device.  Under
// CUDA lazy loading (the default) the first launch of a kernel may need a
// context synchronisation; if a barrier kernel is already spinning for a
// signal a peer's not-yet-loaded kernel is to produce, that is a deadlock
// (broken only by the wait's timeout).  So the runtime loads all of its
// kernels up front, once per device.
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
  GetModule get_module = nullptr;
  Count count = nullptr;
  Enum enumerate = nullptr;
  Load load = nullptr;
  struct {
    const char *name;
    void **fn;
  } eps[] = {{"cuFuncGetModule", (void **)&get_module},
             {"cuModuleGetFunctionCount", (void **)&count},
             {"cuModuleEnumerateFunctions", (void **)&enumerate},
             {"cuFuncLoad", (void **)&load}};
  for (auto &e : eps) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !*e.fn) return set_err(RCV_ECUDA, "%s unavailable", e.name);
  }
  cudaFunction_t f0 = nullptr;
  CK(cudaGetFuncBySymbol(&f0, (const void *)barrier_kernel));
  CUmodule mod = nullptr;
  if (get_module(&mod, (CUfunction)f0) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuFuncGetModule");
  unsigned int n = 0;
  if (count(&n, mod) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuModuleGetFunctionCount");
  std::vector<CUfunction> fs(n);
  if (n && enumerate(fs.data(), n, mod) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuModuleEnumerateFunctions");
  for (CUfunction f : fs)
    if (load(f) != CUDA_SUCCESS) return set_err(RCV_ECUDA, "cuFuncLoad");
  done.push_back(dev);
  return RCV_OK;
}

// SM shares of the concurrent streams: a full-occupancy grid of any kernel
// would keep the others off the GPU until its last wave drains, and more
// CTAs streaming HBM at once lower its efficiency.  Pre-reduce: 0.6 of the
// SMs (N=4 62.7 -> 64.2 M tokens/s, N=2 56.1 -> 57.9 M against round 2's
// 0.75 / 0.65; 0.3-0.5 and 0.85 are slower: profiles/r2/pre_share_ab.txt).
// Combine: its owner slice shrinks as 1/n with n live ranks, so its share
// does too, 0.45/n but at least 0.15 (N=2 0.225, N=4 0.15: N=4 60.1 -> 63.1
// M against round 2's fixed 0.25 / 0.35; profiles/r2/comb_share_ab.txt).
// RCV_COMB_CTAS / RCV_PRE_CTAS override (an absolute CTA count > 2, or a
// fraction of the SMs; 0: uncapped).
int env_ctas(const char *name, int sms, double dflt_frac) {
  const char *v = getenv(name);
  const double f = v ? atof(v) : dflt_frac;
  if (f <= 0) return 0;
  if (f > 2.0) return (int)f;
  return std::max(1, (int)(f * sms));
}

double pre_share(const rcv_plan_desc *) { return 0.6; }

double comb_share(const rcv_plan_desc *d) {
  return std::max(0.15, 0.45 / std::max(1, d->slice_nr));
}

}  // namespace

extern "C" {

int rcv_pool_sets(void) {
  // RCV_POOL_SETS (3..8) is a measurement A/B; the allocator (dist.py) and
  // the context read the same value
  const char *v = getenv("RCV_POOL_SETS");
  return v ? std::min(kMaxSets, std::max(3, atoi(v))) : 4;
}

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
  c->err = status + 1;
  c->no_stamps = getenv("RCV_NO_STAMPS") && atoi(getenv("RCV_NO_STAMPS"));
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->bstream, cudaStreamNonBlocking));
  {
    // the barrier stream gets the highest priority: its one-CTA kernel must
    // find a slot while the pre-reduce and combine grids occupy the SMs
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->bar_st, cudaStreamNonBlocking, hi));
  }
  if (const char *v = getenv("RCV_BARRIER_LAG")) c->lag = atoi(v) == 1 ? 1 : 2;
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (int i = 0; i < kMaxSets; ++i) CK(cudaEventCreateWithFlags(&c->ev_comb[i], cudaEventDisableTiming));
  c->sets = rcv_pool_sets();
  CK(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_trans, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_bcast, cudaEventDisableTiming));
  for (int i = 0; i < kMaxSets; ++i) CK(cudaEventCreateWithFlags(&c->ev_arrived[i], cudaEventDisableTiming));
  *out = c;
  return RCV_OK;
}

int rcv_ctx_destroy(rcv_ctx *c) {
  if (!c) return RCV_OK;
  cudaStreamSynchronize(c->side);
  cudaStreamSynchronize(c->bstream);
  cudaStreamSynchronize(c->bar_st);
  for (auto &r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->spare_events) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_main, c->ev_ready, c->ev_trans, c->ev_bcast}) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_join);
  for (int i = 0; i < kMaxSets; ++i) {
    cudaEventDestroy(c->ev_arrived[i]);
    cudaEventDestroy(c->ev_comb[i]);
  }
  cudaStreamDestroy(c->bar_st);
  cudaStreamDestroy(c->bstream);
  cudaStreamDestroy(c->side);
  delete c;
  return RCV_OK;
}

int rcv_ctx_set_liveness(rcv_ctx *c, const uint32_t *device_dead_word) {
  c->bar.host_dead = (const volatile unsigned int *)device_dead_word;
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

// The side and broadcast streams' tails join the caller's stream.
static int join_tails(rcv_ctx *c, cudaStream_t st, bool clear) {
  if (!c->in_step) return RCV_OK;
  int rc = join(c, c->side, st);
  if (rc) return rc;
  if (c->bstream_dirty) {
    if ((rc = join(c, c->bstream, st))) return rc;
    if (clear) c->bstream_dirty = false;
  }
  return RCV_OK;
}

int rcv_ctx_finish(rcv_ctx *c, uint64_t live_mask, int participate, void *main_stream) {
  cudaStream_t st = (cudaStream_t)main_stream;
  int rc = join_tails(c, st, true);
  if (rc) return rc;
  // ranks that left after this step's last bucket call: one barrier over the
  // mask they last took part in
  if ((rc = ctx_transition(c, live_mask, st))) return rc;
  // the closing barrier: every live peer finished every combine of the step
  if ((rc = full_barrier(c, live_mask, participate != 0, st))) return rc;
  if ((rc = ctx_flush(c, st, -1))) return rc;
  c->in_step = false;
  c->last_live = 0;  // the closing barrier synchronised every live rank
  return RCV_OK;
}

int rcv_ctx_poll(rcv_ctx *c, uint64_t live_mask, int participate, void *main_stream) {
  cudaStream_t st = (cudaStream_t)main_stream;
  int rc = join_tails(c, st, false);
  if (rc) return rc;
  if ((rc = ctx_transition(c, live_mask, st))) return rc;
  return full_barrier(c, live_mask, participate != 0, st);
}

int rcv_plan_create(rcv_ctx *ctx, const rcv_plan_desc *d, rcv_plan **out) {
  rcv_plan *p = new rcv_plan();
  p->ctx = ctx;
  p->set_stride = d->set_stride;
  p->variant = d->variant;
  p->comb_variant = d->comb_variant;
  p->live_mask = d->live_mask;
  p->participate = d->participate != 0;
  p->perfect = d->n_comb > 0 && d->n_comb == d->slice_nr;
  p->remote_in = d->remote_in;
  p->remote_out = d->remote_out;
  const int pre_ctas = env_ctas("RCV_PRE_CTAS", ctx->sms, pre_share(d));
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
    r.max_ctas = pre_ctas;
    p->pre.push_back(r);
    p->pre_count.push_back(d->pre_counts[i]);
    off += d->pre_counts[i];
  }
  // several full pre-reduce nodes (each 2^level leaves, all present) fuse
  // into one forest launch; plain nodes stay separate requests
  if (d->n_pre > 1 && d->n_pre <= 8) {
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
      r.max_ctas = pre_ctas;
      p->has_forest = true;
      p->forest_count = k;
    }
  }
  if (d->n_comb > 0 && d->participate) {
    int rc = prepare_tree(d->comb_blocks, d->n_comb, d->n_leaves, d->n_comb_out, d->comb_out,
                          d->acc_dtype, d->divisor, p->comb);
    if (rc) {
      delete p;
      return rc;
    }
    p->comb.max_ctas = env_ctas("RCV_COMB_CTAS", ctx->sms, comb_share(d));
    // branchy trees (fragmented covers) evaluate 8-element vectors: half the
    // control flow per byte (N=2 degraded combine 167 -> 99 us)
    // (straight-line fixed programs keep 4-element vectors, two per thread,
    // like the perfect trees; RCV_WIDE_FIXED=1 measures the alternative)
    p->comb.wide32 = p->comb.full_L < 0 && (p->comb.shape < 0 || getenv("RCV_WIDE_FIXED"));
    // perfect trees over <= 8 nodes: two vectors per thread in flight
    p->comb.pair = true;
    if (d->guarded) {
      // the combine reads live peers' partials: skip it once one timed out
      p->comb.guard = (const unsigned int *)ctx->bar.status;
      p->comb.guard_mask = (unsigned int)(d->live_mask & ~(1ull << ctx->me));
    }
    if (d->comb_rank) {
      for (int i = 0; i < d->n_comb; ++i) {
        const int rk = d->comb_rank[i];
        if (rk < 0 || rk >= ctx->n_ranks) {
          delete p;
          return set_err(RCV_ERANGE, "rcv_plan_create: cover node %d from rank %d", i, rk);
        }
        if (std::find(p->producers.begin(), p->producers.end(), rk) == p->producers.end())
          p->producers.push_back(rk);
      }
    }
    // outputs that are multicast addresses: one store reaches every live
    // rank's landing buffer through the switch (rcv_mc_*)
    p->comb.mc_mask = d->comb_out_mc;
    p->has_comb = true;
    p->slice_q = d->slice_q;
    p->slice_nr = d->slice_nr;
  }
  if (d->n_bcast > 0) {
    FoldReq &r = p->bcast;
    r.n_in = 1;
    r.in[0] = (const char *)d->bcast_src;
    r.in_dt[0] = d->acc_dtype;
    r.op[0] = 0;
    r.n_out = d->n_bcast;
    for (int j = 0; j < d->n_bcast; ++j) r.out[j] = (char *)d->bcast_out[j];
    r.full_L = 0;  // a one-leaf tree: the straight-line DIRECT (256-bit) copy
    r.acc_dt = d->acc_dtype;
    // one copy per bucket (two replicas per rank) runs beside the combine
    // and the next pre-reduce: 0.3 of the SMs leaves them their share
    // (N=4 failure-free step 1.85 -> 1.60 ms); several copies (N=2: three)
    // are the HBM-bound part of the step and run uncapped
    // (profiles/r2/bcast_cap_ab.txt)
    r.max_ctas = env_ctas("RCV_BCAST_CTAS", ctx->sms, d->n_bcast == 1 ? 0.3 : 0.0);
    p->has_bcast = true;
  }
  *out = p;
  return RCV_OK;
}

int rcv_plan_destroy(rcv_plan *p) {
  delete p;
  return RCV_OK;
}

// One bucket call j of the step (see include/rcv.h for the schedule).  Four
// streams: side (pre-reduces), bar (barriers), main (combines), bstream
// (perfect covers' local broadcasts).  With barrier lag L (rcv_ctx::lag),
// barrier j waits for this rank's pre-reduce j and its combine j-L, so
// passing it proves every live peer finished both.  S pool sets
// (rcv_pool_sets): call j's pre-reduce overwrites the set last read by
// combine j-S, which every peer finished before its barrier j-S+L, so the
// side stream waits only for that barrier and runs up to S-L-1 pre-reduces
// ahead of the barriers; bucket b's outputs are complete in every primary
// once barrier b+L passed (its local broadcast).
int rcv_plan_bucket(rcv_plan *p, size_t lo, size_t n, void *main_stream) {
  if (n == 0) return RCV_OK;
  rcv_ctx *c = p->ctx;
  cudaStream_t main = (cudaStream_t)main_stream;
  // while timing launch by launch everything runs on the caller's stream, so
  // each kernel's duration is its own (no cross-stream overlap stretching it)
  cudaStream_t side = c->timing ? main : c->side;
  cudaStream_t bar = bar_stream(c, main);
  const int es = esize(p->has_comb ? p->comb.acc_dt : RCV_F32);
  const long long L = c->lag;
  if (!c->in_step) {
    // leaves were produced on the caller's stream
    c->in_step = true;
    CK(cudaEventRecord(c->ev_main, main));
    CK(cudaStreamWaitEvent(c->side, c->ev_main, 0));
  }
  int rc = ctx_transition(c, p->live_mask, main);
  if (rc) return rc;
  const unsigned long long j = c->calls++;
  const long long jj = (long long)j;
  const unsigned long long S = (unsigned long long)c->sets;
  const int set = (int)(j % S);
  const size_t set_off = set * p->set_stride;
  // perfect covers (pre-reduce-bound) broadcast on their own stream right
  // behind each barrier; fragmented ones (combine-bound) keep them on the
  // side stream, off the SMs the NVLink-bound combine needs
  // (profiles/r1f/schedule_ab.txt)
  const bool bstream = !c->timing && p->perfect;
  if (jj - (long long)S + L >= 0) {
    CK(cudaStreamWaitEvent(side, c->ev_arrived[(j - S + L) % S], 0));
    if (j >= S && !bstream) {
      if (c->bstream_dirty) {
        // an earlier broadcast of the same bucket may still be on bstream
        CK(cudaEventRecord(c->ev_bcast, c->bstream));
        CK(cudaStreamWaitEvent(side, c->ev_bcast, 0));
        c->bstream_dirty = false;
      }
      if ((rc = ctx_flush(c, side, jj - (long long)S))) return rc;
    }
  }
  // this call's pool set is stamped j+1 by barrier j once the pre-reduce is
  // done, and marked 0 by barrier j-S+L (which the side stream waited for
  // above) before it is overwritten: no stream operation between the
  // pre-reduces (a system-scope stream memop costs up to ~20 us on a GPU
  // busy with NVLink traffic)
  const bool writes = p->participate && (p->has_forest || !p->pre.empty()) && !c->no_stamps;
  bool forest_done = false;
  if (p->has_forest && n % 64 == 0) {
    FoldReq r = p->forest;
    shift(r, lo, set_off);
    // the forest evaluator needs 16-byte aligned whole vectors; misaligned
    // leaves (a caller's odd tensor offsets) take the per-node launches
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
  if (side != bar) {
    CK(cudaEventRecord(c->ev_ready, side));
    CK(cudaStreamWaitEvent(bar, c->ev_ready, 0));
  }
  if (bar != main && jj - L >= 0) CK(cudaStreamWaitEvent(bar, c->ev_comb[(j - L) % S], 0));
  size_t a = 0, z = 0;
  std::vector<const unsigned long long *> now;
  if (p->has_comb) {
    const size_t units = (n + 63) / 64;
    a = std::min(n, p->slice_at(units, p->slice_q));
    z = std::min(n, p->slice_at(units, p->slice_q + 1));
    if (z > a && !c->no_stamps)
      for (int rk : p->producers) now.push_back(c->stamp_of(rk, set));
  }
  // the barrier re-checks the stamps of the combines it is ordered behind
  // (calls <= j-L; all earlier ones while timing on one stream)
  if ((rc = ctx_barrier(c, p->live_mask, p->participate, bar, bar == main ? jj - 1 : jj - L, j,
                        &now, j + 1, writes ? c->stamp_of(c->me, set) : nullptr,
                        c->no_stamps ? nullptr : c->stamp_of(c->me, (int)((j + S - L) % S)))))
    return rc;
  CK(cudaEventRecord(c->ev_arrived[j % S], bar));
  if (bar != main) CK(cudaStreamWaitEvent(main, c->ev_arrived[j % S], 0));
  if (bstream && jj - L >= 0) {
    // the buckets combined at calls <= j-L are complete in this rank's primary
    CK(cudaStreamWaitEvent(c->bstream, c->ev_arrived[j % S], 0));
    if ((rc = ctx_flush(c, c->bstream, jj - L))) return rc;
    c->bstream_dirty = true;
  }
  if (z > a) {
    FoldReq r = p->comb;
    shift(r, set_off + a, lo + a);
    const double sl = (double)(z - a) * es;
    const double local = (double)(r.n_in - p->remote_in + r.n_out - p->remote_out) * sl;
    rc = timed(c, main, 3, local, p->remote_in * sl, p->remote_out * sl,
               [&]() { return run_fold(r, z - a, p->comb_variant, main, c->sms); });
    if (rc) return rc;
  }
  CK(cudaEventRecord(c->ev_comb[j % S], main));
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

}  // extern "C"
