// HBM probe for the N=1 fused commit (diagnostics, not the product).
//
// The bench's dominant kernel folds 32 microbatch-gradient streams into 8
// replica outputs per bucket (fold_direct_kernel<float, ProgFull<5>>, 995 MB
// per launch).  This probe replays that access pattern -- 32 separate
// 498 MB leaves, 8 separate 498 MB outputs, 20 buckets of 6,221,952 fp32 --
// with kernel variants that differ only in how they move bytes, to find the
// HBM ceiling of a 4:1 read:write stream mix on this B200:
//
//   base      the product's scheme: grid-stride float4, volatile
//             ld.global.nc.L1::no_allocate, depth-first tree, plain stores
//   nv        the same loads without `volatile` (the compiler may batch them)
//   hint      nv + st.global.cs stores
//   w256*     32-byte vectors per thread (sm_100 LDG/STG .256): volatile,
//             non-volatile, and with L2::evict_first loads
//   batch     all 32 loads of a vector issued before the first add
//   pair      two vectors per thread per iteration (both vectors' loads first)
//   read      read ceiling: 32 inputs, no outputs (a predicated store that
//             never fires keeps the loads alive)
//   copy      1 input -> 1 output (what MEASURED_PEAKS.json's copy measures)
//
// Each variant runs at several grid sizes; every line is one JSON object with
// the best-of-5 time of a 20-bucket pass and its algorithmic GB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/hbm_probe tools/hbm_probe.cu
//   /tmp/hbm_probe > gpurun_out/hbm_probe.jsonl

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));  \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

constexpr int NIN = 32, NOUT = 8, K = 20;
constexpr size_t D = 124439808;         // GPT-2 124M
constexpr size_t BUCKET = D / K / 64 * 64;  // 6,221,952 fp32

struct P {
  const float4 *in[NIN];
  float4 *out[NOUT];
  unsigned long long nvec;
  float inv;
};

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float d) {
  return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d), __fdiv_rn(a.w, d));
}

template <int MODE>
__device__ __forceinline__ float4 ld(const float4 *p) {
  float4 v;
  if constexpr (MODE == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else if constexpr (MODE == 1) {
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  }
  return v;
}

template <int MODE>
__device__ __forceinline__ void st(float4 *p, float4 v) {
  if constexpr (MODE == 2) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  } else {
    *p = v;
  }
}

template <int MODE, int LEVEL, int IDX>
__device__ __forceinline__ float4 tree(const P &p, unsigned long long v) {
  if constexpr (LEVEL == 0) {
    return ld<MODE>(p.in[IDX] + v);
  } else {
    const float4 a = tree<MODE, LEVEL - 1, 2 * IDX>(p, v);
    const float4 b = tree<MODE, LEVEL - 1, 2 * IDX + 1>(p, v);
    return add4(a, b);
  }
}

// base (MODE 0), nv (MODE 1), hint (MODE 2)
template <int MODE>
__global__ void __launch_bounds__(256) k_tree(const __grid_constant__ P p) {
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.nvec;
       v += (unsigned long long)gridDim.x * blockDim.x) {
    float4 r = div4(tree<MODE, 5, 0>(p, v), 32.f);
#pragma unroll
    for (int j = 0; j < NOUT; ++j) st<MODE>(p.out[j] + v, r);
  }
}

template <int LEVEL, int IDX>
__device__ __forceinline__ float4 tree_x(const float4 (&x)[NIN]) {
  if constexpr (LEVEL == 0) {
    return x[IDX];
  } else {
    return add4(tree_x<LEVEL - 1, 2 * IDX>(x), tree_x<LEVEL - 1, 2 * IDX + 1>(x));
  }
}

// batch: every input's vector loaded before the first add
__global__ void __launch_bounds__(256) k_batch(const __grid_constant__ P p) {
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.nvec;
       v += (unsigned long long)gridDim.x * blockDim.x) {
    float4 x[NIN];
#pragma unroll
    for (int i = 0; i < NIN; ++i) x[i] = ld<0>(p.in[i] + v);
    float4 r = div4(tree_x<5, 0>(x), 32.f);
#pragma unroll
    for (int j = 0; j < NOUT; ++j) p.out[j][v] = r;
  }
}

// pair: two vectors per thread, 16 inputs at a time for both
__global__ void __launch_bounds__(256) k_pair(const __grid_constant__ P p) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.nvec;
       v += 2 * stride) {
    const unsigned long long w = v + stride;
    const bool hw = w < p.nvec;
    float4 h[2][2];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float4 a[16], b[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a[i] = ld<0>(p.in[half * 16 + i] + v);
        b[i] = hw ? ld<0>(p.in[half * 16 + i] + w) : make_float4(0, 0, 0, 0);
      }
      // perfect subtree of 16 over a[] and b[]
#pragma unroll
      for (int s = 8; s >= 1; s >>= 1)
#pragma unroll
        for (int i = 0; i < s; ++i) {
          a[i] = add4(a[2 * i], a[2 * i + 1]);
          b[i] = add4(b[2 * i], b[2 * i + 1]);
        }
      h[0][half] = a[0];
      h[1][half] = b[0];
    }
    const float4 ra = div4(add4(h[0][0], h[0][1]), 32.f);
#pragma unroll
    for (int j = 0; j < NOUT; ++j) p.out[j][v] = ra;
    if (hw) {
      const float4 rb = div4(add4(h[1][0], h[1][1]), 32.f);
#pragma unroll
      for (int j = 0; j < NOUT; ++j) p.out[j][w] = rb;
    }
  }
}

// read ceiling
__global__ void __launch_bounds__(256) k_read(const __grid_constant__ P p) {
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.nvec;
       v += (unsigned long long)gridDim.x * blockDim.x) {
    float4 r = tree<0, 5, 0>(p, v);
    if (r.x == 1234.5f && r.y == -1.f) p.out[0][v] = r;  // never true for the data
  }
}

// copy ceiling
__global__ void __launch_bounds__(256) k_copy(const __grid_constant__ P p) {
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < p.nvec;
       v += (unsigned long long)gridDim.x * blockDim.x)
    p.out[0][v] = ld<0>(p.in[0] + v);
}

struct __align__(32) F8v { float4 a, b; };

template <int MODE>
__device__ __forceinline__ F8v ld8(const F8v *p) {
  F8v v;
  if constexpr (MODE == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y),
                   "=f"(v.b.z), "=f"(v.b.w) : "l"(p));
  } else if constexpr (MODE == 1) {
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y),
          "=f"(v.b.z), "=f"(v.b.w) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y),
          "=f"(v.b.z), "=f"(v.b.w) : "l"(p));
  }
  return v;
}
template <int SMODE = 0>
__device__ __forceinline__ void st8(F8v *p, const F8v &v) {
  if constexpr (SMODE == 0) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.a.x), "f"(v.a.y),
                 "f"(v.a.z), "f"(v.a.w), "f"(v.b.x), "f"(v.b.y), "f"(v.b.z), "f"(v.b.w)
                 : "memory");
  } else {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.a.x), "f"(v.a.y),
                 "f"(v.a.z), "f"(v.a.w), "f"(v.b.x), "f"(v.b.y), "f"(v.b.z), "f"(v.b.w)
                 : "memory");
  }
}
__device__ __forceinline__ F8v add8(const F8v &x, const F8v &y) { return F8v{add4(x.a, y.a), add4(x.b, y.b)}; }

template <int MODE, int LEVEL, int IDX>
__device__ __forceinline__ F8v tree8(const P &p, unsigned long long v) {
  if constexpr (LEVEL == 0) {
    return ld8<MODE>(reinterpret_cast<const F8v *>(p.in[IDX]) + v);
  } else {
    const F8v a = tree8<MODE, LEVEL - 1, 2 * IDX>(p, v);
    const F8v b = tree8<MODE, LEVEL - 1, 2 * IDX + 1>(p, v);
    return add8(a, b);
  }
}

template <int MODE, int SMODE = 0>
__global__ void __launch_bounds__(256) k_tree8(const __grid_constant__ P p) {
  const unsigned long long n8 = p.nvec / 2;
  for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < n8;
       v += (unsigned long long)gridDim.x * blockDim.x) {
    F8v r = tree8<MODE, 5, 0>(p, v);
    r.a = div4(r.a, 32.f);
    r.b = div4(r.b, 32.f);
#pragma unroll
    for (int j = 0; j < NOUT; ++j) st8<SMODE>(reinterpret_cast<F8v *>(p.out[j]) + v, r);
  }
}

__global__ void fill(float *x, size_t n, unsigned seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed * 40503u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    x[i] = (float)(h & 0xffff) / 65536.f - 0.5f;
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float *> in(NIN), out(NOUT);
  for (int i = 0; i < NIN; ++i) {
    CK(cudaMalloc(&in[i], D * 4));
    fill<<<4 * sms, 256>>>(in[i], D, i + 1);
  }
  for (int j = 0; j < NOUT; ++j) CK(cudaMalloc(&out[j], D * 4));
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const unsigned long long nvec = BUCKET / 4;

  auto run = [&](const char *name, int nin, int nout, int grid, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      CK(cudaEventRecord(a));
      for (int k = 0; k < K; ++k) {
        P p;
        for (int i = 0; i < NIN; ++i) p.in[i] = (const float4 *)(in[i] + (size_t)k * BUCKET);
        for (int j = 0; j < NOUT; ++j) p.out[j] = (float4 *)(out[j] + (size_t)k * BUCKET);
        p.nvec = nvec;
        p.inv = 1.f / 32;
        launch(grid, p);
      }
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (rep > 0 && ms < best) best = ms;
    }
    const double bytes = (double)(nin + nout) * BUCKET * 4 * K;
    printf("{\"variant\": \"%s\", \"grid\": %d, \"ms_per_pass\": %.4f, \"us_per_launch\": %.2f, \"gbs\": %.1f}\n",
           name, grid, best, best * 1e3 / K, bytes / (best * 1e-3) / 1e9);
    fflush(stdout);
  };
  const char *only = getenv("PROBE_ONLY");
  if (only) {  // the follow-up: 256-bit loads with streaming stores, larger grids
    const int grids2[] = {sms * 3, sms * 6, sms * 12, sms * 16, sms * 24, sms * 32};
    for (int g : grids2) {
      run("w256", 32, 8, g, [](int grid, const P &p) { k_tree8<1, 0><<<grid, 256>>>(p); });
      run("w256cs", 32, 8, g, [](int grid, const P &p) { k_tree8<1, 1><<<grid, 256>>>(p); });
      run("w256vcs", 32, 8, g, [](int grid, const P &p) { k_tree8<0, 1><<<grid, 256>>>(p); });
      run("hint", 32, 8, g, [](int grid, const P &p) { k_tree<2><<<grid, 256>>>(p); });
      run("read", 32, 0, g, [](int grid, const P &p) { k_read<<<grid, 256>>>(p); });
    }
    return 0;
  }
  const int grids[] = {sms * 2, sms * 4, sms * 5, sms * 8, sms * 16};
  for (int g : grids) {
    run("base", 32, 8, g, [](int grid, const P &p) { k_tree<0><<<grid, 256>>>(p); });
    run("nv", 32, 8, g, [](int grid, const P &p) { k_tree<1><<<grid, 256>>>(p); });
    run("hint", 32, 8, g, [](int grid, const P &p) { k_tree<2><<<grid, 256>>>(p); });
    run("w256", 32, 8, g, [](int grid, const P &p) { k_tree8<0><<<grid, 256>>>(p); });
    run("w256nv", 32, 8, g, [](int grid, const P &p) { k_tree8<1><<<grid, 256>>>(p); });
    run("w256ef", 32, 8, g, [](int grid, const P &p) { k_tree8<2><<<grid, 256>>>(p); });
    run("batch", 32, 8, g, [](int grid, const P &p) { k_batch<<<grid, 256>>>(p); });
    run("pair", 32, 8, g, [](int grid, const P &p) { k_pair<<<grid, 256>>>(p); });
    run("read", 32, 0, g, [](int grid, const P &p) { k_read<<<grid, 256>>>(p); });
    run("copy", 1, 1, g, [](int grid, const P &p) { k_copy<<<grid, 256>>>(p); });
  }
  return 0;
}
