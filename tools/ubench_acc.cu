// Microbenchmark: fp64 scatter-accumulate primitives into an 8192-slot window
// (the column-tile part's dense window), 2 blocks x 512 threads per SM, each
// warp doing rounds of 32 adds.  Address patterns: 0 = 32 consecutive
// columns (dense run), 1 = uniform random columns, 2 = sorted random columns
// with mean gap 4 (a sparse B-row segment).  Variants:
//   0 atomicAdd(double) on smem  (ATOMS.CAST.SPIN.64 loop)
//   1 CAS guessing 0 first       (ATOMS.CAS.64, one round trip on a first touch)
//   2 plain LDS/DADD/STS          (racy: the no-atomic upper bound)
//   3 warp-private 512-slot windows, plain RMW (columns folded mod 512)
//   4 red.global.add.f64 into a per-block global window (L2 atomics)
//   5 atomicAdd(double) + atomicOr occupancy bit (the current dense path)
// Prints adds / clock / SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_acc ubench_acc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int W = 8192;

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

__global__ void kgen(unsigned *tab, int n, int sorted) {
  // R-MAT-like columns in [0, 8192): each bit set with probability 0.24;
  // sorted = 1: each group of 32 sorted (a B-row segment's round)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned x = 0, hh = hash32(i * 2654435761u + 17u);
  for (int bit = 0; bit < 13; ++bit) {
    hh = hash32(hh + bit);
    if ((hh & 1023) < 246) x |= 1u << bit;
  }
  unsigned c = x;
  if (sorted) {
    const int lane = threadIdx.x & 31;
    for (int k = 2; k <= 32; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        const unsigned o = __shfl_xor_sync(0xffffffffu, c, j);
        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
        c = (lower == up) ? min(c, o) : max(c, o);
      }
    // drop duplicates inside the round (a segment has distinct columns)
    const unsigned prev = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane > 0 && prev == c) c = (c + 4096u * (lane & 1) + lane) & 8191u;
  }
  tab[i] = c;
}

template <int VAR>
__global__ void __launch_bounds__(512, 2) kacc(int pattern, int rounds, double *gwin, double *sink,
                                               const unsigned *tab, int tabn) {
  extern __shared__ double win[];
  unsigned *bm = reinterpret_cast<unsigned *>(win + W);
  for (int s = threadIdx.x; s < W; s += 512) win[s] = 0.0;
  for (int s = threadIdx.x; s < W / 32; s += 512) bm[s] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  double *g = gwin + size_t(blockIdx.x) * W;
  for (int r = 0; r < rounds; ++r) {
    unsigned c;
    const unsigned rr = hash32(seed + r * 7919u);
    if (pattern == 0) c = ((hash32(w * 131 + r) & (W - 1)) & ~31u) + lane;
    else if (pattern == 1) c = rr & (W - 1);
    else if (pattern == 2) c = ((hash32(w * 131 + r) & (W - 1)) + 4 * lane + (rr & 3)) & (W - 1);
    else c = __ldg(tab + ((size_t(blockIdx.x) * 16 + w) * 32 * 61 + size_t(r) * 32 + lane) % tabn);
    const double v = 1.0 + (rr & 7);
    if (VAR == 0) atomicAdd(win + c, v);
    else if (VAR == 1) {
      unsigned long long *a = reinterpret_cast<unsigned long long *>(win + c);
      unsigned long long old = atomicCAS(a, 0ull, (unsigned long long)__double_as_longlong(v));
      while (old != 0ull) {
        const unsigned long long nw = (unsigned long long)__double_as_longlong(__longlong_as_double(old) + v);
        const unsigned long long x = atomicCAS(a, old, nw);
        if (x == old) break;
        old = x;
      }
    } else if (VAR == 2) {
      volatile double *p = win + c;
      *p = *p + v;
    } else if (VAR == 3) {
      volatile double *p = win + w * 512 + (c & 511);
      *p = *p + v;
    } else if (VAR == 4) {
      atomicAdd(g + c, v);  // result unused: RED.E.ADD.F64
    } else {
      atomicAdd(win + c, v);
      atomicOr(bm + (c >> 5), 1u << (c & 31));
    }
  }
  __syncthreads();
  double s = 0;
  for (int q = threadIdx.x; q < W; q += 512) s += win[q] + bm[q >> 5];
  if (s == 12345.678) sink[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  double *gwin, *sink;
  cudaMalloc(&gwin, size_t(2 * sms) * W * 8);
  cudaMemset(gwin, 0, size_t(2 * sms) * W * 8);
  cudaMalloc(&sink, 8);
  const int rounds = 4096;
  const int tabn = 1 << 24;
  unsigned *tab_u, *tab_s;
  cudaMalloc(&tab_u, size_t(tabn) * 4);
  cudaMalloc(&tab_s, size_t(tabn) * 4);
  kgen<<<tabn / 256, 256>>>(tab_u, tabn, 0);
  kgen<<<tabn / 256, 256>>>(tab_s, tabn, 1);
  const size_t smem = W * 8 + W / 8;
  cudaFuncSetAttribute(kacc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kacc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kacc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kacc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kacc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kacc<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char *vn[] = {"atomicAdd(f64) smem", "CAS-guess-0 (ATOMS.CAS.64)", "plain RMW (racy bound)",
                      "warp-private window RMW", "red.global.add.f64 (L2)", "atomicAdd + atomicOr bit"};
  const char *pn[] = {"dense run", "uniform random", "sorted gap 4", "rmat bits", "rmat sorted seg"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int var = 0; var < 6; ++var)
    for (int pat = 0; pat < 5; ++pat) {
      auto launch = [&]() {
        switch (var) {
          case 0: kacc<0><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
          case 1: kacc<1><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
          case 2: kacc<2><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
          case 3: kacc<3><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
          case 4: kacc<4><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
          default: kacc<5><<<2 * sms, 512, smem>>>(pat, rounds, gwin, sink, pat == 3 ? tab_u : tab_s, tabn); break;
        }
      };
      launch();
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double adds = 5.0 * 2 * sms * 512.0 * rounds;
      const double per_clk_sm = adds / (ms * 1e-3) / (sms * clk * 1e3);
      printf("%-30s %-15s %8.3f ms  %6.2f adds/clk/SM\n", vn[var], pn[pat], ms / 5, per_clk_sm);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
