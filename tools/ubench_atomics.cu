// Microbenchmarks of the accumulator primitives on B200 (sm_100a):
// shared-memory LDS/STS, ATOMS.CAS, atomicOr, fp64 add (CAS loop), 32-bit
// add; global RED.F64 / ATOMG.CAS on L2-resident and DRAM-resident tables.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

constexpr int kIters = 4096;

template <int MODE>
__global__ void k_smem(int tsize_log, unsigned long long *sink) {
  extern __shared__ uint32_t sm[];
  double *smd = reinterpret_cast<double *>(sm);
  const int T = 1 << tsize_log;
  for (int i = threadIdx.x; i < T; i += blockDim.x) { if (MODE == 3 || MODE == 5) smd[i] = 0; else sm[i] = 0; }
  __syncthreads();
  uint32_t x = mix(threadIdx.x * 7919u + blockIdx.x * 104729u);
  unsigned long long acc = 0;
  const uint32_t m = T - 1;
  for (int it = 0; it < kIters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t s = (x >> 8) & m;
    if (MODE == 0) { acc += sm[s]; }                                   // LDS
    else if (MODE == 1) { acc += atomicCAS(sm + s, 0u, x); }           // ATOMS.CAS
    else if (MODE == 2) { acc += atomicOr(sm + s, 1u << (x & 31)); }   // ATOMS.OR
    else if (MODE == 3) { atomicAdd(smd + s, 1.0); }                   // fp64 add (CAS loop)
    else if (MODE == 4) { atomicAdd(sm + s, 1u); }                     // ATOMS.ADD (no return)
    else if (MODE == 5) { smd[s] += 1.0; }                             // plain RMW fp64 (racy)
    else if (MODE == 6) { sm[s] = x; }                                 // STS
  }
  if (acc == 12345) sink[0] = acc;
  if (MODE == 3 || MODE == 5) { if (smd[threadIdx.x & m] == -1.0) sink[1] = 1; }
}

template <int MODE>
__global__ void k_gmem(uint32_t *keys, double *vals, uint64_t mask, unsigned long long *sink) {
  uint32_t x = mix(threadIdx.x * 7919u + blockIdx.x * 104729u);
  unsigned long long acc = 0;
  for (int it = 0; it < kIters / 4; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint64_t s = (uint64_t(x) * 2654435761ull) & mask;
    if (MODE == 0) atomicAdd(vals + s, 1.0);                         // RED.F64
    else if (MODE == 1) acc += atomicCAS(keys + s, 0xFFFFFFFFu, x);  // ATOMG.CAS
    else if (MODE == 2) acc += __ldcg(keys + s);                     // LDG (L2)
  }
  if (acc == 12345) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock attr %d kHz\n", sms, clk);
  const char *names[] = {"LDS", "ATOMS.CAS", "ATOMS.OR", "fp64 atomicAdd(smem)", "ATOMS.ADD u32",
                         "plain fp64 RMW", "STS"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int tl : {12, 14}) {
      for (int threads : {256, 1024}) {
        size_t smem = (mode == 3 || mode == 5) ? (size_t(8) << tl) : (size_t(4) << tl);
        int blocks_per_sm = threads == 256 ? 4 : 1;
        auto launch = [&]() {
          switch (mode) {
            case 0: k_smem<0><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 1: k_smem<1><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 2: k_smem<2><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 3: k_smem<3><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 4: k_smem<4><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 5: k_smem<5><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
            case 6: k_smem<6><<<sms * blocks_per_sm, threads, smem>>>(tl, sink); break;
          }
        };
        launch();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = double(sms) * blocks_per_sm * threads * kIters;
        printf("smem %-22s T=2^%d thr=%4d x%d: %8.1f Gop/s  %.2f op/clk/SM (at 1.9GHz)\n", names[mode], tl,
               threads, blocks_per_sm, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
      }
    }
  }
  const char *gn[] = {"RED.F64", "ATOMG.CAS", "LDG.CG"};
  for (int mode = 0; mode < 3; ++mode) {
    for (uint64_t bytes : {uint64_t(16) << 20, uint64_t(64) << 20, uint64_t(4) << 30}) {
      uint64_t n = bytes / 8;
      uint32_t *keys;
      double *vals;
      cudaMalloc(&keys, n * 4);
      cudaMalloc(&vals, n * 8);
      cudaMemset(keys, 0xFF, n * 4);
      cudaMemset(vals, 0, n * 8);
      uint64_t mask = n - 1;
      auto launch = [&]() {
        if (mode == 0) k_gmem<0><<<sms * 8, 256>>>(keys, vals, mask, sink);
        else if (mode == 1) k_gmem<1><<<sms * 8, 256>>>(keys, vals, mask, sink);
        else k_gmem<2><<<sms * 8, 256>>>(keys, vals, mask, sink);
      };
      launch();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = double(sms) * 8 * 256 * (kIters / 4);
      printf("gmem %-10s table %6.0f MB: %8.1f Gop/s\n", gn[mode], n * 8.0 / 1048576, ops / ms / 1e6);
      cudaFree(keys);
      cudaFree(vals);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
