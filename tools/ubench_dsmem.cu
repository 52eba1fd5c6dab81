// Microbenchmark: distributed-shared-memory (cluster) atomics on B200 (sm_100a).
// fp64 add / u32 or / u32 CAS into random slots of a cluster-wide table
// (each CTA owns TPC doubles), vs the same ops into the CTA's own smem.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_dsmem tools/ubench_dsmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int kIters = 2048;
constexpr int TPC = 16384;  // doubles per CTA (128 KB)

template <int MODE>
__global__ void k_dsm(unsigned long long *sink, int local_only) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned ncta = cl.num_blocks();
  for (int i = threadIdx.x; i < TPC; i += blockDim.x) sm[i] = 0.0;
  cl.sync();
  uint32_t x = mix(threadIdx.x * 7919u + blockIdx.x * 104729u);
  const unsigned me = cl.block_rank();
  for (int it = 0; it < kIters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t s = (x >> 9) & (TPC - 1);
    const unsigned dst = local_only ? me : (x >> 2) % ncta;
    double *p = cl.map_shared_rank(sm, dst) + s;
    if (MODE == 0) atomicAdd(p, 1.0);
    else if (MODE == 1) atomicOr(reinterpret_cast<unsigned *>(p), 1u << (x & 31));
    else if (MODE == 2) atomicCAS(reinterpret_cast<unsigned *>(p), 0u, x | 1u);
    else if (MODE == 3) {  // red (no return) f64 add via PTX on the cluster address
      const unsigned a = (unsigned)__cvta_generic_to_shared(sm + s);
      unsigned ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(dst));
      asm volatile("red.shared::cluster.add.f64 [%0], %1;" :: "r"(ra), "d"(1.0) : "memory");
    }
  }
  cl.sync();
  if (sm[threadIdx.x] == -1.0) sink[0] = 1;
}

template <int MODE>
void run(const char *name, int csize, int local_only) {
  cudaLaunchConfig_t cfg = {};
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cfg.gridDim = dim3((sms / csize) * csize);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = TPC * 8;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k_dsm<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, TPC * 8);
  if (csize > 8) cudaFuncSetAttribute(k_dsm<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long *sink; cudaMalloc(&sink, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, k_dsm<MODE>, sink, local_only);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, k_dsm<MODE>, sink, local_only);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 3.0 * cfg.gridDim.x * 1024.0 * kIters;
  printf("%-28s cluster %2d %s: %s %8.1f Gop/s  %.2f op/clk/SM(1.9GHz)\n", name, csize,
         local_only ? "local " : "remote", e == cudaSuccess ? "ok" : cudaGetErrorString(e),
         ops / ms / 1e6, ops / ms / 1e6 / (cfg.gridDim.x * 1.9));
  cudaFree(sink);
}

int main() {
  for (int cs : {1, 2, 4, 8, 16}) {
    run<0>("atomicAdd f64 (generic)", cs, 0);
    run<3>("red.shared::cluster.f64", cs, 0);
    run<1>("atomicOr u32", cs, 0);
    run<2>("atomicCAS u32", cs, 0);
  }
  run<0>("atomicAdd f64 (generic)", 8, 1);
  run<3>("red.shared::cluster.f64", 8, 1);
  return 0;
}
