// Read-bandwidth ceilings for the DSE record stream (development tool).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o membench profiles/tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// minimal TMA bulk-copy helpers (cp.async.bulk + mbarrier)
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(smem_addr(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* d, const void* s, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(d)), "l"(s), "r"(bytes), "r"(smem_addr(b)) : "memory");
}
constexpr int kRec = 29232 / 8;  // doubles per record (E + meta)

__global__ void k_vec(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i); s += v.x + v.y;
  }
  if (s == 1234.5) out[0] = s;
}
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_chunk(const double* __restrict__ rec, double* out) {
  __shared__ double pad[2048];
  const double* R = rec + (size_t)blockIdx.x * kRec;
  double s = 0;
#pragma unroll
  for (int k = 0; k < 27; ++k) s += R[k * 128 + threadIdx.x];
  const int* M = reinterpret_cast<const int*>(R + 27 * 128);
  s += M[threadIdx.x] + M[128 + threadIdx.x] + M[256 + threadIdx.x];
  pad[threadIdx.x] = s;
  __syncthreads();
  if (pad[(threadIdx.x + 1) & 127] == 1234.5) out[0] = s;
}
__global__ void __launch_bounds__(128) k_chunk_tma(const double* __restrict__ rec, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ alignas(8) uint64_t bar;
  const double* R = rec + (size_t)blockIdx.x * kRec;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); mbar_arrive_expect_tx(&bar, kRec * 8); bulk_g2s(sm, R, kRec * 8, &bar); }
  __syncthreads();
  mbar_wait(&bar, 0);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 27; ++k) s += sm[k * 128 + threadIdx.x];
  if (s == 1234.5) out[0] = s;
}
template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaEventRecord(a); for (int r = 0; r < 10; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}
int main() {
  const int nch = 40000;  // ~venice
  const size_t bytes = (size_t)nch * kRec * 8;
  double *rec, *out; cudaMalloc(&rec, bytes); cudaMalloc(&out, 8); cudaMemset(rec, 0, bytes);
  float t;
  t = timeit([&] { k_vec<<<148 * 16, 256>>>((const double2*)rec, bytes / 16, out); });
  printf("vec  read %.1f GB/s\n", bytes / t / 1e6);
  t = timeit([&] { k_chunk<5><<<nch, 128>>>(rec, out); }); printf("chunk5 read %.1f GB/s\n", bytes / t / 1e6);
  t = timeit([&] { k_chunk<8><<<nch, 128>>>(rec, out); }); printf("chunk8 read %.1f GB/s\n", bytes / t / 1e6);
  t = timeit([&] { k_chunk<12><<<nch, 128>>>(rec, out); }); printf("chunk12 read %.1f GB/s\n", bytes / t / 1e6);
  cudaFuncSetAttribute(k_chunk_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kRec * 8);
  t = timeit([&] { k_chunk_tma<<<nch, 128, kRec * 8>>>(rec, out); }); printf("chunk_tma read %.1f GB/s\n", bytes / t / 1e6);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
