// Bisect TMA usage patterns: A = map after a 256-byte struct param,
// B = dynamic smem destination, C = 4 boxes per barrier + ring reuse.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                        const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);
struct Big { double a[32]; };
#ifndef ODD
#define ODD 1
#endif
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int A, int B, int C>
__global__ void k(const Big big, const __grid_constant__ CUtensorMap tm, double *out, int coord) {
  extern __shared__ unsigned char dyn[];
  __shared__ __align__(128) double sbuf[4 * 256];
  __shared__ __align__(8) unsigned long long bar[2];
  double *buf = B ? reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(dyn) + 127) & ~(uintptr_t)127) : sbuf;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbox = C ? 4 : 1;
  double acc = 0;
  for (int it = 0; it < (C ? 6 : 1); ++it) {
    const int st = it & 1;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(2048 * nbox));
      for (int b = 0; b < nbox; ++b)
        asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                     ::"r"(su(buf + (st * 2 + (b & 1)) * 256 * (C ? 1 : 0) + b * 0)), "l"((unsigned long long)&tm), "r"(coord + 256 * b + (ODD ? it : 2 * it)), "r"(su(&bar[st])) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su(&bar[st])), "r"((it >> 1) & 1));
    acc += buf[st * 512 * (C ? 1 : 0) + threadIdx.x];
    __syncthreads();
  }
  out[threadIdx.x] = acc + big.a[0];
}
int main(int argc, char **argv) {
  int a = atoi(argv[1]), b = atoi(argv[2]), c = atoi(argv[3]);
  int N = 100000; double *d, *o; cudaMalloc(&d, N * 8); cudaMalloc(&o, 256 * 8);
  std::vector<double> h(N); for (int i = 0; i < N; ++i) h[i] = i; cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
  void *f; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMap m; cuuint64_t dims[1] = {(cuuint64_t)N}; cuuint64_t str[1] = {0}; cuuint32_t box[1] = {256}; cuuint32_t es[1] = {1};
  CUresult r = ((Enc)f)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  Big big{}; size_t dsm = 5 * 2048 + 128;
  void (*kp)(const Big, const CUtensorMap, double *, int) = nullptr;
  if (!a && !b && !c) kp = k<0,0,0>; if (a && !b && !c) kp = k<1,0,0>; if (!a && b && !c) kp = k<0,1,0>;
  if (!a && !b && c) kp = k<0,0,1>; if (a && b && c) kp = k<1,1,1>; if (!a && b && c) kp = k<0,1,1>;
  cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  kp<<<1, 256, dsm>>>(big, m, o, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("A%d B%d C%d encode %d -> %d (%s)\n", a, b, c, (int)r, (int)e, cudaGetErrorString(e));
  return 0;
}
