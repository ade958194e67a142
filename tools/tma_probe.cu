// Standalone probe: 1-D TMA tensor load of fp64 rows and plain bulk copy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                        const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const double *src, double *out, int coord) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(2048));
    if (MODE == 0)
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(su(buf)), "l"((unsigned long long)&tm), "r"(coord), "r"(su(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(buf)), "l"(src + coord), "r"(2048), "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su(&bar)));
  out[threadIdx.x] = buf[threadIdx.x];
}
int main(int argc, char **argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  int N = 100000;
  double *d, *o;
  cudaMalloc(&d, N * 8); cudaMalloc(&o, 256 * 8);
  std::vector<double> h(N); for (int i = 0; i < N; ++i) h[i] = i;
  cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
  void *f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  printf("entry %d q %d f %p\n", (int)e, (int)q, f);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)N, 1}; cuuint64_t str[2] = {0, 0}; cuuint32_t box[2] = {256, 1}; cuuint32_t es[2] = {1, 1};
  CUresult r = ((Enc)f)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int coord = 1000;
  if (mode == 0) k<0><<<1, 256>>>(m, d, o, coord); else k<1><<<1, 256>>>(m, d, o, coord);
  e = cudaDeviceSynchronize();
  printf("mode %d kernel %d (%s)\n", mode, (int)e, cudaGetErrorString(e));
  std::vector<double> ho(256); cudaMemcpy(ho.data(), o, 2048, cudaMemcpyDeviceToHost);
  printf("out[0]=%g out[255]=%g\n", ho[0], ho[255]);
  return 0;
}
