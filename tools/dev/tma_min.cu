// Minimal TMA 2-D box load test (same descriptor shape as the tile kernel's prefetch).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -o tools/dev/tma_min tools/dev/tma_min.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int x, int y) {
  extern __shared__ __align__(16) float raw[];
  float* sm = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    if (MODE & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(28 * 27 * 4) : "memory");
    if (MODE & 4) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(sm)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x), "r"(y), "r"(su32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(su32(&bar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < 28 * 27; i += blockDim.x) out[i] = sm[i];
}

template <int M>
int run(int cluster) {
  const int cols = 4124, rows = 90;
  float* g;
  cudaMalloc(&g, cols * rows * 4);
  float* h = new float[cols * rows];
  for (int i = 0; i < cols * rows; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, cols * rows * 4, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 28 * 27 * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {28, 27}, es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  cudaError_t e;
  float r[28 * 27];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 8192;
  cudaLaunchAttribute attr[1];
  if (cluster) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
  }
  const int X = getenv("TX") ? atoi(getenv("TX")) : 4120, Y = getenv("TY") ? atoi(getenv("TY")) : 60;
  if (getenv("CHEV")) {
    k<M><<<1, 128, 8192>>>(tm, out, X, Y);
    e = cudaGetLastError();
  } else {
    e = cudaLaunchKernelEx(&cfg, k<M>, tm, out, X, Y);
  }
  printf("xy %d %d ", X, Y);
  printf("launchEx issue: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("launchEx (OOB right/bottom): %s\n", cudaGetErrorString(e));
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  printf("out[0]=%g expect %g  out[5]=%g expect 0\n", r[0], (float)(60 * cols + 4120), r[5]);
  return 0;
}

int main(int argc, char** argv) {
  const int mode = atoi(argv[1]), cluster = atoi(argv[2]);
  printf("mode %d cluster %d\n", mode, cluster);
  switch (mode) {
    case 0: return run<0>(cluster);
    case 1: return run<1>(cluster);
    case 2: return run<2>(cluster);
    case 3: return run<3>(cluster);
    case 4: return run<4>(cluster);
    case 7: return run<7>(cluster);
  }
  return 0;
}
