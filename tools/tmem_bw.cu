// TMEM <-> register bandwidth microbenchmark (tcgen05.ld / tcgen05.st, sm_100a).
// One CTA per SM, W warps; each warp repeatedly moves 32 lanes x NCOL columns (32-bit)
// between TMEM and registers.  Prints bytes/clock/SM for loads and for stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NCOL = 32;   // columns per ld/st (x32)
constexpr int REPS = 4096;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tmem_kernel(long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase;
  // lane quarter of this warp, and a column slice per warp of the same quarter
  const uint32_t lane_q = (warp & 3) * 32;
  const uint32_t col0 = (warp >> 2) * NCOL * 2 % 512;
  const uint32_t taddr = base + (lane_q << 16) + col0;
  uint32_t r[NCOL];
#pragma unroll
  for (int i = 0; i < NCOL; ++i) r[i] = threadIdx.x * 7u + i;
  // --- stores
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < REPS; ++it) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  long long t1 = clock64();
  // --- loads
  uint32_t acc = 0;
  for (int it = 0; it < REPS; ++it) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr + (it & 1) * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    acc += r[it & 31];
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    cycles[blockIdx.x * 2 + 0] = t1 - t0;
    cycles[blockIdx.x * 2 + 1] = t2 - t1;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = static_cast<float>(acc);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

template <int WARPS>
void run() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sms * 2 * sizeof(long long));
  cudaMalloc(&sink, sms * WARPS * 32 * sizeof(float));
  tmem_kernel<WARPS><<<sms, WARPS * 32>>>(cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[2];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = double(WARPS) * 32 * NCOL * 4 * REPS;
  printf("{\"warps\": %d, \"st_bytes_per_clk_per_sm\": %.1f, \"ld_bytes_per_clk_per_sm\": %.1f, "
         "\"st_cycles\": %lld, \"ld_cycles\": %lld}\n",
         WARPS, bytes / h[0], bytes / h[1], h[0], h[1]);
}

int main() {
  run<4>();
  run<8>();
  run<16>();
  return 0;
}
