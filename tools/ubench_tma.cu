// ubench_tma.cu -- TMA bulk-copy (cp.async.bulk global->shared) ring throughput per SM on B200.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_tma tools/ubench_tma.cu
//
// One CTA per SM: a producer lane streams NSEG segments of SEG bytes from a source buffer
// into a STAGES-deep shared-memory ring; W consumer warps wait for each segment, touch one
// word of it, and release it.  Prints GB/s per SM and aggregate.  Measurement tool only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s line %d\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void k_ring(const char* src, size_t src_bytes, int nseg, int seg, int stages, int chunks,
                       double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* full = (unsigned long long*)sm;
  unsigned long long* empty = full + 16;
  char* buf = (char*)(sm + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, nw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nw) {
    if (lane == 0) {
      for (int q = 0; q < nseg; ++q) {
        const int st = q % stages;
        mbar_wait(empty + st, ((q / stages) & 1) ^ 1);
        mbar_expect_tx(full + st, seg);
        const size_t off = ((size_t)q * seg) % src_bytes;
        // `chunks` bulk copies per segment (same total bytes)
        for (int c = 0; c < chunks; ++c)
          bulk_g2s(buf + (size_t)st * seg + (size_t)c * (seg / chunks), src + off + (size_t)c * (seg / chunks),
                   seg / chunks, full + st);
      }
    }
    return;
  }
  double acc = 0;
  for (int q = 0; q < nseg; ++q) {
    const int st = q % stages;
    mbar_wait(full + st, (q / stages) & 1);
    acc += ((const double*)(buf + (size_t)st * seg))[lane + 32 * warp];
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* src;
  double* out;
  const size_t big = (size_t)1 << 30;
  CK(cudaMalloc(&src, big));
  CK(cudaMemset(src, 1, big));
  CK(cudaMalloc(&out, (size_t)sms * 1024 * 8));
  CK(cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("src_MB seg_KB stages chunks warps  us/seg  GB/s/SM  GB/s_total\n");
  struct C { size_t src; int seg, stages, chunks, warps; };
  C cs[] = {{8 << 20, 32768, 4, 1, 16}, {8 << 20, 32768, 2, 1, 16}, {8 << 20, 32768, 6, 1, 16},
            {8 << 20, 16384, 8, 1, 16}, {8 << 20, 65536, 3, 1, 16}, {8 << 20, 32768, 4, 4, 16},
            {8 << 20, 32768, 4, 8, 16}, {8 << 20, 8192, 16, 1, 16}, {big, 32768, 4, 1, 16},
            {8 << 20, 32768, 4, 1, 4}, {64 << 20, 32768, 4, 1, 16}};
  for (C c : cs) {
    const int nseg = 2048;
    size_t smem = 256 * 8 + (size_t)c.seg * c.stages;
    int block = 32 * (c.warps + 1);
    k_ring<<<sms, block, smem>>>(src, c.src, nseg, c.seg, c.stages, c.chunks, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_ring<<<sms, block, smem>>>(src, c.src, nseg, c.seg, c.stages, c.chunks, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per_sm = (double)nseg * c.seg / (ms * 1e-3) / 1e9;
    printf("%6zu %6d %6d %6d %5d  %6.2f  %7.1f  %9.0f\n", c.src >> 20, c.seg / 1024, c.stages, c.chunks,
           c.warps, ms * 1e3 / nseg, per_sm, per_sm * sms);
  }
  return 0;
}
