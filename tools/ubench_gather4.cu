// ubench_gather4.cu -- can TMA tile::gather4 beat the one-L1-wavefront-per-gather ceiling of
// random 8-byte LDG gathers (~281-291 G/s, the L1tex wavefront rate)?
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/ug4 tools/ubench_gather4.cu
//   /tmp/ug4
//
// x: V doubles viewed as a 2-D tensor of V/2 rows x 2 columns (16-byte rows, the TMA minimum).
// (a) LDG: every thread gathers x[label] for a stream of random labels (the k_tiles pattern);
// (b) gather4: per CTA, W producer lanes each keep a ring of D in-flight
//     cp.async.bulk.tensor.2d...tile::gather4 ops (4 random rows = 64 bytes each, one mbarrier
//     per op), and sum the wanted half of every row from shared memory.
// Reported: gathered labels per second.  Measurement tool only -- not part of libpsi.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s line %d\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_ldg(const double* __restrict__ x, uint32_t V, long long n_per_thread, double* out) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (long long i = 0; i < n_per_thread; i += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t l = hash32((uint32_t)(tid * 1315423911ull + i + q)) % V;
      v[q] = __ldcg(x + l);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];
  }
  out[tid] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int kW = 8;        // producer warps per CTA (lane 0 of each issues)
constexpr int kD = 32;       // ops in flight per producer

__global__ void __launch_bounds__(kW * 32) k_gather4(const __grid_constant__ CUtensorMap map,
                                                     uint32_t rows, long long ops_per_producer,
                                                     double* out) {
  __shared__ __align__(128) double buf[kW][kD][16];     // 4 rows x 2 doubles per op (128-B slots)
  __shared__ __align__(8) unsigned long long bar[kW][kD];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
  if (lane == 0) {
    for (int d = 0; d < kD; ++d)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][d])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t seed = (blockIdx.x * kW + w) * 2654435761u;
    long long issued = 0, done = 0;
    uint32_t phase[kD];
    for (int d = 0; d < kD; ++d) phase[d] = 0;
    auto issue = [&](int d, long long k) {
      const uint32_t h = hash32(seed + (uint32_t)k * 4u);
      const int r0 = hash32(h + 1) % rows, r1 = hash32(h + 2) % rows, r2 = hash32(h + 3) % rows,
                r3 = hash32(h + 4) % rows;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" :: "r"(smem_u32(&bar[w][d])) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          :: "r"(smem_u32(&buf[w][d][0])), "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
             "r"(smem_u32(&bar[w][d]))
          : "memory");
    };
    for (; issued < kD && issued < ops_per_producer; ++issued) issue((int)issued, issued);
    while (done < ops_per_producer) {
      const int d = (int)(done % kD);
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra W_%=;\n}\n" :: "r"(smem_u32(&bar[w][d])), "r"(phase[d]) : "memory");
      phase[d] ^= 1u;
      s += buf[w][d][0] + buf[w][d][3] + buf[w][d][4] + buf[w][d][7];
      ++done;
      if (issued < ops_per_producer) { issue(d, issued); ++issued; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = (EncodeFn)fn;
  for (uint32_t V : {1u << 20, 1u << 23, 1u << 26}) {          // 8 MB, 64 MB, 512 MB of x
    double *x = nullptr, *out = nullptr;
    CK(cudaMalloc(&x, (size_t)V * 8));
    CK(cudaMemset(x, 0, (size_t)V * 8));
    CK(cudaMalloc(&out, (size_t)sms * 8 * 1024 * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // (a) LDG
    const int thr = 1024, blocks = sms;
    const long long per = 4096;
    k_ldg<<<blocks, thr>>>(x, V, per, out);
    cudaEventRecord(e0);
    k_ldg<<<blocks, thr>>>(x, V, per, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double g_ldg = (double)blocks * thr * per / (ms * 1e-3) / 1e9;
    // (b) gather4
    CUtensorMap map;
    cuuint64_t dims[2] = {2, V / 2};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    for (int ctas_per_sm : {1, 2, 4}) {
      const long long ops = 20000;
      k_gather4<<<sms * ctas_per_sm, kW * 32>>>(map, V / 2, ops, out);
      CK(cudaGetLastError());
      cudaEventRecord(e0);
      k_gather4<<<sms * ctas_per_sm, kW * 32>>>(map, V / 2, ops, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double g4 = (double)sms * ctas_per_sm * kW * ops * 4 / (ms * 1e-3) / 1e9;
      printf("x %4u MB  LDG random 8B: %6.1f G/s   gather4 (%d CTA/SM x %d producers x %d in flight): %6.1f G rows/s\n",
             V / 131072, g_ldg, ctas_per_sm, kW, kD, g4);
    }
    cudaFree(x);
    cudaFree(out);
  }
  return 0;
}
