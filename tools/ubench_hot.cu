// ubench_hot.cu -- L2 retention of a hot gather region under cold-gather + streaming pressure.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_hot tools/ubench_hot.cu
//
// 1 Gi random labels: a fraction `hot` uniform in [0, H) (the hot region), the rest uniform in
// [H, 64 Mi) (cold); 8-byte gathers from a 512 MiB vector, index stream read once
// (evict_first).  Hot gathers use an L2 evict_last (or normal) policy, cold evict_first (or
// normal).  Prints G gathers/s per configuration.  Measurement tool only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void k_fill(uint32_t* idx, long long n, uint32_t H, uint32_t V, float hot) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t a = hash32((uint32_t)i * 2654435761u + 7u), b = hash32((uint32_t)i + 0x9e3779b9u);
    const bool h = (a & 0xffffff) < (uint32_t)(hot * 16777216.f);
    idx[i] = h ? b % H : H + b % (V - H);
  }
}
// MODE 0: hot evict_last, cold evict_first; 1: no hints; 2: hot evict_last, cold
// evict_unchanged; 3: plain loads inside a persisting access-policy window over [0, H)
template <int MODE>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ idx, long long n4,
                                                 const double* __restrict__ x, uint32_t H, double* out) {
  unsigned long long pl, pf, pu;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pu));
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 u;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(idx + 4 * i), "l"(pf));
    const uint32_t l[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double v;
      if (MODE == 0 || MODE == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(v) : "l"(x + l[q]), "l"(l[q] < H ? pl : (MODE == 0 ? pf : pu)));
      } else {
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + l[q]));
      }
      acc += v;
    }
  }
  out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long NI = 1ll << 30;
  const uint32_t V = 1u << 26;
  uint32_t* idx; double *x, *out;
  CK(cudaMalloc(&idx, NI * 4)); CK(cudaMalloc(&x, (size_t)V * 8)); CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * 8));
  CK(cudaMemset(x, 0, (size_t)V * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("H_MB hot_frac mode  ms  Ggather/s\n");
  for (uint32_t hmb : {8u, 24u, 40u, 56u}) {
    for (float hot : {0.77f}) {
      const uint32_t H = hmb * 131072u;
      k_fill<<<sms * 8, 256>>>(idx, NI, H, V, hot);
      CK(cudaDeviceSynchronize());
      for (int mode = 0; mode < 4; ++mode) {
        cudaStreamAttrValue v{};
        if (mode == 3) {
          int maxp = 0;
          cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
          v.accessPolicyWindow.base_ptr = x;
          v.accessPolicyWindow.num_bytes = (size_t)H * 8;
          v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxp / (float)((size_t)H * 8));
          v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
          cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &v);
        }
        auto run = [&] {
          if (mode == 0) k_gather<0><<<sms * 8, 256>>>(idx, NI / 4, x, H, out);
          else if (mode == 2) k_gather<2><<<sms * 8, 256>>>(idx, NI / 4, x, H, out);
          else k_gather<1><<<sms * 8, 256>>>(idx, NI / 4, x, H, out);
        };
        run();
        cudaEventRecord(e0); run(); run(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1); ms /= 2;
        if (mode == 3) {
          v.accessPolicyWindow.num_bytes = 0;
          cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &v);
          cudaCtxResetPersistingL2Cache();
        }
        const char* names[4] = {"hints", "plain", "unchg", "persist"};
        printf("%4u %.2f %s %7.3f %6.1f\n", hmb, hot, names[mode], ms, NI / ms / 1e6);
        fflush(stdout);
      }
    }
  }
  return 0;
}
