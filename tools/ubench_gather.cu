// ubench_gather.cu -- ceilings for the Power-psi sweep's random 8-byte gathers on B200.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench tools/ubench_gather.cu
//   ./ubench            (prints one line per variant: Ggathers/s and index-stream GB/s)
//
// A stream of NI random u32 labels (> L2, read once with 128-bit evict_first loads) drives
// 8-byte gathers from a vector x of V doubles held in (a) global memory (L2/HBM), (b) the
// CTA's shared memory, (c) a thread-block cluster's distributed shared memory.  The sum is
// written per thread so nothing is dead code.  Measurement tool only -- not part of libpsi.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s line %d\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// labels: uniform in [0, V) or skewed (label = floor(V * u^k)), k > 1 concentrates on small labels
__global__ void k_fill(uint32_t* idx, long long n, uint32_t V, float skew, uint32_t seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint32_t h = hash32((uint32_t)i * 2654435761u + seed);
    double u = (h + 0.5) / 4294967296.0;
    double v = skew > 1.f ? pow(u, (double)skew) : u;
    uint32_t l = (uint32_t)(v * V);
    idx[i] = l < V ? l : V - 1;
  }
}

__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint4 ld_stream4(const uint32_t* p, unsigned long long pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_na(const double* p) {
  double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}

// MODE 0: global, default caching (L1 allocate); 1: global, L1::no_allocate; 2: shared memory
template <int MODE, int UNROLL>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ idx, long long n4,
                                                 const double* __restrict__ x, uint32_t V, double* out) {
  extern __shared__ double sx[];
  if (MODE == 2) {
    for (uint32_t i = threadIdx.x; i < V; i += blockDim.x) sx[i] = x[i];
    __syncthreads();
  }
  const unsigned long long pf = pol_first();
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n4; i += UNROLL * stride) {
    uint4 u[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) u[k] = ld_stream4(idx + 4 * (i + k * stride), pf);
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t l[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (MODE == 0) acc += __ldg(x + l[q]);
        else if (MODE == 1) acc += ld_na(x + l[q]);
        else acc += sx[l[q]];
      }
    }
  }
  for (; i < n4; i += stride) {
    uint4 u = ld_stream4(idx + 4 * i, pf);
    const uint32_t l[4] = {u.x, u.y, u.z, u.w};
    for (int q = 0; q < 4; ++q) acc += MODE == 2 ? sx[l[q]] : __ldg(x + l[q]);
  }
  out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

// distributed shared memory: cluster of CS CTAs, each holds V/CS doubles; label l lives in
// CTA l / per at offset l % per.
template <int UNROLL>
__global__ void __launch_bounds__(256) k_gather_dsmem(const uint32_t* __restrict__ idx, long long n4,
                                                       const double* __restrict__ x, uint32_t V,
                                                       uint32_t per, double* out) {
  extern __shared__ double sx[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t r = cl.block_rank();
  for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) sx[i] = x[r * per + i];
  cl.sync();
  const unsigned long long pf = pol_first();
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n4; i += UNROLL * stride) {
    uint4 u[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) u[k] = ld_stream4(idx + 4 * (i + k * stride), pf);
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t l[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t rk = l[q] / per, off = l[q] - rk * per;
        const double* p = cl.map_shared_rank(sx, rk);
        acc += p[off];
      }
    }
  }
  cl.sync();
  out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long NI = 1ll << 30;            // 1 Gi labels = 4 GiB stream
  uint32_t* idx;
  double *x, *out;
  CK(cudaMalloc(&idx, NI * 4));
  CK(cudaMalloc(&x, (size_t)(1u << 26) * 8));   // up to 64 Mi doubles (512 MiB)
  CK(cudaMalloc(&out, (size_t)sms * 64 * 1024 * 8));
  CK(cudaMemset(x, 0, (size_t)(1u << 26) * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) -> float {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 3;
  };
  const long long n4 = NI / 4;
  printf("variant V(doubles) skew blocks/SM ms Ggather/s idxGB/s\n");
  // index stream only (no gathers) reference: V = 1, smem
  struct Cfg { uint32_t V; float skew; };
  Cfg all[] = {{1u << 12, 1.f}, {1u << 14, 1.f}, {1u << 17, 1.f}, {1u << 20, 1.f}, {1u << 22, 1.f},
               {1u << 24, 1.f}, {1u << 26, 1.f}, {1u << 26, 4.f}, {1u << 26, 8.f}};
  // L2 capacity sweep: 16 .. 128 MiB uniform
  Cfg cap[] = {{2u << 20, 1.f}, {4u << 20, 1.f}, {5u << 20, 1.f}, {6u << 20, 1.f}, {7u << 20, 1.f},
               {8u << 20, 1.f}, {9u << 20, 1.f}, {10u << 20, 1.f}, {12u << 20, 1.f}, {14u << 20, 1.f}};
  const bool capmode = argc > 1;
  std::vector<Cfg> cfgs = capmode ? std::vector<Cfg>(cap, cap + 10) : std::vector<Cfg>(all, all + 9);
  for (Cfg c : cfgs) {
    k_fill<<<sms * 8, 256>>>(idx, NI, c.V, c.skew, 12345u);
    CK(cudaDeviceSynchronize());
    for (int mode = 0; mode < 2; ++mode) {
      for (int bps : {4}) {
        int grid = sms * bps;
        float ms = timeit([&] {
          if (mode == 0) k_gather<0, 4><<<grid, 256>>>(idx, n4, x, c.V, out);
          else k_gather<1, 4><<<grid, 256>>>(idx, n4, x, c.V, out);
        });
        CK(cudaGetLastError());
        printf("global%s %u %.0f %d %.3f %.1f %.0f\n", mode ? "_noL1" : "", c.V, c.skew, bps, ms,
               NI / ms / 1e6, NI * 4.0 / ms / 1e6);
      }
    }
    if (c.V <= (1u << 14)) {   // up to 128 KiB in smem
      size_t sm = (size_t)c.V * 8;
      CK(cudaFuncSetAttribute(k_gather<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      for (int bps : {1, 2}) {
        if (sm * bps > 220 * 1024) continue;
        int grid = sms * bps;
        float ms = timeit([&] { k_gather<2, 4><<<grid, 256, sm>>>(idx, n4, x, c.V, out); });
        CK(cudaGetLastError());
        printf("smem %u %.0f %d %.3f %.1f %.0f\n", c.V, c.skew, bps, ms, NI / ms / 1e6, NI * 4.0 / ms / 1e6);
      }
    }
    if (c.V >= (1u << 14) && c.V <= (1u << 18)) {
      for (int cs : {8, 16}) {
        uint32_t per = (c.V + cs - 1) / cs;
        size_t sm = (size_t)per * 8;
        if (sm > 200 * 1024) continue;
        CK(cudaFuncSetAttribute(k_gather_dsmem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        if (cs > 8) CK(cudaFuncSetAttribute(k_gather_dsmem<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int grid = (sms / cs) * cs;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        float ms = timeit([&] { cudaLaunchKernelEx(&cfg, k_gather_dsmem<4>, (const uint32_t*)idx, n4, (const double*)x, c.V, per, out); });
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { printf("dsmem cs=%d: %s\n", cs, cudaGetErrorString(e)); continue; }
        printf("dsmem%d %u %.0f 1 %.3f %.1f %.0f\n", cs, c.V, c.skew, ms, NI / ms / 1e6, NI * 4.0 / ms / 1e6);
      }
    }
    fflush(stdout);
  }
  return 0;
}
