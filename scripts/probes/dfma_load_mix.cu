// Probe: FP64 FMA-pipe throughput of a DFMA stream interleaved with uniform
// constant loads (LDCU.128, two coefficients each), as a function of loads
// per DFMA and warps per SM sub-partition. The sectioned C4 walk issues
// ~0.40 loads per FP64 instruction at 4 warps per sub-partition; C2 0.125;
// C3 none. Prints one JSON line per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_load_mix dfma_load_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double carr[8192];

// USES = pairs of DFMAs per 16-byte load (1 -> 0.5 loads per DFMA, 2 -> 0.25,
// 4 -> 0.125, 0 -> loop-invariant coefficients: no loads in the loop)
template <int USES, int CHAINS, int J>
__device__ __forceinline__ void step(double (&a)[CHAINS], double v, double& lx, double& ly) {
  if constexpr (USES == 0) {
    lx = carr[(J / 2) % 8 * 2];
    ly = carr[(J / 2) % 8 * 2 + 1];
  } else if constexpr ((J / 2) % USES == 0) {
    // volatile: stays in the loop at an immediate address (LDCU.128), as
    // in the generated walk kernels
    asm volatile("ld.const.v2.f64 {%0, %1}, [carr+%2];" : "=d"(lx), "=d"(ly) : "n"(J * 8));
  }
  a[J % CHAINS] = fma(a[J % CHAINS], v, lx);
  a[(J + 1) % CHAINS] = fma(a[(J + 1) % CHAINS], v, ly);
  if constexpr (J + 2 < 128) step<USES, CHAINS, J + 2>(a, v, lx, ly);
}

template <int USES, int CHAINS>
__global__ void __launch_bounds__(1024) mix(const double* x, double* out, int iters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = x[i];
  double a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) a[c] = v + c;
  for (int it = 0; it < iters; ++it) {
    double lx = 0, ly = 0;
    step<USES, CHAINS, 0>(a, v, lx, ly);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  out[i] = s;
}

template <int USES, int CHAINS>
void run(const char* name, int block, const double* x, double* out, int sms) {
  const int iters = 2000;
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
    const int grid = sms * ctas_per_sm;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(s);
      mix<USES, CHAINS><<<grid, block>>>(x, out, iters);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      if (r >= 2 && ms < best) best = ms;
    }
    const double fma = double(grid) * block * iters * 128.0;
    std::printf("{\"variant\": \"%s\", \"chains\": %d, \"block\": %d, \"ctas_per_sm\": %d, "
                "\"warps_per_smsp\": %d, \"ms\": %.4f, \"tfma_per_s\": %.3f}\n",
                name, CHAINS, block, ctas_per_sm, block / 32 * ctas_per_sm / 4, best,
                fma / (best * 1e-3) / 1e12);
  }
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double h[8192];
  for (int i = 0; i < 8192; ++i) h[i] = 1.0 / (i + 3);
  cudaMemcpyToSymbol(carr, h, sizeof h);
  double *x, *out;
  cudaMalloc(&x, sizeof(double) * sms * 2 * 1024);
  cudaMalloc(&out, sizeof(double) * sms * 2 * 1024);
  cudaMemset(x, 0, sizeof(double) * sms * 2 * 1024);
  for (int block : {256, 512}) {
    run<0, 8>("no_loads", block, x, out, sms);
    run<4, 8>("0.125_loads_per_dfma", block, x, out, sms);
    run<2, 8>("0.25_loads_per_dfma", block, x, out, sms);
    run<1, 8>("0.5_loads_per_dfma", block, x, out, sms);
    run<1, 2>("0.5_loads_per_dfma", block, x, out, sms);
    run<2, 2>("0.25_loads_per_dfma", block, x, out, sms);
    run<0, 2>("no_loads", block, x, out, sms);
  }
  return 0;
}
