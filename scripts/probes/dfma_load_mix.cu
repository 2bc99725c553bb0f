// Probe: FP64 FMA-pipe throughput of a DFMA stream (2 or 8 independent chains
// per thread) with one other instruction per 2, 4 or 8 DFMAs — a uniform
// constant load (LDCU.64), a shared-memory load (LDS.128), a per-thread
// constant load (LDC.64), a global load through L1 (LDG.128) or an integer
// add — at 2, 4 and 8 warps per SM sub-partition. Shows which instructions
// take FP64 issue cycles: the walk kernels deliver their coefficients with
// such loads (C4: one LDCU.128 per 3.5 and one LDS.128 per 9 FP64
// instructions at 4 warps per sub-partition; C2 an eighth of that; C3 none).
// Prints one JSON line per variant (profiles/r2_probe_dfma_load_mix.jsonl).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_load_mix.bin dfma_load_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ __align__(16) double carr[8192];

// USES = pairs of DFMAs per 16-byte load (1 -> 0.5 loads per DFMA, 2 -> 0.25,
// 4 -> 0.125, 0 -> loop-invariant coefficients: no loads in the loop).
// KIND = the instruction that delivers the pair: 0 uniform constant load
// (LDCU.128), 1 shared memory (LDS.128), 2 per-thread constant load
// (LDC.128), 3 global memory through L1 (LDG.128), 4 no load but one
// integer add in its place (what else can issue beside a DFMA?)
template <int KIND, int USES, int CHAINS>
__global__ void __launch_bounds__(1024) mix(const double* x, double* out, int iters, const double2* g) {
  __shared__ double2 sc[2048];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = threadIdx.x; k < 2048; k += blockDim.x) sc[k] = g[k];
  __syncthreads();
  double v = x[i];
  const unsigned zoff = v == 12345.0 ? 16 : 0;  // zero at run time, per-thread to the compiler
  unsigned acc = 0;
  double a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) a[c] = v + c;
  for (int it = 0; it < iters; ++it) {
    // the base moves with the loop counter so the loads stay in the loop
    const int base = (it & 31) * 64;
    const double2* cu = reinterpret_cast<const double2*>(carr) + base;
    const double2* ct = reinterpret_cast<const double2*>(carr) + base + zoff;
    double2 w = make_double2(0.5, 0.25);
#pragma unroll
    for (int j = 0; j < 128; j += 2) {
      if (USES == 0) {
        w = reinterpret_cast<const double2*>(carr)[(j / 2) % 8];
      } else if ((j / 2) % (USES ? USES : 1) == 0) {
        const int k = j / 2 / (USES ? USES : 1);
        if (KIND == 0) w = cu[k];
        else if (KIND == 1) w = sc[base + k];
        else if (KIND == 2) w = ct[k];
        else if (KIND == 3) w = __ldg(g + base + k);
        else asm volatile("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(zoff));
      }
      a[j % CHAINS] = fma(a[j % CHAINS], v, w.x);
      a[(j + 1) % CHAINS] = fma(a[(j + 1) % CHAINS], v, w.y);
    }
  }
  double s = acc;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  out[i] = s;
}

template <int KIND, int USES, int CHAINS>
void run(const char* name, int block, const double* x, double* out, int sms, const double2* g) {
  const int iters = 2000;
  // SASS: the constant-bank kinds become two 8-byte loads per 16 bytes (UR-indexed)
  static const char* kinds[] = {"2xLDCU.64", "LDS.128", "2xLDC.64", "LDG.128", "IADD"};
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
    const int grid = sms * ctas_per_sm;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(s);
      mix<KIND, USES, CHAINS><<<grid, block>>>(x, out, iters, g);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      if (r >= 2 && ms < best) best = ms;
    }
    const double fma = double(grid) * block * iters * 128.0;
    std::printf("{\"variant\": \"%s\", \"load\": \"%s\", \"chains\": %d, \"block\": %d, \"ctas_per_sm\": %d, "
                "\"warps_per_smsp\": %d, \"ms\": %.4f, \"tfma_per_s\": %.3f}\n",
                name, USES ? kinds[KIND] : "-", CHAINS, block, ctas_per_sm, block / 32 * ctas_per_sm / 4,
                best, fma / (best * 1e-3) / 1e12);
    std::fflush(stdout);
  }
}

template <int KIND>
void kind(int block, const double* x, double* out, int sms, const double2* g) {
  run<KIND, 4, 8>("8_dfma_per_16B", block, x, out, sms, g);
  run<KIND, 2, 8>("4_dfma_per_16B", block, x, out, sms, g);
  run<KIND, 1, 8>("2_dfma_per_16B", block, x, out, sms, g);
  run<KIND, 1, 2>("2_dfma_per_16B", block, x, out, sms, g);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  static double h[8192];
  for (int i = 0; i < 8192; ++i) h[i] = 1.0 / (i + 3);
  cudaMemcpyToSymbol(carr, h, sizeof h);
  double *x, *out;
  double2* g;
  cudaMalloc(&x, sizeof(double) * sms * 2 * 1024);
  cudaMalloc(&out, sizeof(double) * sms * 2 * 1024);
  cudaMalloc(&g, sizeof h);
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, sizeof(double) * sms * 2 * 1024);
  for (int block : {256, 512}) {
    run<0, 0, 8>("no_loads", block, x, out, sms, g);
    run<0, 0, 2>("no_loads", block, x, out, sms, g);
    kind<0>(block, x, out, sms, g);
    kind<1>(block, x, out, sms, g);
    kind<2>(block, x, out, sms, g);
    kind<3>(block, x, out, sms, g);
    kind<4>(block, x, out, sms, g);
  }
  return 0;
}
