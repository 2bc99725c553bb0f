// Host cost per call of the pieces of a small-batch pe_eval_f64 (GPU box):
//   g++ -O2 -std=c++17 -I include -I /usr/local/cuda/include scripts/launch_overhead.cpp \
//       -o gpurun_out/launch_overhead -L paper_1307_5655_b200/_lib -lpolyeval_b200 \
//       -L /usr/local/cuda/lib64 -lcudart -lcuda -Wl,-rpath,$PWD/paper_1307_5655_b200/_lib
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "polyeval_b200.h"

static const char* kPtx = R"(
.version 8.7
.target sm_100a
.address_size 64
.visible .entry empty(.param .u64 p) { ret; }
)";

template <class F>
static double per_call_us(int reps, F&& f) {
  auto t = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count() / reps;
}

extern "C" int lo_main() {
  const int R = 2000;
  cudaSetDevice(0);
  cudaFree(nullptr);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* x;
  double* y;
  const size_t n = 100000;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMemset(x, 0, n * 8);

  cudaLibrary_t lib;
  cudaKernel_t k;
  cudaLibraryLoadData(&lib, kPtx, nullptr, nullptr, 0, nullptr, nullptr, 0);
  cudaLibraryGetKernel(&k, lib, "empty");
  unsigned long long pv = 0;
  void* args[] = {&pv};
  cudaLaunchKernel((const void*)k, dim3(1), dim3(32), args, 0, s);
  cudaStreamSynchronize(s);
  const double lib_launch = per_call_us(R, [&] { cudaLaunchKernel((const void*)k, dim3(1), dim3(32), args, 0, s); });
  cudaStreamSynchronize(s);

  CUkernel ck = reinterpret_cast<CUkernel>(k);
  CUfunction fn;
  cuKernelGetFunction(&fn, ck);
  const double fn_launch = per_call_us(R, [&] { cuLaunchKernel(fn, 1, 1, 1, 32, 1, 1, 0, s, args, nullptr); });
  cudaStreamSynchronize(s);

  const double attrs = per_call_us(R, [&] {
    cudaPointerAttributes a;
    cudaPointerGetAttributes(&a, x);
  });
  const double setdev = per_call_us(R, [&] { cudaSetDevice(0); });

  // Hörner d1000 (C1 shape) through the C ABI, device buffers
  std::vector<uint32_t> e(1001);
  std::vector<double> c(1001);
  for (int i = 0; i <= 1000; ++i) {
    e[i] = 1000 - i;
    c[i] = 1.0 / (1 + i);
  }
  pe_scheme_desc sd{PE_SCHEME_HORNER, 0, 0};
  pe_program* p = nullptr;
  if (pe_program_create(e.data(), c.data(), 1001, 1, &sd, PE_COEFF_F64, &p) != PE_OK) {
    std::printf("create failed: %s\n", pe_last_error());
    return 1;
  }
  pe_exec ex{};
  ex.device = 0;
  ex.stream = s;
  const double* coords[1] = {x};
  pe_eval_f64(p, coords, n, y, &ex);
  cudaStreamSynchronize(s);
  const double eval = per_call_us(R, [&] { pe_eval_f64(p, coords, n, y, &ex); });
  cudaStreamSynchronize(s);
  ex.device = -1;
  const double eval_cur = per_call_us(R, [&] { pe_eval_f64(p, coords, n, y, &ex); });
  cudaStreamSynchronize(s);
  ex.stream = nullptr;  // legacy default stream (torch's default current stream)
  pe_eval_f64(p, coords, n, y, &ex);
  cudaDeviceSynchronize();
  const double eval_legacy = per_call_us(R, [&] { pe_eval_f64(p, coords, n, y, &ex); });
  cudaDeviceSynchronize();
  const double lib_launch_legacy =
      per_call_us(R, [&] { cudaLaunchKernel((const void*)k, dim3(1), dim3(32), args, 0, nullptr); });
  cudaDeviceSynchronize();
  ex.stream = s;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < 200; ++i) pe_eval_f64(p, coords, n, y, &ex);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  std::printf("{\"cudaLaunchKernel_library_kernel_us\": %.2f, \"cuLaunchKernel_function_us\": %.2f, "
              "\"cudaPointerGetAttributes_us\": %.2f, \"cudaSetDevice_us\": %.2f, "
              "\"pe_eval_f64_host_us\": %.2f, \"pe_eval_f64_current_device_host_us\": %.2f, "
              "\"pe_eval_f64_gpu_us_back_to_back\": %.2f, \"pe_eval_f64_legacy_stream_host_us\": %.2f, "
              "\"cudaLaunchKernel_legacy_stream_us\": %.2f}\n",
              lib_launch, fn_launch, attrs, setdev, eval, eval_cur, ms * 1e3 / 200, eval_legacy,
              lib_launch_legacy);
  pe_program_destroy(p);
  return 0;
}

#ifndef LO_SHARED
int main() { return lo_main(); }
#endif
