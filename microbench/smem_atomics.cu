// smem_atomics.cu -- shared-memory atomic throughput on B200 (decides the backward's
// grad_input strategy): native ATOMS.ADD.u32 (spread / same-word), the fp32 CAS-loop
// atomicAdd, and plain LDS/STS of the same pattern for reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_atomics smem_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kWords = 8192;  // 32 KB region
constexpr int kIters = 256;

template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t s[kWords];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t r = seed ^ ((blockIdx.x * 256 + threadIdx.x) * 2654435761u);
  uint32_t acc = 0;
  for (int it = 0; it < kIters; ++it) {
    r = r * 1664525u + 1013904223u;
    const int a = (r >> 8) & (kWords - 1);
    if (MODE == 0) atomicAdd(&s[a], (r >> 30) | 1u);                        // ATOMS.ADD spread
    if (MODE == 1) atomicAdd(reinterpret_cast<float*>(&s[a]), 1.0f);       // CAS loop spread
    if (MODE == 2) acc += s[a];                                            // LDS spread
    if (MODE == 3) s[a] = acc + it;                                        // STS spread
    if (MODE == 4) { float v = __uint_as_float(s[a]); s[a] = __float_as_uint(v + 1.f); }  // RMW (racy)
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[acc & (kWords - 1)] + acc;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 20));
  long long* d;
  CK(cudaMalloc(&d, 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"ATOMS.ADD.u32 spread", "atomicAdd f32 (CAS loop) spread", "LDS.32 spread",
                         "STS.32 spread", "LDS+FADD+STS (non-atomic RMW)"};
  const int blocks = sms * 8;
  void (*ks[])(uint32_t*, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  for (int m = 0; m < 5; ++m) {
    ks[m]<<<blocks, 256>>>(out, 1);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      ks[m]<<<blocks, 256>>>(out, 7 + rep);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    const double ops = (double)blocks * 256 * kIters;
    // lane-ops per SM per cycle at the nominal 1.965 GHz
    printf("{\"bench\": \"smem\", \"op\": \"%s\", \"ms\": %.4f, \"Gops\": %.1f, \"lane_ops_per_clk_per_SM\": %.2f}\n",
           names[m], best, ops / best / 1e6, ops / (best * 1e-3) / 1.965e9 / sms);
  }
  return 0;
}
