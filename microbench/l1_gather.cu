// l1_gather.cu -- B200 microbenchmarks that decide the DCNv4 kernel design
// (SURVEY.md 8(d).2 "verify first"):
//   1. L1-hit 16-byte gather bandwidth (B/clk/SM) under the lane -> address patterns the
//      forward kernel can produce (random 16-B vectors, 32/64/128-B segments per lane
//      group, bank-quad staggered or not);
//   2. global vector-reduction (red.global.add.v4.f32) payload throughput for scattered
//      16-B targets, L2-resident and HBM-sized;
//   3. SM clock calibration.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1_gather l1_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int kBufBytes = 32 * 1024;  // L1-resident gather source
constexpr int kIters = 512;
constexpr int kUnroll = 8;

// pattern ids
enum { P_COAL = 0, P_RAND16, P_RAND16_STAG, P_SEG32, P_SEG64, P_SEG64_STAG, P_SEG128, P_SEG32_STAG, NPAT };
static const char* kNames[NPAT] = {"coalesced 512B", "random 16B", "random 16B, quad-staggered",
                                   "32B segments (2 lanes)", "64B segments (4 lanes)",
                                   "64B segments, bit6-staggered", "128B lines (8 lanes)",
                                   "32B segments, quad-staggered"};

template <int PAT>
__device__ __forceinline__ uint32_t addr_of(uint32_t r, int lane) {
  const uint32_t lines = kBufBytes / 128;
  switch (PAT) {
    case P_COAL: return ((r >> 8) % (kBufBytes / 512)) * 512 + lane * 16;
    case P_RAND16: return (r >> 4) % (kBufBytes / 16) * 16;
    case P_RAND16_STAG: return ((r >> 8) % lines) * 128 + (lane & 7) * 16;
    case P_SEG32: return ((r >> 8) % (kBufBytes / 32)) * 32 + (lane & 1) * 16;
    case P_SEG64: return ((r >> 8) % (kBufBytes / 64)) * 64 + (lane & 3) * 16;
    case P_SEG64_STAG: return ((r >> 8) % lines) * 128 + ((lane >> 2) & 1) * 64 + (lane & 3) * 16;
    case P_SEG128: return ((r >> 8) % lines) * 128 + (lane & 7) * 16;
    case P_SEG32_STAG: return ((r >> 8) % lines) * 128 + ((lane >> 1) & 3) * 32 + (lane & 1) * 16;
  }
  return 0;
}

template <int PAT>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ buf, uint32_t* out,
                                              uint32_t seed) {
  const int lane = threadIdx.x & 31;
  // lanes that share a segment must share the random draw: derive r from the segment id
  int share = 1;
  if (PAT == P_SEG32 || PAT == P_SEG32_STAG) share = 2;
  if (PAT == P_SEG64 || PAT == P_SEG64_STAG) share = 4;
  if (PAT == P_SEG128 || PAT == P_RAND16_STAG) share = (PAT == P_SEG128) ? 8 : 1;
  if (PAT == P_COAL) share = 32;
  uint32_t r = seed ^ ((blockIdx.x * 256 + (threadIdx.x - lane) + lane / share) * 2654435761u);
  uint32_t acc = 0;
  const char* base = reinterpret_cast<const char*>(buf);
  for (int it = 0; it < kIters; it += kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      r = r * 1664525u + 1013904223u;
      v[u] = __ldg(reinterpret_cast<const uint4*>(base + addr_of<PAT>(r, lane)));
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Scattered vector reductions: each lane issues red.global.add.v4.f32 to a random 16-B
// slot of a `span`-byte buffer; `seg` lanes share a contiguous (seg*16)-byte segment.
template <int SEG>
__global__ void __launch_bounds__(256) reds(float* buf, uint64_t span16, uint32_t seed, int iters) {
  const int lane = threadIdx.x & 31;
  uint32_t r = seed ^ ((blockIdx.x * 256 + (threadIdx.x - lane) + lane / SEG) * 2654435761u);
  for (int it = 0; it < iters; ++it) {
    r = r * 1664525u + 1013904223u;
    uint64_t slot = ((uint64_t)r * 7919u) % (span16 / SEG) * SEG + (lane % SEG);
    float* p = buf + slot * 4;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f),
                 "f"(1.f), "f"(1.f) : "memory");
  }
}

__global__ void spin(long long cycles, long long* out) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  long long* dcyc;
  CK(cudaMalloc(&dcyc, 8));
  const long long spin_cyc = 200000000LL;
  float spin_ms = time_ms([&] { spin<<<sms, 32>>>(spin_cyc, dcyc); }, 2);
  const double ghz = spin_cyc / (spin_ms * 1e6);
  printf("{\"sms\": %d, \"sm_clock_ghz_measured\": %.4f}\n", sms, ghz);

  uint4* buf;
  uint32_t* out;
  CK(cudaMalloc(&buf, kBufBytes));
  CK(cudaMemset(buf, 1, kBufBytes));
  CK(cudaMalloc(&out, 4));
  const int blocks = sms * 8;
  const double bytes = (double)blocks * 256 * kIters * 16;
  auto run = [&](auto kern, int pat) {
    float ms = time_ms([&] { kern<<<blocks, 256>>>(buf, out, 1234u); });
    double bpc = bytes / (ms * 1e-3) / (ghz * 1e9) / sms;
    printf("{\"bench\": \"l1_gather\", \"pattern\": \"%s\", \"ms\": %.4f, \"TB_s\": %.2f, \"B_per_clk_per_SM\": %.1f}\n",
           kNames[pat], ms, bytes / (ms * 1e-3) / 1e12, bpc);
  };
  run(gather<P_COAL>, P_COAL);
  run(gather<P_RAND16>, P_RAND16);
  run(gather<P_RAND16_STAG>, P_RAND16_STAG);
  run(gather<P_SEG32>, P_SEG32);
  run(gather<P_SEG32_STAG>, P_SEG32_STAG);
  run(gather<P_SEG64>, P_SEG64);
  run(gather<P_SEG64_STAG>, P_SEG64_STAG);
  run(gather<P_SEG128>, P_SEG128);

  // reductions
  const int iters = 256;
  for (uint64_t span : {(uint64_t)64 << 20, (uint64_t)2 << 30}) {
    float* rb;
    CK(cudaMalloc(&rb, span));
    CK(cudaMemset(rb, 0, span));
    const double payload = (double)blocks * 256 * iters * 16;
    float ms1 = time_ms([&] { reds<1><<<blocks, 256>>>(rb, span / 16, 77u, iters); }, 3);
    float ms4 = time_ms([&] { reds<4><<<blocks, 256>>>(rb, span / 16, 77u, iters); }, 3);
    float ms8 = time_ms([&] { reds<8><<<blocks, 256>>>(rb, span / 16, 77u, iters); }, 3);
    printf("{\"bench\": \"red_v4_f32\", \"span_MB\": %llu, \"random16_TB_s\": %.3f, \"seg64_TB_s\": %.3f, \"seg128_TB_s\": %.3f, \"Gred_s_random\": %.1f}\n",
           (unsigned long long)(span >> 20), payload / (ms1 * 1e-3) / 1e12, payload / (ms4 * 1e-3) / 1e12,
           payload / (ms8 * 1e-3) / 1e12, payload / 16 / (ms1 * 1e-3) / 1e9);
    CK(cudaFree(rb));
  }
  return 0;
}
