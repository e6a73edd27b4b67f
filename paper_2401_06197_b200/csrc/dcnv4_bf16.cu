// dcnv4_bf16.cu -- instantiations of the DCNv4 kernels for storage type __nv_bfloat16.
#include "dcnv4_dispatch.cuh"

namespace dcnv4 {

cudaError_t launch_fwd_bf16(const Launch& lc, const Geo& g, const void* x, const void* om,
                          void* y) {
  DCNV4_TABLE(fwd_variant, __nv_bfloat16, x, om, y)
}

cudaError_t launch_bwd_bf16(const Launch& lc, const Geo& g, const void* x, const void* om,
                          const void* gy, float* gx32, void* gom) {
  DCNV4_TABLE(bwd_variant, __nv_bfloat16, x, om, gy, gx32, gom)
}

cudaError_t launch_convert_bf16(const float* src, void* dst, long long nchunk,
                              cudaStream_t stream) {
  if (nchunk <= 0) return cudaSuccess;
  long long blocks = (nchunk + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  convert_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, stream>>>(src, static_cast<__nv_bfloat16*>(dst), nchunk);
  return cudaGetLastError();
}

}  // namespace dcnv4
