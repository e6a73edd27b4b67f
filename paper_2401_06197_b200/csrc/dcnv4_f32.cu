// dcnv4_f32.cu -- instantiations of the DCNv4 kernels for storage type float.
#include "dcnv4_dispatch.cuh"

namespace dcnv4 {

cudaError_t launch_fwd_f32(const Launch& lc, const Geo& g, const void* x, const void* om,
                          void* y) {
  DCNV4_TABLE(fwd_variant, float, x, om, y)
}

cudaError_t launch_bwd_f32(const Launch& lc, const Geo& g, const void* x, const void* om,
                          const void* gy, float* gx32, void* gom) {
  DCNV4_TABLE(bwd_variant, float, x, om, gy, gx32, gom)
}

cudaError_t launch_convert_f32(const float* src, void* dst, long long nchunk,
                              cudaStream_t stream) {
  if (nchunk <= 0) return cudaSuccess;
  long long blocks = (nchunk + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  convert_kernel<float><<<(unsigned)blocks, 256, 0, stream>>>(src, static_cast<float*>(dst), nchunk);
  return cudaGetLastError();
}

}  // namespace dcnv4
