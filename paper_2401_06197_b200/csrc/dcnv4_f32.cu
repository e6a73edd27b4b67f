// dcnv4_f32.cu -- instantiations of the DCNv4 kernels for storage type float.
#include "dcnv4_dispatch.cuh"

namespace dcnv4 {

DCNV4_DEFINE(f32, float)

}  // namespace dcnv4
