// dcnv4_f16.cu -- instantiations of the DCNv4 kernels for storage type __half.
#include "dcnv4_dispatch.cuh"

namespace dcnv4 {

DCNV4_DEFINE(f16, __half)

}  // namespace dcnv4
