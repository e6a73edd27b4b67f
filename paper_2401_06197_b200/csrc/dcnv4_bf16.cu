// dcnv4_bf16.cu -- instantiations of the DCNv4 kernels for storage type __nv_bfloat16.
#include "dcnv4_dispatch.cuh"

namespace dcnv4 {

DCNV4_DEFINE(bf16, __nv_bfloat16)

}  // namespace dcnv4
