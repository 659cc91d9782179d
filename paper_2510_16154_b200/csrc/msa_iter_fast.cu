// msa_iter_fast.cu - specialised fused iteration kernel K1 (placeholder: no
// specialisation yet; the driver falls back to the generic kernel).
#include "msa_internal.h"

cudaError_t msa_launch_iter_fast(const MsaGeom&, const MsaIterConsts&, const MsaOffsetTable&, int, const float*,
                                 const float*, const float*, const float*, const float*, float*, float*, float*,
                                 cudaStream_t, int* launched) {
  *launched = 0;
  return cudaErrorNotSupported;
}
