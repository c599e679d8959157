// xterm_f32.cu -- float-trace variant (a6): placeholder until the bf16 hi/lo
// tcgen05 kernel lands.
#include "xterm_f32.h"

namespace cpa {

cudaError_t xterm_f32_accumulate(XtermF32Scratch &, const float *, int64_t, const uint8_t *, int64_t, int32_t,
                                 const uint8_t *, double *, int, cudaStream_t, int *)
{
    return cudaErrorNotSupported;
}

void xterm_f32_free(XtermF32Scratch &s)
{
    cudaFree(s.hi);
    cudaFree(s.lo);
    s.hi = s.lo = nullptr;
    s.cap_bytes = 0;
}

}  // namespace cpa
