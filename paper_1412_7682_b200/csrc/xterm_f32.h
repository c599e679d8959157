// xterm_f32.h -- float-trace variant of the Phase-2 sums (a6) [P:201-217].
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace cpa {

struct XtermF32Scratch {
    void *hi = nullptr;      // bf16 high parts of W, N x ldh
    void *lo = nullptr;      // bf16 residuals W - hi
    int64_t cap_bytes = 0;   // bytes per buffer
};

// Adds sum_hw, sum_w, sum_w2 (fp64, packed accumulator layout) for n float traces.
cudaError_t xterm_f32_accumulate(XtermF32Scratch &s, const float *d_w, int64_t ld, const uint8_t *d_texts,
                                 int64_t n, int32_t M, const uint8_t *d_vtab, double *d_accum, int num_sms,
                                 cudaStream_t stream, int *launches);
void xterm_f32_free(XtermF32Scratch &s);

}  // namespace cpa
