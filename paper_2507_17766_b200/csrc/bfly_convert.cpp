// bfly_convert.cpp — host conversion of fp64 payloads to the fp32 wire ("<f4",
// butterfly.py:213, numpy's astype: IEEE round-to-nearest-even), the inner loop of the
// drop-in upload (bfly_host.cu).  Compiled by the host compiler at -O3 with function
// multi-versioning: the widest vector unit of the machine it runs on (AVX-512: 8
// doubles per conversion instruction) is picked at load time.
#include <stdint.h>

extern "C" {

__attribute__((target_clones("avx512f", "avx2", "default")))
void bfly_host_f64_to_f32(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = 0; i < n; ++i) dst[i] = (float)src[i];
}

}  // extern "C"
