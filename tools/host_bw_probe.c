// Host memory bandwidth of the box (the e2e's host-side roofline): T threads stream-read
// a large fp64 array (sum), and stream-read + convert + write fp32 (the upload's own
// access pattern, into a small per-thread ring that stays in cache).
//   gcc -O3 -march=native -fopenmp -o /tmp/host_bw tools/host_bw_probe.c && /tmp/host_bw [GiB] [threads]
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? (size_t)atol(argv[1]) : 16;
  const int T = argc > 2 ? atoi(argv[2]) : omp_get_max_threads();
  const size_t n = gib * (1ull << 30) / sizeof(double);
  double* a = (double*)aligned_alloc(64, n * sizeof(double));
#pragma omp parallel for num_threads(T) schedule(static)
  for (size_t i = 0; i < n; ++i) a[i] = (double)(i & 1023) * 0.5;
  for (int rep = 0; rep < 3; ++rep) {
    double s = 0, t0 = omp_get_wtime();
#pragma omp parallel for num_threads(T) reduction(+ : s) schedule(static)
    for (size_t i = 0; i < n; ++i) s += a[i];
    const double t1 = omp_get_wtime();
    const size_t ring = 3 * (384u << 10);  // the upload's per-thread staging ring (floats)
    float* st = (float*)aligned_alloc(64, (size_t)T * ring * sizeof(float));
    const double t2 = omp_get_wtime();
#pragma omp parallel num_threads(T)
    {
      const int t = omp_get_thread_num();
      const size_t lo = n * t / T, hi = n * (t + 1) / T;
      float* my = st + (size_t)t * ring;
      for (size_t i = lo; i < hi; i += ring) {
        const size_t m = hi - i < ring ? hi - i : ring;
        for (size_t k = 0; k < m; ++k) my[k] = (float)a[i + k];
      }
    }
    const double t3 = omp_get_wtime();
    printf("threads %d  read %.1f GB/s  read+convert %.1f GB/s (of fp64 read)  [%g %g]\n", T,
           n * 8.0 / (t1 - t0) / 1e9, n * 8.0 / (t3 - t2) / 1e9, s, (double)st[5]);
    free(st);
  }
  return 0;
}
