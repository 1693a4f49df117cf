/* Host (C) twin of synth/__init__.py: the seeded counter-based input generator.
 * Holds no arithmetic of the OmniMoE method; it turns (seed, tensor id, index)
 * into v * 2^-e exactly like the numpy and CUDA twins and decodes the stored
 * value (bf16 by integer round-to-nearest-even, or fp32) to double.  It exists
 * only for speed: the parity tests regenerate hundreds of thousands of expert
 * rows on the host.  tests/test_synth.py::test_c_twin_matches_numpy
 * checks bit identity with the numpy twin.  Built into synth/libsynth_host.so
 * with gcc (no CUDA). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double value(uint64_t seed, uint64_t tid, uint64_t index, int e, int mode, int bf16) {
  uint64_t key = ((seed & 0xFF) << 56) ^ ((tid & 0xFF) << 48) ^ index;
  uint64_t h = splitmix64(key);
  int64_t v;
  if (mode == 1) {
    v = (int64_t)(h % 9ull) - 4;
  } else {
    uint64_t s = (h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + (h >> 48);
    v = (int64_t)s - 131070;
  }
  float f = ldexpf((float)v, -e); /* exact: |v| < 2^18 */
  if (bf16) {
    uint32_t b;
    memcpy(&b, &f, 4);
    b = ((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16) << 16;
    memcpy(&f, &b, 4);
  }
  return (double)f;
}

typedef struct {
  uint64_t seed, tid;
  const int64_t* rows;
  int64_t r0, r1, ncols;
  int e, mode, bf16;
  double* out;
} job_t;

static void* run(void* p) {
  job_t* j = (job_t*)p;
  for (int64_t r = j->r0; r < j->r1; ++r) {
    uint64_t base = (uint64_t)j->rows[r] * (uint64_t)j->ncols;
    double* o = j->out + r * j->ncols;
    for (int64_t c = 0; c < j->ncols; ++c) o[c] = value(j->seed, j->tid, base + (uint64_t)c, j->e, j->mode, j->bf16);
  }
  return 0;
}

/* out[r][c] = decoded element (rows[r], c) of the [*, ncols] tensor (seed, tid). */
void synth_rows_f64(uint64_t seed, uint64_t tid, const int64_t* rows, int64_t nrows, int64_t ncols, int e, int mode,
                    int bf16, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nrows < 64 * nthreads) nthreads = (int)(nrows / 64) + 1;
  pthread_t th[256];
  job_t jobs[256];
  int64_t per = (nrows + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t a = t * per, b = a + per < nrows ? a + per : nrows;
    jobs[t] = (job_t){seed, tid, rows, a < nrows ? a : nrows, b, ncols, e, mode, bf16, out};
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, run, &jobs[t]);
  run(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
}
