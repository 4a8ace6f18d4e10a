/*
 * C restatement of the reference's window spreading / gathering loops --
 * TEST INFRASTRUCTURE ONLY (the CPU baseline and `bench.py --impl reference`).
 *
 * Restates _spread_nb / _gather_nb (reference _kernels.py:48-136): full
 * width W = 2m+2 stencil per node, skip zero w0 and w0*w1, grid flattened
 * C-order with periodic wrap.  Values here are real (the reference casts
 * real data to complex, transform.py:218; the imaginary part stays 0).
 * Threads: pthreads over contiguous node ranges; the spread keeps one
 * private grid per thread and reduces them in thread order.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static inline int64_t wrapi(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

int orc_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }

typedef struct {
  const double* values;
  const int64_t* base;
  const double* w;
  int64_t lo, hi;
  int d, width;
  const int64_t* nos;
  double* grid;  /* spread: private grid; gather: out */
  int64_t size;
} Job;

static void spread_range(const Job* jb);
static void gather_range(const Job* jb);

static void* spread_main(void* a) { spread_range((const Job*)a); return NULL; }
static void* gather_main(void* a) { gather_range((const Job*)a); return NULL; }

static void run_jobs(Job* jobs, int nt, void* (*fn)(void*)) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
  for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
  fn(&jobs[0]);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
  free(th);
}

static void spread_range(const Job* jb) {
  const int d = jb->d, width = jb->width;
  const int64_t* nos = jb->nos;
  double* g = jb->grid;
  for (int64_t j = jb->lo; j < jb->hi; ++j) {
    const double v = jb->values[j];
    const double* wj = jb->w + j * d * width;
    const int64_t* bj = jb->base + j * d;
    if (d == 1) {
      for (int i0 = 0; i0 < width; ++i0)
        g[wrapi(bj[0] + i0, nos[0])] += v * wj[i0];
    } else if (d == 2) {
      for (int i0 = 0; i0 < width; ++i0) {
        double w0 = wj[i0];
        if (w0 == 0.0) continue;
        int64_t row = wrapi(bj[0] + i0, nos[0]) * nos[1];
        double vv = v * w0;
        for (int i1 = 0; i1 < width; ++i1)
          g[row + wrapi(bj[1] + i1, nos[1])] += vv * wj[width + i1];
      }
    } else {
      for (int i0 = 0; i0 < width; ++i0) {
        double w0 = wj[i0];
        if (w0 == 0.0) continue;
        int64_t p0 = wrapi(bj[0] + i0, nos[0]) * nos[1];
        for (int i1 = 0; i1 < width; ++i1) {
          double w01 = w0 * wj[width + i1];
          if (w01 == 0.0) continue;
          int64_t row = (p0 + wrapi(bj[1] + i1, nos[1])) * nos[2];
          double vv = v * w01;
          const double* w2 = wj + 2 * width;
          for (int i2 = 0; i2 < width; ++i2)
            g[row + wrapi(bj[2] + i2, nos[2])] += vv * w2[i2];
        }
      }
    }
  }
}

void orc_spread(const double* values, const int64_t* base, const double* w,
                int64_t n_nodes, int d, int width, const int64_t* nos,
                double* grid, int nthreads) {
  int64_t size = 1;
  for (int s = 0; s < d; ++s) size *= nos[s];
  if (nthreads < 1) nthreads = orc_max_threads();
  double* priv = (double*)calloc((size_t)size * nthreads, sizeof(double));
  Job* jobs = (Job*)malloc(sizeof(Job) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    Job jb = {values, base, w, n_nodes * t / nthreads, n_nodes * (t + 1) / nthreads,
              d, width, nos, priv + (size_t)t * size, size};
    jobs[t] = jb;
  }
  run_jobs(jobs, nthreads, spread_main);
  memset(grid, 0, sizeof(double) * size);
  for (int t = 0; t < nthreads; ++t) {
    const double* g = priv + (size_t)t * size;
    for (int64_t i = 0; i < size; ++i) grid[i] += g[i];
  }
  free(jobs);
  free(priv);
}

/* complex grid (interleaved re, im), real weights -> complex out */
static void gather_range(const Job* jb) {
  const int d = jb->d, width = jb->width;
  const int64_t* nos = jb->nos;
  const double* grid = jb->values;
  double* out = jb->grid;
  for (int64_t j = jb->lo; j < jb->hi; ++j) {
    const double* wj = jb->w + j * d * width;
    const int64_t* bj = jb->base + j * d;
    double ar = 0.0, ai = 0.0;
    if (d == 1) {
      for (int i0 = 0; i0 < width; ++i0) {
        int64_t k = wrapi(bj[0] + i0, nos[0]);
        ar += grid[2 * k] * wj[i0];
        ai += grid[2 * k + 1] * wj[i0];
      }
    } else if (d == 2) {
      for (int i0 = 0; i0 < width; ++i0) {
        double w0 = wj[i0];
        if (w0 == 0.0) continue;
        int64_t row = wrapi(bj[0] + i0, nos[0]) * nos[1];
        double sr = 0.0, si = 0.0;
        for (int i1 = 0; i1 < width; ++i1) {
          int64_t k = row + wrapi(bj[1] + i1, nos[1]);
          sr += grid[2 * k] * wj[width + i1];
          si += grid[2 * k + 1] * wj[width + i1];
        }
        ar += w0 * sr;
        ai += w0 * si;
      }
    } else {
      for (int i0 = 0; i0 < width; ++i0) {
        double w0 = wj[i0];
        if (w0 == 0.0) continue;
        int64_t p0 = wrapi(bj[0] + i0, nos[0]) * nos[1];
        for (int i1 = 0; i1 < width; ++i1) {
          double w01 = w0 * wj[width + i1];
          if (w01 == 0.0) continue;
          int64_t row = (p0 + wrapi(bj[1] + i1, nos[1])) * nos[2];
          const double* w2 = wj + 2 * width;
          double sr = 0.0, si = 0.0;
          for (int i2 = 0; i2 < width; ++i2) {
            int64_t k = row + wrapi(bj[2] + i2, nos[2]);
            sr += grid[2 * k] * w2[i2];
            si += grid[2 * k + 1] * w2[i2];
          }
          ar += w01 * sr;
          ai += w01 * si;
        }
      }
    }
    out[2 * j] = ar;
    out[2 * j + 1] = ai;
  }
}

/* complex grid (interleaved re, im), real weights -> complex out */
void orc_gather(const double* grid, const int64_t* base, const double* w,
                int64_t n_nodes, int d, int width, const int64_t* nos,
                double* out, int nthreads) {
  if (nthreads < 1) nthreads = orc_max_threads();
  Job* jobs = (Job*)malloc(sizeof(Job) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    Job jb = {grid, base, w, n_nodes * t / nthreads, n_nodes * (t + 1) / nthreads,
              d, width, nos, out, 0};
    jobs[t] = jb;
  }
  run_jobs(jobs, nthreads, gather_main);
  free(jobs);
}
