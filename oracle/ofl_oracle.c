/*
 * ofl_oracle.c — CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (its cpu_baseline leg and --impl reference) may load this; the
 * product path (paper_1810_11482_b200/) never does.
 *
 * Each function restates one kernel of the reference package (`offloadrt`,
 * /root/reference/pkg/src/offloadrt) as the reference's sequential executor
 * evaluates it (kernel/codegen.py:107-128: every work item in gtid order,
 * every binary operation a separate IEEE double operation, u32 arithmetic
 * mod 2^32).  Built with -ffp-contract=off so no FMA is ever formed.  Loops
 * over independent items may be split across `threads` pthreads (<= 0: all
 * cores); the results do not depend on the split.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---- minimal static-partition parallel-for on pthreads ------------------ */
typedef void (*range_fn)(int64_t lo, int64_t hi, void* ctx);

struct job {
  range_fn fn;
  void* ctx;
  int64_t lo, hi;
};

static void* run_job(void* p) {
  struct job* j = (struct job*)p;
  j->fn(j->lo, j->hi, j->ctx);
  return NULL;
}

int oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* split [0, n) into `threads` contiguous chunks (threads <= 0: all cores) */
static void parallel_for(int64_t n, int threads, range_fn fn, void* ctx) {
  if (threads <= 0) threads = oracle_max_threads();
  if (threads > 256) threads = 256;
  if (threads > n) threads = (int)n;
  if (threads <= 1) {
    fn(0, n, ctx);
    return;
  }
  pthread_t tid[256];
  struct job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    if (t) pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  }
  run_job(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* STREAM (no reference kernel; semantics of paper_1810_11482_b200/kernels/
 * stream.k run through the reference executor): op 0 copy a=b, 1 scale a=s*b,
 * 2 add a=b+c, 3 triad a=b+s*c, for i < n. */
struct stream_ctx {
  int op;
  double* a;
  const double *b, *c;
  double s;
};

static void stream_range(int64_t lo, int64_t hi, void* p) {
  struct stream_ctx* k = (struct stream_ctx*)p;
  double* a = k->a;
  const double *b = k->b, *c = k->c;
  const double s = k->s;
  for (int64_t i = lo; i < hi; ++i) {
    double v;
    switch (k->op) {
      case 0: v = b[i]; break;
      case 1: v = s * b[i]; break;
      case 2: v = b[i] + c[i]; break;
      default: {
        double t = s * c[i];
        v = b[i] + t;
      } break;
    }
    a[i] = v;
  }
}

void oracle_stream(int op, double* a, const double* b, const double* c, double s, uint64_t n,
                   int threads) {
  struct stream_ctx k = {op, a, b, c ? c : b, s};
  parallel_for((int64_t)n, threads, stream_range, &k);
}

/* stencil.k (bench/kernels/stencil.k:2-10) for items gtid < min(n, items);
 * oracle harness.py:123-126, tests/oracles.py:13-20. */
struct stencil_ctx {
  const double* x;
  double* y;
  uint64_t n;
};

static void stencil_range(int64_t lo, int64_t hi, void* p) {
  struct stencil_ctx* k = (struct stencil_ctx*)p;
  const double* x = k->x;
  double* y = k->y;
  for (int64_t i = lo; i < hi; ++i) {
    if (i == 0 || (uint64_t)i == k->n - 1) {
      y[i] = x[i];
    } else {
      double l = 0.5 * x[i - 1];
      double t = l + x[i];
      double r = 0.5 * x[i + 1];
      y[i] = t + r;
    }
  }
}

void oracle_stencil(const double* x, double* y, uint64_t n, uint64_t items, int threads) {
  uint64_t m = items < n ? items : n;
  struct stencil_ctx k = {x, y, n};
  parallel_for((int64_t)m, threads, stencil_range, &k);
}

/* `steps` applications of stencil.k ping-ponging x <-> y (BASELINE config 2);
 * result in x if steps is even, else y. */
void oracle_heat(double* x, double* y, uint64_t n, uint64_t steps, int threads) {
  double* src = x;
  double* dst = y;
  for (uint64_t s = 0; s < steps; ++s) {
    oracle_stencil(src, dst, n, n, threads);
    double* t = src;
    src = dst;
    dst = t;
  }
}

/* stencil2d.k (paper_1810_11482_b200/kernels/stencil2d.k; the reference
 * language, executed as the reference executor does, kernel/codegen.py:
 * 107-128): items gtid < min((w*h) mod 2^32, items), u32 row/col, boundary
 * ring held, interior 0.25 * (((N + W) + E) + S) left to right. */
struct stencil2d_ctx {
  const double* x;
  double* y;
  uint32_t w, h;
};

static void stencil2d_range(int64_t lo, int64_t hi, void* p) {
  struct stencil2d_ctx* k = (struct stencil2d_ctx*)p;
  const double* x = k->x;
  double* y = k->y;
  const uint32_t w = k->w, h = k->h;
  for (int64_t i = lo; i < hi; ++i) {
    const uint32_t g = (uint32_t)i;
    const uint32_t row = g / w;
    const uint32_t col = g - row * w;
    if (row == 0 || row == h - 1u || col == 0 || col == w - 1u) {
      y[g] = x[g];
    } else {
      double t = x[g - w] + x[g - 1];
      t = t + x[g + 1];
      t = t + x[g + w];
      y[g] = 0.25 * t;
    }
  }
}

void oracle_stencil2d(const double* x, double* y, uint32_t w, uint32_t h, uint64_t items,
                      int threads) {
  const uint64_t cells = (uint64_t)(uint32_t)(w * h);
  const uint64_t m = items < cells ? items : cells;
  struct stencil2d_ctx k = {x, y, w, h};
  parallel_for((int64_t)m, threads, stencil2d_range, &k);
}

/* mandelbrot.k (bench/kernels/mandelbrot.k:6-29); validator harness.py:133-158,
 * tests/oracles.py:30-55.  Pixels gtid < min((w*h) mod 2^32, items), rows
 * py = row_first + k*row_step only. */
static uint32_t escape(double cre, double cim, double esc, uint32_t max_iter) {
  double zr = 0.0, zi = 0.0;
  uint32_t count = 0;
  for (uint32_t i = 0; i < max_iter; ++i) {
    double zr2 = zr * zr;
    double zi2 = zi * zi;
    double mag = zr2 + zi2;
    if (mag > esc) break;
    double d = zr2 - zi2;
    double t = d + cre;
    double tz = 2.0 * zr;
    double p = tz * zi;
    zi = p + cim;
    zr = t;
    count = count + 1;
  }
  return count;
}

struct mandel_ctx {
  uint32_t* out;
  uint32_t width, height, max_iter, row_first, row_step, nthreads;
  double re0, re1, im0, im1, esc;
  uint64_t limit;
};

/* rows are dealt cyclically to the chunks (chunk t takes rows t, t+T, ...)
 * so the expensive bounded region is shared evenly */
static void mandel_range(int64_t lo, int64_t hi, void* p) {
  struct mandel_ctx* k = (struct mandel_ctx*)p;
  const double dre = k->re1 - k->re0, dim = k->im1 - k->im0;
  const uint64_t nrows =
      k->row_first < k->height ? (k->height - k->row_first + k->row_step - 1) / k->row_step : 0;
  for (int64_t t = lo; t < hi; ++t) {
    for (uint64_t r = (uint64_t)t; r < nrows; r += k->nthreads) {
      uint64_t py = k->row_first + r * k->row_step;
      for (uint32_t px = 0; px < k->width; ++px) {
        uint64_t g = py * k->width + px;
        if (g >= k->limit) break;
        double fx = ((double)px + 0.5) * dre;
        double cre = k->re0 + fx / (double)k->width;
        double fy = ((double)py + 0.5) * dim;
        double cim = k->im0 + fy / (double)k->height;
        k->out[g] = escape(cre, cim, k->esc, k->max_iter);
      }
    }
  }
}

void oracle_mandelbrot(uint32_t* out, uint32_t width, uint32_t height, double re0, double re1,
                       double im0, double im1, double esc, uint32_t max_iter, uint64_t items,
                       uint32_t row_first, uint32_t row_step, int threads) {
  uint64_t total = (uint64_t)(uint32_t)(width * height);
  uint64_t limit = items < total ? items : total;
  if (!limit || !width || row_step == 0) return;
  if (threads <= 0) threads = oracle_max_threads();
  struct mandel_ctx k = {out, width, height, max_iter, row_first, row_step, (uint32_t)threads,
                         re0, re1, im0, im1, esc, limit};
  parallel_for(threads, threads, mandel_range, &k);
}

/* sum.k (bench/kernels/sum.k:3-11), oracle harness.py:129-130: mod 2^32. */
struct sum_ctx {
  const uint32_t* in;
  uint64_t n;
  uint32_t part[256];
  int chunks;
};

static void sum_range(int64_t lo, int64_t hi, void* p) {
  struct sum_ctx* k = (struct sum_ctx*)p;
  for (int64_t c = lo; c < hi; ++c) {
    uint64_t a = k->n * (uint64_t)c / (uint64_t)k->chunks;
    uint64_t b = k->n * (uint64_t)(c + 1) / (uint64_t)k->chunks;
    uint32_t acc = 0;
    for (uint64_t i = a; i < b; ++i) acc += k->in[i];
    k->part[c] = acc;
  }
}

uint32_t oracle_sum_u32(const uint32_t* in, uint64_t n, int threads) {
  if (threads <= 0) threads = oracle_max_threads();
  if (threads > 256) threads = 256;
  struct sum_ctx k;
  k.in = in;
  k.n = n;
  k.chunks = threads;
  parallel_for(threads, threads, sum_range, &k);
  uint32_t acc = 0;  /* addition mod 2^32 is associative: same as in order */
  for (int c = 0; c < threads; ++c) acc += k.part[c];
  return acc;
}

/* fp32 dot product, fp64 accumulation (BASELINE config 4; no reference
 * kernel exists — parity is by tolerance).  Fixed chunking of 2^16 items
 * summed in order, so the result does not depend on the thread count. */
struct dot_ctx {
  const float *a, *b;
  uint64_t n;
  double* partial;
};

#define DOT_CHUNK (1u << 16)

static void dot_range(int64_t lo, int64_t hi, void* p) {
  struct dot_ctx* k = (struct dot_ctx*)p;
  for (int64_t c = lo; c < hi; ++c) {
    uint64_t a = (uint64_t)c * DOT_CHUNK;
    uint64_t b = a + DOT_CHUNK < k->n ? a + DOT_CHUNK : k->n;
    double s = 0.0;
    for (uint64_t i = a; i < b; ++i) s += (double)k->a[i] * (double)k->b[i];
    k->partial[c] = s;
  }
}

double oracle_dot_f32(const float* a, const float* b, uint64_t n, int threads) {
  int64_t nchunks = (int64_t)((n + DOT_CHUNK - 1) / DOT_CHUNK);
  double* partial = (double*)calloc((size_t)(nchunks ? nchunks : 1), sizeof(double));
  struct dot_ctx k = {a, b, n, partial};
  parallel_for(nchunks, threads, dot_range, &k);
  double total = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) total += partial[c];
  free(partial);
  return total;
}

/* The reference's own order for the same dot product: the dot_seq kernel of
 * tests/golden/make_golden.py (reference language, pattern
 * bench/kernels/sum.k:3-11) run by the reference executor — work item 0
 * adds the exact fp64 products of the fp32 values in index order.
 * Bit-identical to golden_long.json["dot"]. */
double oracle_dot_f32_seq(const float* a, const float* b, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc = acc + (double)a[i] * (double)b[i];
  return acc;
}

/* partition.k (bench/kernels/partition.k:3-8). */
struct part_ctx {
  double* out;
  uint32_t offset;
};

static void part_range(int64_t lo, int64_t hi, void* p) {
  struct part_ctx* k = (struct part_ctx*)p;
  for (int64_t i = lo; i < hi; ++i) {
    double v = (double)(uint32_t)(k->offset + (uint32_t)i);
    double s = sin(v), c = cos(v);
    double ss = s * s, cc = c * c;
    k->out[i] = sqrt(ss + cc);
  }
}

void oracle_partition(double* out, uint32_t offset, uint64_t count, int threads) {
  struct part_ctx k = {out, offset};
  parallel_for((int64_t)count, threads, part_range, &k);
}
