// Host copy kernels on the GPU box's host: glibc memcpy vs non-temporal
// (streaming) stores, T threads from a persistent pool, 256 MiB, best of 5.
// Destinations: pre-faulted memory (the pinned staging slots of a pageable
// write) and fresh MADV_HUGEPAGE memory (a read into a new bytes object).
// gcc -O2 -pthread -mavx2 nt_copy_probe.c -o nt_copy_probe
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

static void copy_nt(char* d, const char* s, size_t n) {
  size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head > n) head = n;
  memcpy(d, s, head);
  d += head, s += head, n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
    __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
    __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
    __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
    _mm256_stream_si256((__m256i*)(d + i), a);
    _mm256_stream_si256((__m256i*)(d + i + 32), b);
    _mm256_stream_si256((__m256i*)(d + i + 64), c);
    _mm256_stream_si256((__m256i*)(d + i + 96), e);
  }
  memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

typedef struct {
  char* d;
  const char* s;
  size_t n, part;
  int nt;
  int T;
} Job;

static Job g_job;
static pthread_barrier_t g_start, g_end;
static int g_quit;

static void* worker(void* p) {
  int id = (int)(intptr_t)p;
  for (;;) {
    pthread_barrier_wait(&g_start);
    if (g_quit) return NULL;
    // tasks of `part` bytes dealt round robin (like the copy pool's tasks)
    for (size_t off = (size_t)id * g_job.part; off < g_job.n; off += (size_t)g_job.T * g_job.part) {
      size_t len = g_job.n - off < g_job.part ? g_job.n - off : g_job.part;
      if (g_job.nt)
        copy_nt(g_job.d + off, g_job.s + off, len);
      else
        memcpy(g_job.d + off, g_job.s + off, len);
    }
    pthread_barrier_wait(&g_end);
  }
}

static double run(char* d, const char* s, size_t n, int nt, size_t part, int T) {
  g_job = (Job){d, s, n, part, nt, T};
  double t0 = now();
  pthread_barrier_wait(&g_start);
  pthread_barrier_wait(&g_end);
  return n / (now() - t0) / 1e9;
}

int main(void) {
  const size_t n = 256u << 20;
  char* src = aligned_alloc(4096, n);
  memset(src, 7, n);
  char* warm = aligned_alloc(4096, n);
  memset(warm, 1, n);
  int Ts[] = {4, 8, 12, 15};
  for (int k = 0; k < 4; ++k) {
    int T = Ts[k];
    pthread_t th[64];
    pthread_barrier_init(&g_start, NULL, T + 1);
    pthread_barrier_init(&g_end, NULL, T + 1);
    g_quit = 0;
    for (int i = 0; i < T; ++i) pthread_create(&th[i], NULL, worker, (void*)(intptr_t)i);
    for (int nt = 0; nt < 2; ++nt) {
      double best_w = 0, best_f = 0;
      for (int r = 0; r < 5; ++r) {
        double w = run(warm, src, n, nt, 1u << 20, T);
        if (w > best_w) best_w = w;
        char* f = mmap(NULL, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        madvise(f, n, MADV_HUGEPAGE);
        double x = run(f + 48, src, n - 64, nt, 2u << 20, T);
        if (x > best_f) best_f = x;
        munmap(f, n);
      }
      printf("threads %2d %-8s prefaulted dst %6.1f GB/s   fresh huge-page dst %6.1f GB/s\n", T,
             nt ? "NT" : "memcpy", best_w, best_f);
      fflush(stdout);
    }
    g_quit = 1;
    pthread_barrier_wait(&g_start);
    for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
    pthread_barrier_destroy(&g_start);
    pthread_barrier_destroy(&g_end);
  }
  return 0;
}
