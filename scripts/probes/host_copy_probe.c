// Host memcpy bandwidth on the GPU box's host: T threads copying 256 MiB
// into (a) fresh malloc memory (first touch), (b) fresh memory advised
// MADV_HUGEPAGE, (c) pre-faulted memory.  gcc -O2 -pthread host_copy_probe.c
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>

typedef struct { char* d; const char* s; size_t n; } Job;
static void* run(void* p) { Job* j = (Job*)p; memcpy(j->d, j->s, j->n); return NULL; }
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + t.tv_nsec * 1e-9; }

static double copy_par(char* d, const char* s, size_t n, int T) {
  pthread_t th[64]; Job j[64];
  size_t per = (n + T - 1) / T;
  double t0 = now();
  for (int i = 0; i < T; ++i) {
    size_t lo = i * per; size_t len = lo + per <= n ? per : n - lo;
    j[i] = (Job){d + lo, s + lo, len};
    pthread_create(&th[i], NULL, run, &j[i]);
  }
  for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
  return n / (now() - t0) / 1e9;
}

int main(void) {
  size_t n = 256u << 20;
  char* src = aligned_alloc(4096, n);
  memset(src, 7, n);
  int Ts[] = {1, 2, 4, 8, 12, 16, 24, 32};
  for (int k = 0; k < 8; ++k) {
    int T = Ts[k];
    char* a = malloc(n);
    double fresh = copy_par(a, src, n, T);
    double warm = copy_par(a, src, n, T);
    free(a);
    char* b = mmap(NULL, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(b, n, MADV_HUGEPAGE);
    double huge = copy_par(b, src, n, T);
    munmap(b, n);
    printf("threads %2d: fresh %6.1f GB/s  fresh+MADV_HUGEPAGE %6.1f GB/s  prefaulted %6.1f GB/s\n", T, fresh, huge, warm);
  }
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char buf[256] = {0};
  if (f) { fgets(buf, sizeof buf, f); fclose(f); }
  printf("THP enabled: %s", buf);
  return 0;
}
