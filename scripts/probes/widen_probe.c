// u16 -> u32 widening of a 7680x4320 count image on the GPU box's host:
// T threads, resident (pinned-like, pre-faulted) destination, AVX2 streaming
// stores vs a plain loop.  gcc -O2 -mavx2 -pthread widen_probe.c
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + t.tv_nsec * 1e-9; }
typedef struct { uint32_t* d; const uint16_t* s; size_t n; int nt; } Job;
static void widen_nt(uint32_t* d, const uint16_t* s, size_t n) {
  size_t i = 0;
  while (i < n && ((uintptr_t)(d + i) & 31)) { d[i] = s[i]; ++i; }
  for (; i + 16 <= n; i += 16) {
    __m256i a = _mm256_cvtepu16_epi32(_mm_loadu_si128((const __m128i*)(s + i)));
    __m256i b = _mm256_cvtepu16_epi32(_mm_loadu_si128((const __m128i*)(s + i + 8)));
    _mm256_stream_si256((__m256i*)(d + i), a);
    _mm256_stream_si256((__m256i*)(d + i + 8), b);
  }
  for (; i < n; ++i) d[i] = s[i];
  _mm_sfence();
}
static void* run(void* p) {
  Job* j = p;
  if (j->nt) widen_nt(j->d, j->s, j->n);
  else for (size_t i = 0; i < j->n; ++i) j->d[i] = j->s[i];
  return NULL;
}
int main(void) {
  const size_t n = 7680u * 4320u;
  uint16_t* s = aligned_alloc(4096, n * 2);
  uint32_t* d = aligned_alloc(4096, n * 4);
  for (size_t i = 0; i < n; ++i) s[i] = (uint16_t)(i * 2654435761u >> 21);
  memset(d, 1, n * 4);
  int Ts[] = {1, 4, 8, 15};
  for (int k = 0; k < 4; ++k)
    for (int nt = 0; nt < 2; ++nt) {
      int T = Ts[k];
      double best = 1e9;
      for (int r = 0; r < 5; ++r) {
        pthread_t th[32]; Job j[32];
        size_t per = (n + T - 1) / T;
        double t0 = now();
        for (int i = 0; i < T; ++i) {
          size_t lo = i * per, len = lo + per <= n ? per : n - lo;
          j[i] = (Job){d + lo, s + lo, len, nt};
          pthread_create(&th[i], NULL, run, &j[i]);
        }
        for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
        double t = now() - t0;
        if (t < best) best = t;
      }
      for (size_t i = 0; i < n; i += 4099) if (d[i] != s[i]) { printf("MISMATCH\n"); return 1; }
      printf("threads %2d %-6s %.3f ms\n", T, nt ? "NT" : "plain", best * 1e3);
    }
  return 0;
}
