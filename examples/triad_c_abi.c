/* A futurized STREAM triad driven through the C-ABI alone (no Python):
 * what a non-Python host (a cgo / JNI / N-API binding of the reference's
 * dispatch seam) would do.  Pinned host buffers, stream-ordered copies, the
 * sm_100a triad, and ticket-based completion (ofl_wait).  Checks the result
 * bit for bit against a plain C loop without FMA contraction.
 *
 *   gcc -O2 -ffp-contract=off -Iinclude examples/triad_c_abi.c \
 *       -Lpaper_1810_11482_b200/lib -lofl -Wl,-rpath,$PWD/paper_1810_11482_b200/lib -o /tmp/triad_c
 *   /tmp/triad_c   (needs a GPU)
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ofl.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    int st_ = (call);                                                      \
    if (st_) {                                                             \
      fprintf(stderr, "%s failed (%d): %s\n", #call, st_, ofl_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(void) {
  const uint64_t n = (1u << 22) + 7;  /* odd: exercises the tail */
  const uint64_t bytes = n * sizeof(double);
  int count = 0;
  CHECK(ofl_device_count(&count));
  if (count < 1) {
    fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  ofl_stream* s = NULL;
  CHECK(ofl_stream_create(0, &s));
  void *a = NULL, *b = NULL, *c = NULL, *hb = NULL, *hc = NULL, *ha = NULL;
  CHECK(ofl_malloc(0, bytes, &a));
  CHECK(ofl_malloc(0, bytes, &b));
  CHECK(ofl_malloc(0, bytes, &c));
  CHECK(ofl_host_alloc(bytes, &hb));
  CHECK(ofl_host_alloc(bytes, &hc));
  CHECK(ofl_host_alloc(bytes, &ha));
  double *pb = (double*)hb, *pc = (double*)hc, *pa = (double*)ha;
  uint64_t seed = 20180214;
  for (uint64_t i = 0; i < n; ++i) {
    seed = seed * 6364136223846793005ull + 1442695040888963407ull;
    pb[i] = (double)(seed >> 11) * 0x1p-53;
    seed = seed * 6364136223846793005ull + 1442695040888963407ull;
    pc[i] = (double)(seed >> 11) * 0x1p-53;
  }
  uint64_t t = 0;
  CHECK(ofl_h2d(s, b, hb, bytes, &t));
  CHECK(ofl_h2d(s, c, hc, bytes, &t));
  CHECK(ofl_stream_op(s, OFL_STREAM_TRIAD, (double*)a, (const double*)b, (const double*)c, 3.0,
                      n, &t));
  CHECK(ofl_d2h(s, ha, a, bytes, &t));
  CHECK(ofl_wait(s, t)); /* the read's ticket covers everything before it */
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    volatile double prod = 3.0 * pc[i];
    double want = pb[i] + prod;
    if (memcmp(&want, &pa[i], sizeof(double)) != 0) ++bad;
  }
  printf("triad via the C-ABI: n=%llu, %llu mismatches, last ticket %llu\n",
         (unsigned long long)n, (unsigned long long)bad, (unsigned long long)t);
  ofl_free(0, a);
  ofl_free(0, b);
  ofl_free(0, c);
  ofl_host_free(hb);
  ofl_host_free(hc);
  ofl_host_free(ha);
  ofl_stream_destroy(s);
  return bad ? 2 : 0;
}
