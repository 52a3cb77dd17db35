/* Test double of libofl.so for CPU-only host-logic profiling: every entry
 * point of include/ofl.h, no device, no data movement (buffers are host
 * malloc).  NEVER used by the product path; load it explicitly with
 * OFL_LIB=tests/fakes/_build/libnull_ofl.so in probes/tests that only
 * exercise Python-side logic. */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <sys/eventfd.h>
#include <unistd.h>

typedef struct { uint64_t tail, done; } S;
static uint64_t launches;
static int efd = -1;
int ofl_abi_version(void) { return 1; }
const char* ofl_last_error(void) { return "null"; }
uint64_t ofl_kernel_launches(void) { return launches; }
int ofl_device_count(int* c) { *c = 1; return 0; }
int ofl_device_props(int d, char* name, int cap, int* ma, int* mi, uint64_t* mem, int* sms, uint64_t* l2) {
  (void)d; strncpy(name, "null", cap); *ma = 10; *mi = 0; *mem = 1ull << 37; *sms = 148; *l2 = 1 << 27; return 0; }
int ofl_device_pci_bus_id(int d, char* out, int cap) {
  (void)d; if (!out || cap < 13) return 2; strncpy(out, "0000:00:00.0", cap); return 0; }
int ofl_stream_create(int d, void** out) { (void)d; *out = calloc(1, sizeof(S)); return 0; }
int ofl_stream_destroy(void* s) { free(s); return 0; }
uint64_t ofl_stream_tail(void* s) { return ((S*)s)->tail; }
uint64_t ofl_stream_done(void* s) { return ((S*)s)->done; }
void* ofl_stream_handle(void* s) { return s; }
int ofl_malloc(int d, uint64_t n, void** p) { (void)d; *p = calloc(1, n); return 0; }
int ofl_free(int d, void* p) { (void)d; free(p); return 0; }
int ofl_trim_memory(int d) { (void)d; return 0; }
int ofl_malloc_shareable(int d, uint64_t n, void** p) { (void)d; *p = calloc(1, n); return 0; }
int ofl_host_alloc(uint64_t n, void** p) { *p = calloc(1, n ? n : 1); return 0; }
int ofl_host_free(void* p) { free(p); return 0; }
static int op(void* s, uint64_t* t) { S* st = (S*)s; if (!st) return 2; *t = ++st->tail; return 0; }
int ofl_h2d(void* s, void* d, const void* x, uint64_t n, uint64_t* t) { memcpy(d, x, n); return op(s, t); }
int ofl_d2h(void* s, void* d, const void* x, uint64_t n, uint64_t* t) { memcpy(d, x, n); return op(s, t); }
int ofl_d2d(void* s, void* d, const void* x, uint64_t n, uint64_t* t) { memmove(d, x, n); return op(s, t); }
int ofl_p2p(void* s, void* d, int dd, const void* x, int sd, uint64_t n, uint64_t* t) { (void)dd; (void)sd; memmove(d, x, n); return op(s, t); }
int ofl_stream_wait(void* w, void* o, uint64_t t) { (void)w; (void)o; (void)t; return 0; }
int ofl_query(void* s, uint64_t t, int* r) { S* st = (S*)s; st->done = st->tail; *r = t <= st->done; return 0; }
int ofl_wait(void* s, uint64_t t) { S* st = (S*)s; (void)t; st->done = st->tail; return 0; }
static void post(void) { uint64_t one = 1; if (efd < 0) efd = eventfd(0, 0); if (write(efd, &one, 8) < 0) {} }
static uint64_t q[1 << 16]; static int qn;
int ofl_notify(void* s, uint64_t t, uint64_t id) { (void)t; ((S*)s)->done = ((S*)s)->tail; q[qn++ & 0xffff] = id; post(); return 0; }
int ofl_completion_fd(void) { if (efd < 0) efd = eventfd(0, 0); return efd; }
int ofl_completion_post(uint64_t id) { q[qn++ & 0xffff] = id; post(); return 0; }
int ofl_drain(uint64_t* ids, int cap, int* c) { int n = qn < cap ? qn : cap; memcpy(ids, q, n * 8); memmove(q, q + n, (qn - n) * 8); qn -= n; *c = n; return 0; }
int ofl_event_create(int d, void** e) { (void)d; *e = calloc(1, 8); return 0; }
int ofl_event_record(void* e, void* s) { (void)e; (void)s; return 0; }
int ofl_event_elapsed_ms(void* a, void* b, float* ms) { (void)a; (void)b; *ms = 1; return 0; }
int ofl_event_destroy(void* e) { free(e); return 0; }
int ofl_stream_op(void* s, int o, void* a, const void* b, const void* c, double x, uint64_t n, uint64_t* t) { (void)o; (void)a; (void)b; (void)c; (void)x; (void)n; launches++; return op(s, t); }
int ofl_stencil(void* s, const void* x, void* y, uint64_t n, uint64_t m, uint64_t* t) { (void)x; (void)y; (void)n; (void)m; launches++; return op(s, t); }
int ofl_heat(void* s, void* x, void* y, uint64_t n, uint64_t k, int tb, uint64_t* t) { (void)x; (void)y; (void)n; (void)k; (void)tb; launches++; return op(s, t); }
int ofl_heat_slab(void* s, const void* x, void* y, uint64_t n, int k, uint64_t lo, uint64_t hi, void* l, int ld, void* r, int rd, uint64_t h, uint64_t* t) { (void)x; (void)y; (void)n; (void)k; (void)lo; (void)hi; (void)l; (void)ld; (void)r; (void)rd; (void)h; launches++; return op(s, t); }
int ofl_stencil2d(void* s, const void* x, void* y, uint32_t w, uint32_t h, uint64_t m, uint64_t lx, uint64_t* t) { (void)x; (void)y; (void)w; (void)h; (void)m; (void)lx; launches++; return op(s, t); }
int ofl_stencil2d_slab(void* s, const void* x, void* y, uint32_t w, uint32_t h, uint32_t lo, uint32_t hi, void* u, int ud, void* d, int dd, uint64_t* t) { (void)x; (void)y; (void)w; (void)h; (void)lo; (void)hi; (void)u; (void)ud; (void)d; (void)dd; launches++; return op(s, t); }
int ofl_xchg_bytes(void) { return 272; }
int ofl_dot_f32_allreduce(void* s, const void* a, const void* b, void* r, uint64_t n, int rk, int nr, void* const* x, const int* d, uint64_t rd, uint64_t* t) { (void)a; (void)b; (void)r; (void)n; (void)rk; (void)nr; (void)x; (void)d; (void)rd; launches++; return op(s, t); }
int ofl_mandelbrot(void* s, void* o, uint32_t w, uint32_t h, double a, double b, double c, double d, double e, uint32_t mi, uint64_t it, uint32_t rf, uint32_t rs, int cp, uint64_t* t) {
  (void)o; (void)w; (void)h; (void)a; (void)b; (void)c; (void)d; (void)e; (void)mi; (void)it; (void)rf; (void)rs; (void)cp; launches++; return op(s, t); }
int ofl_sum_u32(void* s, const void* i, void* r, uint64_t n, uint64_t* t) { (void)i; (void)r; (void)n; launches++; return op(s, t); }
int ofl_dot_f32(void* s, const void* a, const void* b, void* r, uint64_t n, uint64_t* t) { (void)a; (void)b; (void)r; (void)n; launches++; return op(s, t); }
int ofl_partition(void* s, void* o, uint32_t off, uint64_t n, uint64_t* t) { (void)o; (void)off; (void)n; launches++; return op(s, t); }
int ofl_bench_raw_chain(void* s, void* d, const void* x, uint64_t b, void* a, const void* bb, const void* c, uint64_t n, uint64_t k, int m, double* sec) {
  (void)s; (void)d; (void)x; (void)b; (void)a; (void)bb; (void)c; (void)n; (void)k; (void)m; *sec = 0; return 0; }
int ofl_nccl_available(const char* p) { (void)p; return 8; }
int ofl_nccl_unique_id(char* id) { memset(id, 0, 128); return 8; }
int ofl_nccl_init_all(int n, const int* d, void** c) { (void)n; (void)d; (void)c; return 8; }
int ofl_nccl_init_rank(int n, int r, int d, const char* id, void** c) { (void)n; (void)r; (void)d; (void)id; (void)c; return 8; }
int ofl_allreduce(void* c, void* s, const void* a, void* b, uint64_t n, int d, int o, uint64_t* t) { (void)c; (void)s; (void)a; (void)b; (void)n; (void)d; (void)o; (void)t; return 8; }
int ofl_allreduce_group(int n, void** c, void** s, void** a, void** b, uint64_t k, int d, int o, uint64_t* t) { (void)n; (void)c; (void)s; (void)a; (void)b; (void)k; (void)d; (void)o; (void)t; return 8; }
int ofl_comm_destroy(void* c) { (void)c; return 0; }
int ofl_bench_fp64_peak(void* s, double* v) { (void)s; *v = 0; return 0; }
int ofl_jit_available(const char* p) { (void)p; return 3; }
int ofl_jit_compile(int d, const char* s, const char* e, void** o, char* l, int c) { (void)d; (void)s; (void)e; (void)o; (void)l; (void)c; return 3; }
int ofl_jit_launch(void* s, void* k, void** p, uint64_t b, int t, uint64_t* tk) { (void)k; (void)p; (void)b; (void)t; return op(s, tk); }
int ofl_jit_destroy(void* k) { (void)k; return 0; }
int ofl_fill_ones(void* s, void* d, uint64_t n, uint64_t* t) { memset(d, 0xff, n); return op(s, t); }
int ofl_d2h_rows(void* s, void* d, uint64_t dp, const void* x, uint64_t rb, uint64_t r, uint64_t* t) { for (uint64_t i = 0; i < r; ++i) memcpy((char*)d + i * dp, (const char*)x + i * rb, rb); return op(s, t); }
int ofl_ipc_handle(void* d, char* o) { (void)d; memset(o, 0, 64); return 2; }
int ofl_ipc_open(int dev, const char* h, void** d) { (void)dev; (void)h; (void)d; return 2; }
int ofl_ipc_close(int dev, void* d) { (void)dev; (void)d; return 0; }
int ofl_gate_signal(void* s, void* c, uint64_t v, uint64_t* t) { (void)c; (void)v; return op(s, t); }
int ofl_gate_wait(void* s, const void* c, int n, uint64_t tg, void* st, uint64_t* t) { (void)c; (void)n; (void)tg; (void)st; return op(s, t); }
int ofl_h2d_pageable(void* s, void* d, const void* x, uint64_t n, uint64_t* t) { memcpy(d, x, n); return op(s, t); }
int ofl_host_memcpy(void* d, const void* s, uint64_t n) { memcpy(d, s, n); return 0; }
typedef struct { void* staging; uint64_t bytes; } R;
int ofl_d2h_chunked(void* s, void* st, const void* x, uint64_t n, uint64_t c, void** out, uint64_t* t) {
  (void)c; memcpy(st, x, n); R* r = malloc(sizeof(R)); r->staging = st; r->bytes = n; *out = r; return op(s, t); }
int ofl_collect(void* r, void* dst) { memcpy(dst, ((R*)r)->staging, ((R*)r)->bytes); return 0; }
int ofl_read_release(void* r) { free(r); return 0; }
