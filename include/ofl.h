/*
 * ofl.h — C-ABI of libofl.so, the B200 (sm_100a) execution engine behind the
 * futurized device/buffer/program API of arXiv 1810.11482 (reference package
 * `offloadrt`, /root/reference/pkg/src/offloadrt).
 *
 * The reference has no FFI; its plug-in seam is the dispatch surface that
 * `Runtime.dispatch(gid)` selects (runtime.py:178-184), implemented by
 * `LocalDispatch` (runtime.py:30-120).  Everything *below* that seam —
 * DeviceObject stream workers (device.py:129-157,247-328), BufferObject
 * storage (buffer.py:26-66), the numba whole-grid executor
 * (kernel/codegen.py:107-128,319-337) — is replaced by the entry points
 * declared here.  They are called only from `CudaDispatch`
 * (paper_1810_11482_b200/runtime.py) through ctypes.  Each entry point names
 * the reference interface it replaces.
 *
 * Conventions
 *   - Every function returns an int status: 0 = OFL_OK, otherwise one of the
 *     codes below.  1..5 are the reference wire codes (errors.py:92-96);
 *     6..9 extend them for allocation, CUDA driver/runtime and NCCL failures.
 *     The message of the most recent failure on the calling thread is
 *     returned by ofl_last_error().
 *   - Stream-ordered operations return a *ticket*: the 1-based position of
 *     the operation on its stream.  Ticket t is complete once every operation
 *     up to and including t on that stream has finished on the device.
 *     Completion is observed lazily (ofl_query / ofl_wait / ofl_notify):
 *     a completion marker (CUDA event or host function) is only placed on
 *     the stream when a ticket is actually observed.
 *   - Every entry point is thread-safe; ctypes drops the GIL around calls.
 *     Host functions enqueued by ofl_notify never call CUDA.
 *   - Pointers are raw device / pinned-host addresses; sizes are bytes unless
 *     the name says elements.  No torch types cross this boundary.
 */
#ifndef OFL_H
#define OFL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OFL_ABI_VERSION 1

/* status codes — errors.py:92-96 (1..5), extended */
#define OFL_OK 0
#define OFL_ERR_UNKNOWN_GID 1
#define OFL_ERR_BAD_ARGS 2
#define OFL_ERR_COMPILE 3
#define OFL_ERR_OOB_ACCESS 4
#define OFL_ERR_INTERNAL 5
#define OFL_ERR_OOM 6
#define OFL_ERR_CUDA 7
#define OFL_ERR_NCCL 8

typedef struct ofl_stream ofl_stream; /* one CUDA stream + its ticket log */
typedef struct ofl_event ofl_event;   /* timing event (bench only) */
typedef struct ofl_comm ofl_comm;     /* one NCCL communicator rank */

/* ---- library ------------------------------------------------------------ */
int ofl_abi_version(void);
const char* ofl_last_error(void);
/* number of kernels this library has launched (evidence for gpu_launches) */
uint64_t ofl_kernel_launches(void);

/* ---- discovery: replaces Runtime._device_infos / DeviceInfo
 *      (runtime.py:161-174, device.py:37-48) ------------------------------ */
int ofl_device_count(int* count);
int ofl_device_props(int dev, char* name, int name_cap, int* cc_major, int* cc_minor,
                     uint64_t* mem_bytes, int* sms, uint64_t* l2_bytes);
/* PCI address "dddd:bb:dd.f" (lower case, as in /sys/bus/pci/devices): the
 * host side binds a GPU's process to the CPUs / NUMA node nearest to it */
int ofl_device_pci_bus_id(int dev, char* out, int cap);

/* ---- streams: replaces DeviceObject.create_stream / _StreamWorker
 *      (device.py:129-157,232-233) ---------------------------------------- */
int ofl_stream_create(int dev, ofl_stream** out);
int ofl_stream_destroy(ofl_stream* s);
/* last ticket enqueued (0 if none) and highest ticket known complete */
uint64_t ofl_stream_tail(ofl_stream* s);
uint64_t ofl_stream_done(ofl_stream* s);
/* raw cudaStream_t, for interop (bench timing) */
void* ofl_stream_handle(ofl_stream* s);

/* ---- memory: replaces DeviceObject.allocate/release + BufferObject storage
 *      (device.py:217-228, buffer.py:26-38); device memory is zero-filled
 *      like np.zeros (buffer.py:32) ----------------------------------------- */
/* ofl_malloc: from the device's stream-ordered pool (cudaMallocAsync);
 * ofl_free of such a buffer is ordered on the device after the work enqueued
 * so far on every stream of the process (cudaFreeAsync after fence events),
 * never a device-wide synchronisation.  ofl_malloc_shareable: a plain
 * cudaMalloc allocation that ofl_ipc_handle can export (stream-ordered
 * allocations have no CUDA IPC handle); ofl_free releases it with cudaFree. */
int ofl_malloc(int dev, uint64_t bytes, void** dptr);
int ofl_malloc_shareable(int dev, uint64_t bytes, void** dptr);
/* CUDA IPC: share a device allocation (from ofl_malloc_shareable) with the other
 * processes of the node (one process per GPU); handles are 64 bytes.  Used
 * by the fused cross-process reduction (collectives.ProcessPeerGroup). */
int ofl_ipc_handle(void* dptr, char* out64);
int ofl_ipc_open(int dev, const char* handle64, void** dptr);
int ofl_ipc_close(int dev, void* dptr);
/* Device-side ordering between processes (ofl_gate.cu): a one-thread kernel
 * that publishes a 64-bit completion counter (after a system fence), and one
 * that polls other ranks' counters (device pointers, e.g. IPC-mapped; the
 * pointer array itself lives in device memory) until each reaches `target`,
 * recording a timeout in *status after ~20 s.  Used by the multi-process
 * heat slabs (bench.ProcessHeatSlabs) so no host round trip orders a pass. */
int ofl_gate_signal(ofl_stream* s, unsigned long long* counter, uint64_t value, uint64_t* ticket);
int ofl_gate_wait(ofl_stream* s, const unsigned long long* const* counters_dev, int count,
                  uint64_t target, unsigned long long* status, uint64_t* ticket);
int ofl_free(int dev, void* dptr);
/* Give the device back every byte released buffers still hold: waits for the
 * frees queued behind other streams' work, trims the pool, unmaps the cached
 * VMM mappings (torch.cuda.empty_cache's role; an allocation that runs out
 * does this by itself, the cheap part first). */
int ofl_trim_memory(int dev);
int ofl_host_alloc(uint64_t bytes, void** hptr); /* pinned, portable */
int ofl_host_free(void* hptr);

/* ---- stream-ordered copies: replace BufferObject.enqueue_write/read
 *      (buffer.py:40-55) and handles.copy (handles.py:119-145) ------------- */
int ofl_h2d(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket);
int ofl_d2h(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket);
int ofl_d2d(ofl_stream* s, void* dst, const void* src, uint64_t bytes, uint64_t* ticket);
/* `rows` consecutive device rows of row_bytes each -> host rows dst_pitch
 * apart (cudaMemcpy2DAsync): a device's packed rows land directly at their
 * place in a strided host image (config 3's cyclic-row assembly; the
 * reference assembles through bytes, harness.py:393-437). */
int ofl_d2h_rows(ofl_stream* s, void* dst, uint64_t dst_pitch, const void* src,
                 uint64_t row_bytes, uint64_t rows, uint64_t* ticket);
/* H2D from pageable memory through a ring of pinned staging slots, the host
 * copy of one chunk overlapping the DMA of the previous one; returns once the
 * source has been fully staged (it may then be reused).  One ticket. */
int ofl_h2d_pageable(ofl_stream* s, void* dst, const void* src, uint64_t bytes,
                     uint64_t* ticket);
/* host-to-host copy on the library's copy threads (staging <-> pageable) */
int ofl_host_memcpy(void* dst, const void* src, uint64_t bytes);
/* D2H into a pinned staging block in `chunk`-byte pieces, each followed by
 * an event; *out receives the pending read (one ticket for the whole read).
 * ofl_collect waits for each piece and copies it to the pageable `dst` on
 * the copy threads while later pieces are still in flight — the staging
 * half of BufferObject.enqueue_read returning `bytes` (buffer.py:49-55).
 * ofl_read_release frees the handle (after ofl_collect, or unobserved). */
typedef struct ofl_read ofl_read;
int ofl_d2h_chunked(ofl_stream* s, void* staging, const void* src, uint64_t bytes,
                    uint64_t chunk, ofl_read** out, uint64_t* ticket);
int ofl_collect(ofl_read* r, void* dst);
int ofl_read_release(ofl_read* r);
/* cross-device copy over NVLink (peer access enabled on first use) */
int ofl_p2p(ofl_stream* s, void* dst, int dst_dev, const void* src, int src_dev,
            uint64_t bytes, uint64_t* ticket);
/* device-side ordering: `waiter` does not run past this point until `on`
 * has completed `ticket` (cudaStreamWaitEvent on a lazily placed marker).
 * With no marker at or after `ticket` yet, one is recorded at `on`'s tail,
 * so a wait on an older ticket also waits for the work enqueued since;
 * `waiter == on` only places that marker — called right after enqueueing,
 * it pins an exact marker for a later wait. */
int ofl_stream_wait(ofl_stream* waiter, ofl_stream* on, uint64_t ticket);

/* ---- completion: replaces Promise fulfilment by the stream worker
 *      (device.py:143-157, futures.py:76-89) --------------------------------
 *   ofl_query  : non-blocking; *ready = 1 once ticket is complete
 *   ofl_wait   : blocks the calling thread until the ticket completes
 *   ofl_notify : when the ticket completes, `token_id` is pushed into the
 *                completion queue and the eventfd returned by
 *                ofl_completion_fd() becomes readable (cudaLaunchHostFunc)
 *   ofl_drain  : pops up to `cap` token ids                                   */
int ofl_query(ofl_stream* s, uint64_t ticket, int* ready);
int ofl_wait(ofl_stream* s, uint64_t ticket);
int ofl_notify(ofl_stream* s, uint64_t ticket, uint64_t token_id);
int ofl_completion_fd(void);
int ofl_completion_post(uint64_t token_id); /* push from the host (wake-ups) */
int ofl_drain(uint64_t* ids, int cap, int* count);

/* ---- timing events (bench.py; CUDA-event timing on the launch stream) --- */
int ofl_event_create(int dev, ofl_event** out);
int ofl_event_record(ofl_event* e, ofl_stream* s);
int ofl_event_elapsed_ms(ofl_event* start, ofl_event* end, float* ms);
int ofl_event_destroy(ofl_event* e);

/* ---- kernels: replace the numba whole-grid executor
 *      (kernel/codegen.py:107-128) for the bound .k programs --------------- */

/* STREAM copy/scale/add/triad over n fp64 elements (op 0..3):
 *   copy  a[i] = b[i]          scale a[i] = s*b[i]
 *   add   a[i] = b[i] + c[i]   triad a[i] = b[i] + s*c[i]
 * IEEE round-to-nearest, no FMA contraction (bit-exact vs the CPU path). */
#define OFL_STREAM_COPY 0
#define OFL_STREAM_SCALE 1
#define OFL_STREAM_ADD 2
#define OFL_STREAM_TRIAD 3
int ofl_stream_op(ofl_stream* s, int op, double* a, const double* b, const double* c,
                  double scalar, uint64_t n, uint64_t* ticket);

/* stencil.k (bench/kernels/stencil.k:2-10): for i < items, i < n:
 *   y[i] = x[i] at i==0 or i==n-1, else 0.5*x[i-1] + x[i] + 0.5*x[i+1]   */
int ofl_stencil(ofl_stream* s, const double* x, double* y, uint64_t n, uint64_t items,
                uint64_t* ticket);
/* stencil2d.k (paper_1810_11482_b200/kernels/stencil2d.k — the 2-D form
 * of bench/kernels/stencil.k, in the reference's kernel language): for
 * gtid < min(items, (w*h) mod 2^32), row = gtid / w, col = gtid % w:
 *   y[g] = x[g] on the boundary ring, else 0.25*(((x[g-w]+x[g-1])+x[g+1])+x[g+w]).
 * x_elems bounds the loads (cells past it are never executed by a checked
 * launch; see bindings._stencil2d_oob). */
int ofl_stencil2d(ofl_stream* s, const double* x, double* y, uint32_t w, uint32_t h,
                  uint64_t items, uint64_t x_elems, uint64_t* ticket);
/* One stencil2d.k step of a row slab (w x h local rows incl. ghost rows)
 * for the multi-GPU 2-D heat equation: writes only the owned rows
 * [own_lo, own_hi) of y, and stores the first / last owned row straight into
 * up_ghost[0..w) / down_ghost[0..w) — the neighbouring slabs' ghost rows on
 * devices up_dev / down_dev (NVLink peer stores; NULL = no neighbour).  The
 * caller orders each step after the neighbours' previous step. */
int ofl_stencil2d_slab(ofl_stream* s, const double* x, double* y, uint32_t w, uint32_t h,
                       uint32_t own_lo, uint32_t own_hi, double* up_ghost, int up_dev,
                       double* down_ghost, int down_dev, uint64_t* ticket);
/* `steps` applications of stencil.k ping-ponging x <-> y (heat equation,
 * BASELINE config 2); the final state is in x if steps is even else in y.
 * Temporal blocking: `tb` steps are fused per pass through HBM (1 = none). */
int ofl_heat(ofl_stream* s, double* x, double* y, uint64_t n, uint64_t steps, int tb,
             uint64_t* ticket);
/* One slab pass of the multi-GPU heat equation (BASELINE config 2; the
 * reference has no multi-device stencil — harness.py:199-230 is single-device,
 * its cross-device path is copy() through the host, handles.py:119-145):
 * k (1..128) stencil.k steps of slab x -> y (length n, local cells 0 and n-1
 * held fixed), writing y only for the owned cells [own_lo, own_hi), and the
 * first / last h owned cells also straight into left_ghost[0..h) /
 * right_ghost[0..h) — the neighbouring slabs' ghost cells, on devices
 * left_dev / right_dev (peer stores over NVLink from the kernel; either
 * pointer may be NULL).  The caller orders each pass after the neighbours'
 * previous pass (ofl_stream_wait). */
int ofl_heat_slab(ofl_stream* s, const double* x, double* y, uint64_t n, int k, uint64_t own_lo,
                  uint64_t own_hi, double* left_ghost, int left_dev, double* right_ghost,
                  int right_dev, uint64_t h, uint64_t* ticket);

/* mandelbrot.k (bench/kernels/mandelbrot.k:6-29), pixels gtid in
 * [0, min(width*height mod 2^32, items)); counts written at out[gtid].
 * Rows py with (py - row_first) % row_step == 0 only (multi-GPU cyclic row
 * split; row_first=0,row_step=1 for the whole image).  compact=1 packs the
 * launch's rows densely: the k-th owned row lands at out[k*width ...]. */
int ofl_mandelbrot(ofl_stream* s, uint32_t* out, uint32_t width, uint32_t height,
                   double re0, double re1, double im0, double im1, double esc,
                   uint32_t max_iter, uint64_t items, uint32_t row_first,
                   uint32_t row_step, int compact, uint64_t* ticket);

/* sum.k (bench/kernels/sum.k:3-11): res[0] = sum(in[0..n)) mod 2^32 */
int ofl_sum_u32(ofl_stream* s, const uint32_t* in, uint32_t* res, uint64_t n,
                uint64_t* ticket);
/* fp32 dot product with fp64 accumulation: res[0] = sum a[i]*b[i] */
int ofl_dot_f32(ofl_stream* s, const float* a, const float* b, double* res, uint64_t n,
                uint64_t* ticket);

/* partition.k (bench/kernels/partition.k:3-8):
 * out[i] = sqrt(sin(v)^2 + cos(v)^2), v = f64((offset + i) mod 2^32), i < count */
/* Fused dot product + allreduce over `nranks` devices driven by this process
 * (BASELINE config 4 without NCCL): rank `rank` reduces its shard like
 * ofl_dot_f32, then its last CTA stores the fp64 partial into slot `rank` of
 * every rank's exchange block (xchg[r], ofl_xchg_bytes() bytes of zeroed
 * device memory on device devs[r]; NVLink peer stores), bumps every rank's
 * arrival counter (system-scope atomics), waits for all partials of round
 * `round` (0, 1, 2, ... per call on the group) and sums them in rank order,
 * so every rank's res[0] holds the identical total.  A rank that waits
 * longer than 20 s writes NaN and sets the block's status word. */
#define OFL_MAX_PEER_RANKS 16
int ofl_xchg_bytes(void);
int ofl_dot_f32_allreduce(ofl_stream* s, const float* a, const float* b, double* res, uint64_t n,
                          int rank, int nranks, void* const* xchg, const int* devs,
                          uint64_t round, uint64_t* ticket);
int ofl_partition(ofl_stream* s, double* out, uint32_t offset, uint64_t count,
                  uint64_t* ticket);

/* ---- run-time compiled kernels: replace numba compile_ir
 *      (kernel/codegen.py:319-337) for kernels with no hand-written binding.
 *      NVRTC is dlopen'ed (toolkit copy first, `nvrtc_path` as a hint). ---- */
typedef struct ofl_jit ofl_jit;
int ofl_jit_available(const char* nvrtc_path);
int ofl_jit_compile(int dev, const char* src, const char* entry, ofl_jit** out, char* log,
                    int logcap);
/* params: kernel parameter pointers (cudaLaunchKernel convention) */
int ofl_jit_launch(ofl_stream* s, ofl_jit* k, void** params, uint64_t blocks, int threads,
                   uint64_t* ticket);
int ofl_jit_destroy(ofl_jit* k);
/* 0xFF-fill device bytes in stream order (error-record reset) */
int ofl_fill_ones(ofl_stream* s, void* dptr, uint64_t bytes, uint64_t* ticket);

/* ---- raw-CUDA baseline for the futurization-overhead benchmark ----------
 * `steps` x (cudaMemcpyAsync H2D of `bytes` from `src` + one small triad
 * launch over n elements) on the stream, timed on the host clock.
 * mode 0: stream order only; 1: event-chained steps; 2: sync every step. */
int ofl_bench_raw_chain(ofl_stream* s, void* dst, const void* src, uint64_t bytes, double* a,
                        const double* b, const double* c, uint64_t n, uint64_t steps, int mode,
                        double* seconds);

/* FP64 DMUL/DADD issue rate of the device (ops/s), the roofline denominator
 * of the no-FMA Mandelbrot kernel. */
int ofl_bench_fp64_peak(ofl_stream* s, double* ops_per_s);

/* ---- NCCL (dlopen'ed; the process's already-loaded libnccl.so.2 wins) ---- */
#define OFL_DT_U32 0
#define OFL_DT_F64 1
#define OFL_DT_F32 2
#define OFL_OP_SUM 0
#define OFL_OP_MAX 1
int ofl_nccl_available(const char* lib_path);
int ofl_nccl_unique_id(char* id128);
int ofl_nccl_init_all(int ndev, const int* devs, ofl_comm** comms);
int ofl_nccl_init_rank(int nranks, int rank, int dev, const char* id128, ofl_comm** comm);
int ofl_allreduce(ofl_comm* c, ofl_stream* s, const void* send, void* recv, uint64_t count,
                  int dtype, int op, uint64_t* ticket);
/* several ranks of one process in a single NCCL group (ncclGroupStart/End) */
int ofl_allreduce_group(int n, ofl_comm** comms, ofl_stream** streams, void** send,
                        void** recv, uint64_t count, int dtype, int op, uint64_t* tickets);
int ofl_comm_destroy(ofl_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* OFL_H */
