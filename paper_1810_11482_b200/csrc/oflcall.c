/* _oflcall — vectorcall entry points for the per-operation hot calls of the
 * futures layer (BASELINE config 5: per-future overhead).
 *
 * ctypes marshals every argument through its argtypes converters (about
 * 1.3 us for a 5-argument call on the bench host); the futurized write+run
 * chain makes two such calls per step.  This module calls the same libofl
 * entry points through function pointers taken from the already-loaded
 * ctypes library (`bind`), so the one library the rest of the runtime uses —
 * including a substitute loaded through OFL_LIB — is the one called.
 *
 * Every call that can block releases the GIL around the C call (as ctypes
 * does; query never blocks: a cudaEventQuery) and returns
 * the operation's ticket, or -status when libofl reports an error (wait
 * returns the status), so the caller raises exactly what the ctypes path
 * raises (_native.error_for).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <sys/mman.h>

typedef int (*copy_fn)(void*, void*, const void*, uint64_t, uint64_t*);
typedef int (*stream_op_fn)(void*, int, double*, const double*, const double*, double, uint64_t,
                            uint64_t*);

typedef int (*wait_fn)(void*, uint64_t);
typedef int (*query_fn)(void*, uint64_t, int*);
typedef int (*collect_fn)(void*, void*);

static copy_fn p_h2d = NULL;
static stream_op_fn p_stream_op = NULL;
static wait_fn p_wait = NULL;
static query_fn p_query = NULL;
static collect_fn p_collect = NULL;

static int as_u64(PyObject* o, uint64_t* out) {
  if (o == Py_None) {
    *out = 0;
    return 0;
  }
  unsigned long long v = PyLong_AsUnsignedLongLong(o);
  if (v == (unsigned long long)-1 && PyErr_Occurred()) return -1;
  *out = (uint64_t)v;
  return 0;
}

static PyObject* result(int status, uint64_t ticket) {
  if (status) return PyLong_FromLong(-(long)status);
  return PyLong_FromUnsignedLongLong(ticket);
}

/* bind(addr_ofl_h2d, addr_ofl_stream_op, addr_ofl_wait[, addr_ofl_query[, addr_ofl_collect]]) */
static PyObject* oc_bind(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t a[5] = {0, 0, 0, 0, 0};
  if (n < 3 || n > 5) {
    PyErr_SetString(PyExc_TypeError, "bind expects 3 to 5 function addresses");
    return NULL;
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    if (as_u64(args[i], &a[i])) return NULL;
    if (!a[i]) {
      PyErr_SetString(PyExc_ValueError, "null function address");
      return NULL;
    }
  }
  p_h2d = (copy_fn)(uintptr_t)a[0];
  p_stream_op = (stream_op_fn)(uintptr_t)a[1];
  p_wait = (wait_fn)(uintptr_t)a[2];
  p_query = (query_fn)(uintptr_t)a[3];
  p_collect = (collect_fn)(uintptr_t)a[4];
  Py_RETURN_NONE;
}

/* collect_bytes(read_handle, nbytes) -> bytes | -status   (ofl_collect into a
 * new bytes object: allocated uninitialised — no zero fill — and advised
 * to use huge pages, so first-touch page faults cost 512x fewer traps;
 * filled on the library's copy threads with the GIL released) */
static PyObject* oc_collect_bytes(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t h, nbytes;
  if (n != 2) {
    PyErr_SetString(PyExc_TypeError, "collect_bytes expects 2 arguments");
    return NULL;
  }
  if (!p_collect) {
    PyErr_SetString(PyExc_RuntimeError, "_oflcall collect not bound");
    return NULL;
  }
  if (as_u64(args[0], &h) || as_u64(args[1], &nbytes)) return NULL;
  PyObject* out = PyBytes_FromStringAndSize(NULL, (Py_ssize_t)nbytes);
  if (!out) return NULL;
  char* buf = PyBytes_AS_STRING(out);
  const uintptr_t page = 2u << 20;
  const uintptr_t lo = ((uintptr_t)buf + page - 1) & ~(page - 1);
  const uintptr_t hi = ((uintptr_t)buf + nbytes) & ~(page - 1);
  if (hi > lo) (void)madvise((void*)lo, hi - lo, MADV_HUGEPAGE);
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = p_collect((void*)(uintptr_t)h, buf);
  Py_END_ALLOW_THREADS
  if (status) {
    Py_DECREF(out);
    return PyLong_FromLong(-(long)status);
  }
  return out;
}

/* query(stream, ticket) -> 1 ready | 0 pending | -status   (ofl_query; never blocks) */
static PyObject* oc_query(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t s, ticket;
  if (n != 2) {
    PyErr_SetString(PyExc_TypeError, "query expects 2 arguments");
    return NULL;
  }
  if (!p_query) {
    PyErr_SetString(PyExc_RuntimeError, "_oflcall query not bound");
    return NULL;
  }
  if (as_u64(args[0], &s) || as_u64(args[1], &ticket)) return NULL;
  int ready = 0;
  const int status = p_query((void*)(uintptr_t)s, ticket, &ready);
  return PyLong_FromLong(status ? -(long)status : (ready ? 1 : 0));
}

/* wait(stream, ticket) -> status   (ofl_wait; blocks with the GIL released) */
static PyObject* oc_wait(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t s, ticket;
  if (n != 2) {
    PyErr_SetString(PyExc_TypeError, "wait expects 2 arguments");
    return NULL;
  }
  if (!p_wait) {
    PyErr_SetString(PyExc_RuntimeError, "_oflcall not bound");
    return NULL;
  }
  if (as_u64(args[0], &s) || as_u64(args[1], &ticket)) return NULL;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = p_wait((void*)(uintptr_t)s, ticket);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(status);
}

/* h2d(stream, dst, src, bytes) -> ticket | -status   (ofl_h2d) */
static PyObject* oc_h2d(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t s, dst, src, bytes, ticket = 0;
  if (n != 4) {
    PyErr_SetString(PyExc_TypeError, "h2d expects 4 arguments");
    return NULL;
  }
  if (!p_h2d) {
    PyErr_SetString(PyExc_RuntimeError, "_oflcall not bound");
    return NULL;
  }
  if (as_u64(args[0], &s) || as_u64(args[1], &dst) || as_u64(args[2], &src) ||
      as_u64(args[3], &bytes))
    return NULL;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = p_h2d((void*)(uintptr_t)s, (void*)(uintptr_t)dst, (const void*)(uintptr_t)src, bytes,
                 &ticket);
  Py_END_ALLOW_THREADS
  return result(status, ticket);
}

/* stream_op(stream, op, a, b, c, scalar, n) -> ticket | -status   (ofl_stream_op) */
static PyObject* oc_stream_op(PyObject* self, PyObject* const* args, Py_ssize_t n) {
  (void)self;
  uint64_t s, a, b, c, count, ticket = 0;
  if (n != 7) {
    PyErr_SetString(PyExc_TypeError, "stream_op expects 7 arguments");
    return NULL;
  }
  if (!p_stream_op) {
    PyErr_SetString(PyExc_RuntimeError, "_oflcall not bound");
    return NULL;
  }
  const long op = PyLong_AsLong(args[1]);
  if (op == -1 && PyErr_Occurred()) return NULL;
  const double scalar = PyFloat_AsDouble(args[5]);
  if (scalar == -1.0 && PyErr_Occurred()) return NULL;
  if (as_u64(args[0], &s) || as_u64(args[2], &a) || as_u64(args[3], &b) ||
      as_u64(args[4], &c) || as_u64(args[6], &count))
    return NULL;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = p_stream_op((void*)(uintptr_t)s, (int)op, (double*)(uintptr_t)a,
                       (const double*)(uintptr_t)b, (const double*)(uintptr_t)c, scalar, count,
                       &ticket);
  Py_END_ALLOW_THREADS
  return result(status, ticket);
}

static PyMethodDef methods[] = {
    {"bind", (PyCFunction)(void (*)(void))oc_bind, METH_FASTCALL, "bind libofl entry points"},
    {"h2d", (PyCFunction)(void (*)(void))oc_h2d, METH_FASTCALL, "ofl_h2d -> ticket | -status"},
    {"wait", (PyCFunction)(void (*)(void))oc_wait, METH_FASTCALL, "ofl_wait -> status"},
    {"collect_bytes", (PyCFunction)(void (*)(void))oc_collect_bytes, METH_FASTCALL,
     "ofl_collect into a new bytes object -> bytes | -status"},
    {"query", (PyCFunction)(void (*)(void))oc_query, METH_FASTCALL,
     "ofl_query -> 1 ready | 0 pending | -status"},
    {"stream_op", (PyCFunction)(void (*)(void))oc_stream_op, METH_FASTCALL,
     "ofl_stream_op -> ticket | -status"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_oflcall", NULL, -1, methods};

PyMODINIT_FUNC PyInit__oflcall(void) { return PyModule_Create(&module); }
