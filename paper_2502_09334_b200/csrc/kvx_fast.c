/*
 * _kvx_fast: CPython fast-call shims for the two per-hand-off entry points of
 * the native pair (kvx_pair_send / kvx_pair_recv, include/kvx.h).
 *
 * The hand-off itself is one kernel launch per end; for short prompts the
 * host cost of issuing it is part of the hand-off's alpha (the reference's
 * per-hand-off alpha, costs.py:103).  ctypes converts eleven arguments per
 * call through its generic marshalling; these METH_FASTCALL shims take plain
 * Python ints (None = NULL) and call the C-ABI function pointers the Python
 * layer binds from the already-loaded _kvx.so (bind()), so there is exactly
 * one copy of the library and its state.  The GIL is released around the call,
 * as ctypes does.  No CUDA or torch types here: this file only forwards.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*pair_fn)(void*, uint64_t, const void*, const void*, int64_t, const int64_t*,
                       int64_t, int, int, int, void*);

static pair_fn g_send = NULL, g_recv = NULL;

static int as_i64(PyObject* o, long long* out) {
  if (o == Py_None) {
    *out = 0;
    return 0;
  }
  *out = PyLong_AsLongLong(o);
  return (*out == -1 && PyErr_Occurred()) ? -1 : 0;
}

static PyObject* call(pair_fn f, PyObject* const* args, Py_ssize_t nargs) {
  if (!f) {
    PyErr_SetString(PyExc_RuntimeError, "_kvx_fast: bind() the library first");
    return NULL;
  }
  if (nargs != 11) {
    PyErr_SetString(PyExc_TypeError, "_kvx_fast: expected 11 arguments");
    return NULL;
  }
  long long a[11];
  for (int i = 0; i < 11; ++i)
    if (as_i64(args[i], &a[i])) return NULL;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = f((void*)(intptr_t)a[0], (uint64_t)a[1], (const void*)(intptr_t)a[2],
         (const void*)(intptr_t)a[3], (int64_t)a[4], (const int64_t*)(intptr_t)a[5],
         (int64_t)a[6], (int)a[7], (int)a[8], (int)a[9], (void*)(intptr_t)a[10]);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

static PyObject* pair_send(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  return call(g_send, args, nargs);
}

static PyObject* pair_recv(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  return call(g_recv, args, nargs);
}

/* bind(send_addr, recv_addr): addresses of kvx_pair_send / kvx_pair_recv */
static PyObject* bind(PyObject* self, PyObject* args) {
  (void)self;
  unsigned long long s = 0, r = 0;
  if (!PyArg_ParseTuple(args, "KK", &s, &r)) return NULL;
  g_send = (pair_fn)(uintptr_t)s;
  g_recv = (pair_fn)(uintptr_t)r;
  Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"bind", bind, METH_VARARGS, "bind(send_addr, recv_addr)"},
    {"pair_send", (PyCFunction)(void (*)(void))pair_send, METH_FASTCALL,
     "kvx_pair_send(pair, epoch, k, v, src_layer_stride, src_slots, n_tokens, plane_heads, "
     "head_offset, flags, stream) -> rc"},
    {"pair_recv", (PyCFunction)(void (*)(void))pair_recv, METH_FASTCALL,
     "kvx_pair_recv(pair, epoch, k, v, dst_layer_stride, dst_slots, n_tokens, plane_heads, "
     "head_offset, flags, stream) -> rc"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_kvx_fast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__kvx_fast(void) { return PyModule_Create(&module); }
