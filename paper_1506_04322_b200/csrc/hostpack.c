/* _hostpack: CPython helper for GraphBatch (config 4, feature_matrix
 * analytics.py:91-131).  Collecting the data pointers and lengths of
 * thousands of per-graph numpy pair arrays costs ~1 us each through
 * `__array_interface__`; here it is one pass over the sequence through the
 * buffer protocol (no numpy C API, no CPython internals).  The pointers go
 * straight into gd_graph_create_batch_list (include/gd_api.h). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

/* int64 (k, 2) C-contiguous?  format "l" / "q" (optionally prefixed) */
static int pairs_ok(const Py_buffer* v) {
  const char* f = v->format;
  if (!f || v->itemsize != 8 || v->ndim != 2 || v->shape[1] != 2) return 0;
  if (*f == '@' || *f == '=' || *f == '<') f++;
  if ((f[0] != 'l' && f[0] != 'q') || f[1] != 0) return 0;
  return PyBuffer_IsContiguous(v, 'C');
}

/* gather(seq, ptrs, offs) -> index of the first element that is not an
 * int64 (k, 2) C-contiguous buffer, or -1: ptrs[i] = data address of seq[i],
 * offs[0] = 0, offs[i + 1] = offs[i] + k_i.  ptrs / offs: writable uint64 /
 * int64 buffers of len(seq) and len(seq) + 1 elements.  The caller keeps seq
 * alive while the pointers are in use. */
static PyObject* gather(PyObject* self, PyObject* args) {
  PyObject *seq, *ptrs_o, *offs_o;
  if (!PyArg_ParseTuple(args, "OOO", &seq, &ptrs_o, &offs_o)) return NULL;
  PyObject* fast = PySequence_Fast(seq, "gather: a sequence of arrays is required");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  Py_buffer pb, ob;
  if (PyObject_GetBuffer(ptrs_o, &pb, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) < 0) {
    Py_DECREF(fast);
    return NULL;
  }
  if (PyObject_GetBuffer(offs_o, &ob, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) < 0) {
    PyBuffer_Release(&pb);
    Py_DECREF(fast);
    return NULL;
  }
  long bad = -1;
  if (pb.len < (Py_ssize_t)(8 * n) || ob.len < (Py_ssize_t)(8 * (n + 1))) {
    PyErr_SetString(PyExc_ValueError, "gather: output buffers too small");
    bad = -2;
  } else {
    uint64_t* ptrs = (uint64_t*)pb.buf;
    int64_t* offs = (int64_t*)ob.buf;
    offs[0] = 0;
    PyObject** items = PySequence_Fast_ITEMS(fast);
    for (Py_ssize_t i = 0; i < n; i++) {
      Py_buffer v;
      if (PyObject_GetBuffer(items[i], &v, PyBUF_FORMAT | PyBUF_STRIDES) < 0) {
        PyErr_Clear();
        bad = (long)i;
        break;
      }
      const int ok = pairs_ok(&v);
      if (ok) {
        ptrs[i] = (uint64_t)(uintptr_t)v.buf;
        offs[i + 1] = offs[i] + (int64_t)v.shape[0];
      }
      PyBuffer_Release(&v);
      if (!ok) {
        bad = (long)i;
        break;
      }
    }
  }
  PyBuffer_Release(&ob);
  PyBuffer_Release(&pb);
  Py_DECREF(fast);
  if (bad == -2) return NULL;
  return PyLong_FromLong(bad);
}

static PyMethodDef methods[] = {
    {"gather", gather, METH_VARARGS,
     "gather(seq, ptrs, offs) -> first non-conforming index or -1"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostpack",
                                    "pointer/offset gathering for graph batches", -1, methods};

PyMODINIT_FUNC PyInit__hostpack(void) { return PyModule_Create(&module); }
