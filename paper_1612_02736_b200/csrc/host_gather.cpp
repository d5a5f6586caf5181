// Host-side helper of the drop-in API (CPython extension `_hps_host`): gathers a body-load mapping
// {leaf id: (m,) float64} (the reference's convention, solver.py:241-253) into one contiguous
// (n_leaves, m) table in leaf-row order — the page-locked staging buffer of the host->device
// copy. The lookups and shape checks run under the GIL (~30 ns per leaf); the row copies run
// with the GIL released on a few threads (np.concatenate does the same work on one thread with
// per-array dispatch: 0.76 ms for config 2's 4096 x 196 table, half of the device solve).
// Not on the device path: without this module solver.py falls back to numpy.
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <Python.h>
#include <numpy/arrayobject.h>

#include <cstring>
#include <thread>
#include <vector>

namespace {

// gather_rows(mapping, ids, out, nthreads) -> int
//   ids: list of leaf ids (Python ints) in destination row order; out: C-contiguous float64 (n, m).
//   Returns -1 on success. Returns the position (>= 0) of the first value that is not a
//   C-contiguous 1-D float64 array of length m — the caller re-runs its generic path, which
//   converts or raises with the reference's message. A missing key raises KeyError.
PyObject* gather_rows(PyObject*, PyObject* args) {
  PyObject *mapping, *ids, *out_obj;
  int nthreads = 4;
  if (!PyArg_ParseTuple(args, "OOO|i", &mapping, &ids, &out_obj, &nthreads)) return nullptr;
  if (!PyList_Check(ids)) {
    PyErr_SetString(PyExc_TypeError, "ids must be a list");
    return nullptr;
  }
  if (!PyArray_Check(out_obj)) {
    PyErr_SetString(PyExc_TypeError, "out must be a numpy array");
    return nullptr;
  }
  PyArrayObject* out = reinterpret_cast<PyArrayObject*>(out_obj);
  const Py_ssize_t n = PyList_GET_SIZE(ids);
  if (PyArray_TYPE(out) != NPY_DOUBLE || PyArray_NDIM(out) != 2 || !PyArray_IS_C_CONTIGUOUS(out) ||
      !PyArray_ISWRITEABLE(out) || PyArray_DIM(out, 0) != n) {
    PyErr_SetString(PyExc_ValueError, "out must be a writable C-contiguous float64 array of shape (len(ids), m)");
    return nullptr;
  }
  const npy_intp m = PyArray_DIM(out, 1);
  std::vector<const char*> src((size_t)n);
  std::vector<PyObject*> held;  // new references from a generic mapping's __getitem__
  const bool is_dict = PyDict_CheckExact(mapping);
  if (!is_dict) held.reserve((size_t)n);
  Py_ssize_t bad = -1;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* key = PyList_GET_ITEM(ids, i);
    PyObject* v;
    if (is_dict) {
      v = PyDict_GetItemWithError(mapping, key);  // borrowed
      if (!v) {
        if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, key);
        return nullptr;
      }
    } else {
      v = PyObject_GetItem(mapping, key);  // new reference
      if (!v) {
        for (PyObject* h : held) Py_DECREF(h);
        return nullptr;
      }
      held.push_back(v);
    }
    if (!PyArray_Check(v)) {
      bad = i;
      break;
    }
    PyArrayObject* a = reinterpret_cast<PyArrayObject*>(v);
    if (PyArray_TYPE(a) != NPY_DOUBLE || PyArray_NDIM(a) != 1 || PyArray_DIM(a, 0) != m ||
        (m > 1 && PyArray_STRIDE(a, 0) != (npy_intp)sizeof(double)) || !PyArray_ISALIGNED(a) ||
        PyArray_ISBYTESWAPPED(a)) {
      bad = i;
      break;
    }
    src[(size_t)i] = PyArray_BYTES(a);
  }
  if (bad < 0) {
    char* dst = PyArray_BYTES(out);
    const size_t row = (size_t)m * sizeof(double);
    if (nthreads < 1) nthreads = 1;
    if ((size_t)n * row < (1u << 20)) nthreads = 1;  // small tables: not worth the thread starts
    // a dict's values stay alive while we hold the GIL-free section only if nobody mutates the
    // dict meanwhile; the solver holds its own lock and the caller's mapping for the whole call
    Py_BEGIN_ALLOW_THREADS
    auto work = [&](Py_ssize_t i0, Py_ssize_t i1) {
      for (Py_ssize_t i = i0; i < i1; ++i) std::memcpy(dst + (size_t)i * row, src[(size_t)i], row);
    };
    if (nthreads == 1) {
      work(0, n);
    } else {
      std::vector<std::thread> th;
      for (int t = 1; t < nthreads; ++t) th.emplace_back(work, n * t / nthreads, n * (t + 1) / nthreads);
      work(0, n / nthreads);
      for (auto& x : th) x.join();
    }
    Py_END_ALLOW_THREADS
  }
  for (PyObject* h : held) Py_DECREF(h);
  return PyLong_FromSsize_t(bad);
}

PyMethodDef methods[] = {
    {"gather_rows", gather_rows, METH_VARARGS, "gather {id: (m,) float64} rows into a contiguous (n, m) table"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_hps_host", "host-side helpers of the HPS B200 drop-in API", -1, methods,
                      nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__hps_host(void) {
  import_array();
  return PyModule_Create(&moddef);
}
