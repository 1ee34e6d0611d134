/* pyfast.c — CPython binding of the per-update entry points of include/rgg_gpu.h.
 *
 * ctypes spends ~2 us per numpy pointer conversion (ndarray.ctypes), which is a
 * tenth of a c2 update's host-side budget; this module takes the arrays through
 * the buffer protocol instead.  engine.GpuEngine uses it for batch_update.
 * update(handle, ids, rt12, flags, reports) -> rc
 *   ids     int32 contiguous buffer (n), rt12 float64 contiguous buffer (n*12),
 *   reports writable buffer of n rgg_update_report, or None. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "../../include/rgg_gpu.h"

static PyObject* py_update(PyObject* self, PyObject* args) {
    (void)self;
    unsigned long long handle;
    PyObject *ids_o, *rt_o, *rep_o;
    int flags;
    if (!PyArg_ParseTuple(args, "KOOiO", &handle, &ids_o, &rt_o, &flags, &rep_o)) return NULL;
    Py_buffer ids, rt, rep;
    if (PyObject_GetBuffer(ids_o, &ids, PyBUF_C_CONTIGUOUS) < 0) return NULL;
    if (PyObject_GetBuffer(rt_o, &rt, PyBUF_C_CONTIGUOUS) < 0) {
        PyBuffer_Release(&ids);
        return NULL;
    }
    int have_rep = rep_o != Py_None;
    if (have_rep && PyObject_GetBuffer(rep_o, &rep, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) < 0) {
        PyBuffer_Release(&ids);
        PyBuffer_Release(&rt);
        return NULL;
    }
    const Py_ssize_t n = ids.len / (Py_ssize_t)sizeof(int32_t);
    int rc;
    if (rt.len != n * 12 * (Py_ssize_t)sizeof(double) ||
        (have_rep && rep.len < n * (Py_ssize_t)sizeof(rgg_update_report))) {
        rc = -1;
    } else {
        Py_BEGIN_ALLOW_THREADS
        rc = rgg_gpu_update((rgg_gpu*)(uintptr_t)handle, (const int32_t*)ids.buf, (const double*)rt.buf, (int32_t)n,
                            flags, have_rep ? (rgg_update_report*)rep.buf : NULL);
        Py_END_ALLOW_THREADS
    }
    PyBuffer_Release(&ids);
    PyBuffer_Release(&rt);
    if (have_rep) PyBuffer_Release(&rep);
    if (rc == -1) {
        PyErr_SetString(PyExc_ValueError, "ids (int32 n), rt12 (float64 n x 12) and reports (n) sizes disagree");
        return NULL;
    }
    return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {{"update", py_update, METH_VARARGS, "rgg_gpu_update over buffers"},
                                {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_rggfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__rggfast(void) { return PyModule_Create(&module); }
