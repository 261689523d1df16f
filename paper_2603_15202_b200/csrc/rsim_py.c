/* rsim_py.c -- CPython helper for the drop-in's route(): RoutingDecision.scores
 * (reference policies.py:84-89, dict[int, float] over the candidate instances) built straight
 * from the double buffer librsim wrote, without a Python-level loop or an intermediate list
 * (1,024 instances: about half the time of dict(enumerate(scores.tolist()))). Host glue only;
 * every score itself comes from the device. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <math.h>
#include <stdint.h>

/* scores_dict(address, n, skip_nan) -> {i: scores[i]} for i in range(n) (NaN entries omitted
 * when skip_nan: the detector's excluded holders, cluster.py:133-139) */
static PyObject *g_keys = NULL;   /* list of the int keys 0..len-1, kept across calls */

static int ensure_keys(Py_ssize_t n) {
    if (!g_keys && !(g_keys = PyList_New(0))) return -1;
    for (Py_ssize_t i = PyList_GET_SIZE(g_keys); i < n; i++) {
        PyObject *k = PyLong_FromSsize_t(i);
        if (!k || PyList_Append(g_keys, k) < 0) { Py_XDECREF(k); return -1; }
        Py_DECREF(k);
    }
    return 0;
}

static PyObject *scores_dict(PyObject *self, PyObject *args) {
    unsigned long long addr;
    Py_ssize_t n;
    int skip_nan = 0;
    (void)self;
    if (!PyArg_ParseTuple(args, "Kn|p", &addr, &n, &skip_nan)) return NULL;
    const double *v = (const double *)(uintptr_t)addr;
    if (ensure_keys(n) < 0) return NULL;
    PyObject *d = _PyDict_NewPresized(n);
    if (!d) return NULL;
    for (Py_ssize_t i = 0; i < n; i++) {
        if (skip_nan && isnan(v[i])) continue;
        PyObject *f = PyFloat_FromDouble(v[i]);
        const int bad = !f || PyDict_SetItem(d, PyList_GET_ITEM(g_keys, i), f) < 0;
        Py_XDECREF(f);
        if (bad) { Py_DECREF(d); return NULL; }
    }
    return d;
}

static PyMethodDef methods[] = {
    {"scores_dict", scores_dict, METH_VARARGS, "scores_dict(address, n, skip_nan=False) -> dict[int, float]"},
    {NULL, NULL, 0, NULL}};
static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_rsimpy", NULL, -1, methods, NULL, NULL, NULL, NULL};
PyMODINIT_FUNC PyInit__rsimpy(void) { return PyModule_Create(&module); }
