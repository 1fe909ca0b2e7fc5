/* evconv.c — the Trace -> columns conversion of the drop-in object API
 * (paper_1903_06631_b200/trace.py:_events_to_arrays) in one C pass over the
 * event list: per event the five attributes the reference's TraceEvent
 * carries (trace.py:24-31: index, t_us, kind, var, size) go straight into
 * the caller's numpy columns, and each name is interned on first sight
 * (first[i] = position of the first event naming it, as the Python path's
 * dict.setdefault does).
 *
 * Anything outside the plain form — a kind missing from the code table, a
 * non-int index/time/size, a non-str name, an int beyond int64 — makes it
 * return None with no exception set: the Python path then converts the
 * whole list and raises exactly what it raises.  Host glue for the object
 * API, not a compute path. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

static int get_i64(PyObject *o, int64_t *out) {
  if (!PyLong_Check(o)) return -1;
  int overflow = 0;
  long long v = PyLong_AsLongLongAndOverflow(o, &overflow);
  if (overflow || (v == -1 && PyErr_Occurred())) {
    PyErr_Clear();
    return -1;
  }
  *out = (int64_t)v;
  return 0;
}

/* one event into row i; 1 on success, 0 when it is outside the plain form */
static int convert_one(PyObject *ev, Py_ssize_t i, PyObject *code, PyObject *ids, uint8_t *kind, int64_t *size,
                       int64_t *t_us, int64_t *index, int64_t *first, PyObject *a_index, PyObject *a_t,
                       PyObject *a_kind, PyObject *a_var, PyObject *a_size) {
  PyObject *o;
  int64_t v;
  /* index, t_us, size */
  o = PyObject_GetAttr(ev, a_index);
  if (!o || get_i64(o, &v)) { Py_XDECREF(o); return 0; }
  Py_DECREF(o);
  index[i] = v;
  o = PyObject_GetAttr(ev, a_t);
  if (!o || get_i64(o, &v)) { Py_XDECREF(o); return 0; }
  Py_DECREF(o);
  t_us[i] = v;
  o = PyObject_GetAttr(ev, a_size);
  if (!o || get_i64(o, &v)) { Py_XDECREF(o); return 0; }
  Py_DECREF(o);
  size[i] = v;
  /* kind through the code table */
  o = PyObject_GetAttr(ev, a_kind);
  if (!o) return 0;
  PyObject *c = PyDict_GetItemWithError(code, o);
  Py_DECREF(o);
  if (!c || get_i64(c, &v) || v < 0 || v > 255) return 0;
  kind[i] = (uint8_t)v;
  /* name: first position that named it */
  o = PyObject_GetAttr(ev, a_var);
  if (!o || !PyUnicode_Check(o)) { Py_XDECREF(o); return 0; }
  PyObject *pos = PyDict_GetItemWithError(ids, o);
  if (pos) {
    if (get_i64(pos, &v)) { Py_DECREF(o); return 0; }
    first[i] = v;
  } else {
    PyObject *pi = PyErr_Occurred() ? NULL : PyLong_FromSsize_t(i);
    if (!pi || PyDict_SetItem(ids, o, pi) < 0) { Py_XDECREF(pi); Py_DECREF(o); return 0; }
    Py_DECREF(pi);
    first[i] = (int64_t)i;
  }
  Py_DECREF(o);
  return 1;
}

/* columns(events, kind_code, ids, kind_u8, size_i64, t_us_i64, index_i64, first_i64) -> True | None */
static PyObject *columns(PyObject *self, PyObject *args) {
  (void)self;
  PyObject *events, *code, *ids, *bufs[5];
  if (!PyArg_ParseTuple(args, "O!O!O!OOOOO", &PyList_Type, &events, &PyDict_Type, &code, &PyDict_Type, &ids,
                        &bufs[0], &bufs[1], &bufs[2], &bufs[3], &bufs[4]))
    return NULL;
  const Py_ssize_t n = PyList_GET_SIZE(events);
  Py_buffer view[5];
  const Py_ssize_t isz[5] = {1, 8, 8, 8, 8};
  int got = 0;
  for (; got < 5; got++) {
    if (PyObject_GetBuffer(bufs[got], &view[got], PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) < 0) goto fail_release;
    if (view[got].len != n * isz[got]) {
      PyBuffer_Release(&view[got]);
      PyErr_SetString(PyExc_ValueError, "column length does not match the event count");
      goto fail_release;
    }
  }
  {
    uint8_t *kind = (uint8_t *)view[0].buf;
    int64_t *size = (int64_t *)view[1].buf, *t_us = (int64_t *)view[2].buf;
    int64_t *index = (int64_t *)view[3].buf, *first = (int64_t *)view[4].buf;
    PyObject *a_index = PyUnicode_InternFromString("index"), *a_t = PyUnicode_InternFromString("t_us");
    PyObject *a_kind = PyUnicode_InternFromString("kind"), *a_var = PyUnicode_InternFromString("var");
    PyObject *a_size = PyUnicode_InternFromString("size");
    int ok = a_index && a_t && a_kind && a_var && a_size;
    for (Py_ssize_t i = 0; ok && i < n; i++) {
      /* an attribute getter may run Python code: re-check the list and hold the event */
      if (PyList_GET_SIZE(events) != n) { ok = 0; break; }
      PyObject *ev = PyList_GET_ITEM(events, i);
      Py_INCREF(ev);
      ok = convert_one(ev, i, code, ids, kind, size, t_us, index, first, a_index, a_t, a_kind, a_var, a_size);
      Py_DECREF(ev);
    }
    Py_XDECREF(a_index); Py_XDECREF(a_t); Py_XDECREF(a_kind); Py_XDECREF(a_var); Py_XDECREF(a_size);
    for (int k = 0; k < 5; k++) PyBuffer_Release(&view[k]);
    if (!ok) {
      PyErr_Clear();
      Py_RETURN_NONE;  /* the Python path converts (and raises) */
    }
    Py_RETURN_TRUE;
  }
fail_release:
  for (int k = 0; k < got; k++) PyBuffer_Release(&view[k]);
  return NULL;
}

static PyMethodDef methods[] = {
    {"columns", columns, METH_VARARGS, "Fill trace columns from a list of event objects."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_evconv", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__evconv(void) { return PyModule_Create(&mod); }
