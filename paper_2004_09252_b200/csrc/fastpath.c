/* fastpath.c -- CPython entry points for the fault-sized calls.
 *
 * The fault handler (pkg/src/pagecrypt/orchestrator.py:193-200,230-239)
 * crypts 1-2 pages per call, so a call's fixed cost matters as much as the
 * GPU's: a ctypes call with a dozen converted arguments costs ~1.5 us on the
 * B200 host, these METH_FASTCALL wrappers ~0.1 us.  They call straight into
 * libpagecrypt.so (include/pagecrypt.h) with the GIL released and return the
 * library's status code; the Python layer maps a non-zero code to the
 * reference exceptions (_native.check).  Plain integers only -- handles and
 * addresses the Python layer has already validated.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#include "../../include/pagecrypt.h"

static int as_u64(PyObject *o, uint64_t *v) {
  *v = PyLong_AsUnsignedLongLong(o);
  return !(*v == (uint64_t)-1 && PyErr_Occurred());
}

/* crypt_host(engine, key, vaddr0, pid0, src, dst, n, rounds) -> int
 * pc_crypt_pages_host with contiguous vaddrs and a scalar pid. */
static PyObject *crypt_host(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[8];
  if (nargs != 8) {
    PyErr_SetString(PyExc_TypeError, "crypt_host takes 8 integer arguments");
    return NULL;
  }
  for (int i = 0; i < 8; ++i)
    if (!as_u64(args[i], &a[i])) return NULL;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = pc_crypt_pages_host((pc_engine *)(uintptr_t)a[0], (const pc_key *)(uintptr_t)a[1], NULL, NULL, NULL, a[2],
                           (uint32_t)a[3], (const void *)(uintptr_t)a[4], (void *)(uintptr_t)a[5], (size_t)a[6],
                           (int)a[7]);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

/* crypt_host_buf(engine, key, vaddr0, pid0, src, dst, rounds) -> int
 * As crypt_host over two buffer-protocol objects (numpy arrays, bytearray,
 * memoryview, bytes as src): C-contiguous, dst writable, equal sizes, whole
 * pages.  Returns -1 (no exception) when the buffers do not qualify, so the
 * caller's general path produces the reference error. */
static PyObject *crypt_host_buf(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[4], rounds;
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "crypt_host_buf takes 7 arguments");
    return NULL;
  }
  for (int i = 0; i < 4; ++i)
    if (!as_u64(args[i], &a[i])) return NULL;
  if (!as_u64(args[6], &rounds)) return NULL;
  Py_buffer in, out;
  if (PyObject_GetBuffer(args[4], &in, PyBUF_C_CONTIGUOUS) != 0) {
    PyErr_Clear();
    return PyLong_FromLong(-1);
  }
  if (PyObject_GetBuffer(args[5], &out, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) {
    PyErr_Clear();
    PyBuffer_Release(&in);
    return PyLong_FromLong(-1);
  }
  int rc = -1;
  if (in.len == out.len && in.len > 0 && (in.len % PC_PAGE_SIZE) == 0) {
    const size_t n = (size_t)in.len / PC_PAGE_SIZE;
    Py_BEGIN_ALLOW_THREADS
    rc = pc_crypt_pages_host((pc_engine *)(uintptr_t)a[0], (const pc_key *)(uintptr_t)a[1], NULL, NULL, NULL, a[2],
                             (uint32_t)a[3], in.buf, out.buf, n, (int)rounds);
    Py_END_ALLOW_THREADS
  }
  PyBuffer_Release(&out);
  PyBuffer_Release(&in);
  return PyLong_FromLong(rc);
}

/* service_crypt(service, worker, vaddr, pid, src, dst, timeout_us) -> int
 * pc_service_crypt: one page through the persistent worker service. */
static PyObject *service_crypt(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[6];
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "service_crypt takes 7 integer arguments");
    return NULL;
  }
  for (int i = 0; i < 6; ++i)
    if (!as_u64(args[i], &a[i])) return NULL;
  const long long timeout = PyLong_AsLongLong(args[6]);
  if (timeout == -1 && PyErr_Occurred()) return NULL;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = pc_service_crypt((pc_service *)(uintptr_t)a[0], (int)a[1], a[2], (uint32_t)a[3],
                        (const void *)(uintptr_t)a[4], (void *)(uintptr_t)a[5], (int64_t)timeout);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

/* service_crypt_buf(service, worker, vaddr, pid, page, timeout_us) -> int
 * pc_service_crypt in place on one writable 4096-byte buffer (a RamBuf's
 * bytearray, a numpy page); -1 without an exception when it does not
 * qualify (the caller's general path reports why). */
static PyObject *service_crypt_buf(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[4];
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "service_crypt_buf takes 6 arguments");
    return NULL;
  }
  for (int i = 0; i < 4; ++i)
    if (!as_u64(args[i], &a[i])) return NULL;
  const long long timeout = PyLong_AsLongLong(args[5]);
  if (timeout == -1 && PyErr_Occurred()) return NULL;
  Py_buffer pg;
  if (PyObject_GetBuffer(args[4], &pg, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) {
    PyErr_Clear();
    return PyLong_FromLong(-1);
  }
  int rc = -1;
  if (pg.len == PC_PAGE_SIZE) {
    Py_BEGIN_ALLOW_THREADS
    rc = pc_service_crypt((pc_service *)(uintptr_t)a[0], (int)a[1], a[2], (uint32_t)a[3], pg.buf, pg.buf,
                          (int64_t)timeout);
    Py_END_ALLOW_THREADS
  }
  PyBuffer_Release(&pg);
  return PyLong_FromLong(rc);
}

/* store_fault(store, client, pid, fault_vaddr, page_out, evict_vaddr, evict_page) -> (rc, hit)
 * pc_store_fault: refault one page and evict one in a single call. */
static PyObject *store_fault(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[7];
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "store_fault takes 7 integer arguments");
    return NULL;
  }
  for (int i = 0; i < 7; ++i)
    if (!as_u64(args[i], &a[i])) return NULL;
  int hit = 0, rc;
  Py_BEGIN_ALLOW_THREADS
  rc = pc_store_fault((pc_store *)(uintptr_t)a[0], a[1], (uint32_t)a[2], a[3], (void *)(uintptr_t)a[4], a[5],
                      (const void *)(uintptr_t)a[6], &hit);
  Py_END_ALLOW_THREADS
  return Py_BuildValue("(ii)", rc, hit);
}

/* store_fault_buf(store, cid, pid, vaddr, out, evict_vaddr, evict) -> (rc, hit) or None
 * pc_store_fault over buffer-protocol objects: out a writable C-contiguous
 * 4096-byte buffer, evict None or a C-contiguous 4096-byte buffer.  None
 * (no exception) when anything does not qualify -- a pid past u32, an
 * unaligned vaddr, a wrong buffer -- so the caller's general path reports
 * it with the reference's error. */
static PyObject *store_fault_buf(PyObject *self, PyObject *const *args, Py_ssize_t nargs) {
  (void)self;
  uint64_t a[4], ev;
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "store_fault_buf takes 7 arguments");
    return NULL;
  }
  for (int i = 0; i < 4; ++i)
    if (!as_u64(args[i], &a[i])) {
      PyErr_Clear();
      Py_RETURN_NONE;
    }
  if (!as_u64(args[5], &ev)) {
    PyErr_Clear();
    Py_RETURN_NONE;
  }
  if (a[2] > 0xffffffffull || (a[3] & 4095) || (ev & 4095)) Py_RETURN_NONE;
  Py_buffer out, in;
  if (PyObject_GetBuffer(args[4], &out, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) {
    PyErr_Clear();
    Py_RETURN_NONE;
  }
  const int have_in = args[6] != Py_None;
  if (have_in && PyObject_GetBuffer(args[6], &in, PyBUF_C_CONTIGUOUS) != 0) {
    PyErr_Clear();
    PyBuffer_Release(&out);
    Py_RETURN_NONE;
  }
  if (out.len != PC_PAGE_SIZE || (have_in && in.len != PC_PAGE_SIZE)) {
    if (have_in) PyBuffer_Release(&in);
    PyBuffer_Release(&out);
    Py_RETURN_NONE;
  }
  int hit = 0, rc;
  Py_BEGIN_ALLOW_THREADS
  rc = pc_store_fault((pc_store *)(uintptr_t)a[0], a[1], (uint32_t)a[2], a[3], out.buf, ev,
                      have_in ? in.buf : NULL, &hit);
  Py_END_ALLOW_THREADS
  if (have_in) PyBuffer_Release(&in);
  PyBuffer_Release(&out);
  return Py_BuildValue("(ii)", rc, hit);
}

static PyMethodDef methods[] = {
    {"crypt_host", (PyCFunction)(void (*)(void))crypt_host, METH_FASTCALL, "pc_crypt_pages_host, contiguous"},
    {"crypt_host_buf", (PyCFunction)(void (*)(void))crypt_host_buf, METH_FASTCALL, "crypt_host over buffers"},
    {"service_crypt", (PyCFunction)(void (*)(void))service_crypt, METH_FASTCALL, "pc_service_crypt"},
    {"service_crypt_buf", (PyCFunction)(void (*)(void))service_crypt_buf, METH_FASTCALL, "service_crypt in place"},
    {"store_fault", (PyCFunction)(void (*)(void))store_fault, METH_FASTCALL, "pc_store_fault"},
    {"store_fault_buf", (PyCFunction)(void (*)(void))store_fault_buf, METH_FASTCALL, "pc_store_fault on buffers"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pcfast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__pcfast(void) { return PyModule_Create(&module); }
