/* _dashhost: host-side batch gather for StreamState.update(UpdateBatch).
 *
 * The reference stages a batch by concatenating its per-slice row blocks
 * (/root/reference/pkg/src/p2stream/stream.py:286-298).  At the large shape a
 * batch is ~54,000 small numpy arrays (4.5 rows each on average); walking them
 * from Python -- validation, row counts, np.concatenate -- costs more than the
 * 0.8 GB copy itself.  This CPython extension does the walk in C through the
 * buffer protocol (no numpy headers, no per-array Python objects) and copies
 * with several threads while the GIL is released:
 *
 *   plan = scan(arrays, J, counts)      validate every block (2-D, J columns,
 *                                       C-contiguous float64), write its row count
 *                                       into `counts` (int64 buffer); returns a
 *                                       capsule, or the index of the first block that
 *                                       does not conform (the caller converts / reports)
 *   copy(plan, a, b, dst, row0, nthr[, f32])
 *                                       copy blocks [a, b) to dst rows row0.. (dst: a
 *                                       writable (N, J) buffer, e.g. pinned; float64,
 *                                       or float32 with f32 = 1: the FP32 data mode)
 *
 * It is host plumbing (like dash_host_row_ptr), not part of the device C ABI;
 * built in-tree by build.py with gcc.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    Py_ssize_t n;
    Py_ssize_t J;
    Py_buffer *views;   /* n exported buffers (kept until the capsule dies) */
    int64_t *rows;      /* rows per block */
    int64_t *offs;      /* row offset of each block (n + 1) */
} Plan;

static void plan_free(Plan *p) {
    if (!p) return;
    if (p->views) {
        for (Py_ssize_t i = 0; i < p->n; ++i)
            if (p->views[i].obj) PyBuffer_Release(&p->views[i]);
        free(p->views);
    }
    free(p->rows);
    free(p->offs);
    free(p);
}

static void capsule_destroy(PyObject *cap) { plan_free((Plan *)PyCapsule_GetPointer(cap, "dashhost.plan")); }

static int is_f64(const char *fmt) {
    if (!fmt) return 0;
    if (*fmt == '<' || *fmt == '=' || *fmt == '@') ++fmt;  /* native little-endian doubles */
    return fmt[0] == 'd' && fmt[1] == '\0';
}

static PyObject *dh_scan(PyObject *self, PyObject *args) {
    PyObject *seq;
    Py_ssize_t J;
    Py_buffer cb;
    if (!PyArg_ParseTuple(args, "Onw*", &seq, &J, &cb)) return NULL;
    PyObject *fast = PySequence_Fast(seq, "arrays must be a sequence");
    if (!fast) {
        PyBuffer_Release(&cb);
        return NULL;
    }
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
    if (cb.len < (Py_ssize_t)(n * sizeof(int64_t))) {
        Py_DECREF(fast);
        PyBuffer_Release(&cb);
        PyErr_SetString(PyExc_ValueError, "counts buffer too small");
        return NULL;
    }
    int64_t *counts = (int64_t *)cb.buf;
    Plan *p = (Plan *)calloc(1, sizeof(Plan));
    if (p) {
        p->n = n;
        p->J = J;
        p->views = (Py_buffer *)calloc((size_t)(n > 0 ? n : 1), sizeof(Py_buffer));
        p->rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
        p->offs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    }
    if (!p || !p->views || !p->rows || !p->offs) {
        plan_free(p);
        Py_DECREF(fast);
        PyBuffer_Release(&cb);
        return PyErr_NoMemory();
    }
    PyObject **items = PySequence_Fast_ITEMS(fast);
    int64_t acc = 0;
    Py_ssize_t bad = -1;
    for (Py_ssize_t i = 0; i < n; ++i) {
        Py_buffer *v = &p->views[i];
        if (PyObject_GetBuffer(items[i], v, PyBUF_STRIDES | PyBUF_FORMAT) != 0) {
            PyErr_Clear();
            v->obj = NULL;
            bad = i;
            break;
        }
        const int ok = v->ndim == 2 && v->itemsize == 8 && is_f64(v->format) && v->shape[1] == J &&
                       (v->shape[0] == 0 || (v->strides[1] == 8 && (v->shape[0] == 1 || v->strides[0] == 8 * J)));
        if (!ok) {
            bad = i;
            break;
        }
        p->rows[i] = (int64_t)v->shape[0];
        p->offs[i] = acc;
        counts[i] = p->rows[i];
        acc += p->rows[i];
    }
    Py_DECREF(fast);
    PyBuffer_Release(&cb);
    if (bad >= 0) {
        plan_free(p);
        return PyLong_FromSsize_t(bad);  /* an int: index of the first non-conforming block */
    }
    p->offs[n] = acc;
    PyObject *cap = PyCapsule_New(p, "dashhost.plan", capsule_destroy);
    if (!cap) plan_free(p);
    return cap;
}

typedef struct {
    const Plan *p;
    Py_ssize_t a, b;   /* blocks of this thread */
    char *dst;         /* dst row 0 of block `a0` of the call */
    int64_t base;      /* row offset of the call's first block */
    int f32;           /* destination holds floats (FP32 data mode): round while copying */
} Job;

static void *job_run(void *arg) {
    Job *j = (Job *)arg;
    const size_t J = (size_t)j->p->J;
    for (Py_ssize_t i = j->a; i < j->b; ++i) {
        const int64_t r = j->p->rows[i];
        if (r <= 0) continue;
        const size_t off = (size_t)(j->p->offs[i] - j->base) * J;
        if (!j->f32) {
            memcpy(j->dst + off * 8, j->p->views[i].buf, (size_t)r * J * 8);
        } else {
            const double *src = (const double *)j->p->views[i].buf;
            float *d = (float *)j->dst + off;
            for (size_t e = 0; e < (size_t)r * J; ++e) d[e] = (float)src[e];
        }
    }
    return NULL;
}

static PyObject *dh_copy(PyObject *self, PyObject *args) {
    PyObject *cap;
    Py_ssize_t a, b, row0;
    int nthr, f32 = 0;
    Py_buffer db;
    if (!PyArg_ParseTuple(args, "Onnw*ni|i", &cap, &a, &b, &db, &row0, &nthr, &f32)) return NULL;
    Plan *p = (Plan *)PyCapsule_GetPointer(cap, "dashhost.plan");
    if (!p) {
        PyBuffer_Release(&db);
        return NULL;
    }
    if (a < 0 || b > p->n || a > b || row0 < 0) {
        PyBuffer_Release(&db);
        PyErr_SetString(PyExc_ValueError, "block range out of bounds");
        return NULL;
    }
    const size_t rb = (size_t)p->J * (f32 ? 4 : 8);  /* destination row bytes */
    const int64_t rows = p->offs[b] - p->offs[a];
    if ((size_t)db.len < ((size_t)row0 + (size_t)rows) * rb) {
        PyBuffer_Release(&db);
        PyErr_SetString(PyExc_ValueError, "destination buffer too small");
        return NULL;
    }
    if (nthr < 1) nthr = 1;
    if (nthr > 32) nthr = 32;
    if (rows * (int64_t)rb < (1 << 22) || b - a < 2 * nthr) nthr = 1;
    Job jobs[32];
    pthread_t tid[32];
    /* split by rows: thread t takes the blocks whose first row lies in its share */
    Py_ssize_t cut = a;
    for (int t = 0; t < nthr; ++t) {
        const int64_t hi = p->offs[a] + rows * (t + 1) / nthr;
        Py_ssize_t e = cut;
        if (t == nthr - 1) {
            e = b;
        } else {
            Py_ssize_t lo_i = cut, hi_i = b;  /* first block with offs >= hi */
            while (lo_i < hi_i) {
                const Py_ssize_t mid = (lo_i + hi_i) / 2;
                if (p->offs[mid] < hi) lo_i = mid + 1;
                else hi_i = mid;
            }
            e = lo_i;
        }
        jobs[t].p = p;
        jobs[t].a = cut;
        jobs[t].b = e;
        jobs[t].dst = (char *)db.buf + (size_t)row0 * rb;
        jobs[t].base = p->offs[a];
        jobs[t].f32 = f32;
        cut = e;
    }
    Py_BEGIN_ALLOW_THREADS
    int started = 0;
    for (int t = 1; t < nthr; ++t) {
        if (pthread_create(&tid[t], NULL, job_run, &jobs[t]) != 0) break;
        started = t;
    }
    job_run(&jobs[0]);
    for (int t = started + 1; t < nthr; ++t) job_run(&jobs[t]);  /* threads that could not start */
    for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
    Py_END_ALLOW_THREADS
    PyBuffer_Release(&db);
    return PyLong_FromLongLong((long long)rows);
}

static PyMethodDef methods[] = {
    {"scan", dh_scan, METH_VARARGS, "scan(arrays, J, counts) -> plan capsule | index of the first bad block"},
    {"copy", dh_copy, METH_VARARGS, "copy(plan, a, b, dst, row0, nthreads) -> rows copied"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_dashhost", "host-side batch gather", -1, methods};

PyMODINIT_FUNC PyInit__dashhost(void) { return PyModule_Create(&moddef); }
