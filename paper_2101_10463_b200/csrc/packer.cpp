/*
 * packer.cpp -- native packing of TaskSet objects into the engine's blob
 * layout (include/rtgpu.h), as the CPython extension module
 * paper_2101_10463_b200._packer.  Same words as pack.py's pack_set (the
 * tests compare them): per set one time scale S = lcm of every duration's
 * denominator and one interleave denominator A = lcm of the ratios'
 * denominators, tasks in TaskSet.by_priority() order (a stable sort on the
 * priority, reference model.py:107).  Reads the objects by duck typing --
 * the reference's gpusched types and this package's alike: Fraction
 * numerators / denominators (or ints), ExecBounds.lo / .hi,
 * GpuKernelModel.work / .critical_path_overhead / .interleave_ratio.
 *
 *   pack(tasksets) -> (blobs: bytes of int64, set_off: bytes, task_base:
 *                      bytes, scales: list[int], orders: list[tuple[int]])
 *
 * A set whose values leave int64, or whose shape the engine does not take
 * (pack._check_shape), raises; the caller then packs that batch in Python
 * to get the same exception text.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

namespace {

PyObject *s_num, *s_den, *s_lo, *s_hi, *s_tasks, *s_mem_model, *s_platform, *s_sms, *s_cpu, *s_mem, *s_gpu,
    *s_deadline, *s_period, *s_priority, *s_work, *s_ovh, *s_ratio, *s_value;

struct Frac {
    int64_t n, d;
};

/* fractions.Fraction keeps its value in the __slots__ _numerator /
 * _denominator: read them at their offsets instead of through the
 * numerator / denominator properties */
PyTypeObject *g_fraction = nullptr;
Py_ssize_t g_off_num = -1, g_off_den = -1;

void init_fraction_slots() {
    PyObject *mod = PyImport_ImportModule("fractions");
    if (!mod) {
        PyErr_Clear();
        return;
    }
    PyObject *F = PyObject_GetAttrString(mod, "Fraction");
    Py_DECREF(mod);
    if (!F || !PyType_Check(F)) {
        PyErr_Clear();
        Py_XDECREF(F);
        return;
    }
    PyObject *dn = PyObject_GetAttrString(F, "_numerator");
    PyObject *dd = PyObject_GetAttrString(F, "_denominator");
    if (dn && dd && Py_IS_TYPE(dn, &PyMemberDescr_Type) && Py_IS_TYPE(dd, &PyMemberDescr_Type)) {
        PyMemberDef *mn = ((PyMemberDescrObject *)dn)->d_member, *md = ((PyMemberDescrObject *)dd)->d_member;
        if (mn->type == T_OBJECT_EX && md->type == T_OBJECT_EX) {
            g_fraction = (PyTypeObject *)F;
            g_off_num = mn->offset;
            g_off_den = md->offset;
        }
    }
    PyErr_Clear();
    Py_XDECREF(dn);
    Py_XDECREF(dd);
}

bool fail(const char *msg) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, msg);
    return false;
}

bool to_i64(PyObject *o, int64_t &v) {
    int ovf = 0;
    v = PyLong_AsLongLongAndOverflow(o, &ovf);
    if (ovf) return fail("value exceeds int64");
    return !(v == -1 && PyErr_Occurred());
}

/* numerator / denominator of an int or a Fraction-like object */
bool frac(PyObject *x, Frac &f) {
    if (g_fraction && Py_IS_TYPE(x, g_fraction)) {
        PyObject *n = *(PyObject **)((char *)x + g_off_num), *d = *(PyObject **)((char *)x + g_off_den);
        if (n && d) return to_i64(n, f.n) && to_i64(d, f.d);
    }
    if (PyLong_Check(x)) {
        f.d = 1;
        return to_i64(x, f.n);
    }
    PyObject *n = PyObject_GetAttr(x, s_num);
    if (!n) return false;
    PyObject *d = PyObject_GetAttr(x, s_den);
    if (!d) {
        Py_DECREF(n);
        return false;
    }
    const bool ok = to_i64(n, f.n) && to_i64(d, f.d);
    Py_DECREF(n);
    Py_DECREF(d);
    return ok;
}

bool attr_frac(PyObject *o, PyObject *name, Frac &f) {
    PyObject *x = PyObject_GetAttr(o, name);
    if (!x) return false;
    const bool ok = frac(x, f);
    Py_DECREF(x);
    return ok;
}

bool bounds(PyObject *b, Frac &lo, Frac &hi) { return attr_frac(b, s_lo, lo) && attr_frac(b, s_hi, hi); }

int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

bool lcm_into(int64_t &acc, int64_t d) {
    const int64_t g = gcd64(acc, d);
    __int128 v = (__int128)(acc / g) * d;
    if (v > INT64_MAX) return fail("time scale exceeds int64");
    acc = (int64_t)v;
    return true;
}

/* one task's fields */
struct TaskF {
    PyObject *obj;
    int64_t prio;
    Frac D, T, ovh_dummy;
    std::vector<Frac> cl_lo, cl_hi, ml_lo, ml_hi, gw_lo, gw_hi, gl, ratio;
};

bool seq_items(PyObject *o, PyObject *name, PyObject *&seq) {
    PyObject *x = PyObject_GetAttr(o, name);
    if (!x) return false;
    seq = PySequence_Fast(x, "expected a sequence");
    Py_DECREF(x);
    return seq != nullptr;
}

bool read_task(PyObject *t, TaskF &r, int mem_model) {
    r.obj = t;
    PyObject *p = PyObject_GetAttr(t, s_priority);
    if (!p) return false;
    const bool okp = to_i64(p, r.prio);
    Py_DECREF(p);
    if (!okp || !attr_frac(t, s_deadline, r.D) || !attr_frac(t, s_period, r.T)) return false;
    PyObject *cpu, *mem, *gpu;
    if (!seq_items(t, s_cpu, cpu)) return false;
    const Py_ssize_t m = PySequence_Fast_GET_SIZE(cpu);
    bool ok = true;
    for (Py_ssize_t j = 0; ok && j < m; j++) {
        Frac lo, hi;
        ok = bounds(PySequence_Fast_GET_ITEM(cpu, j), lo, hi);
        r.cl_lo.push_back(lo);
        r.cl_hi.push_back(hi);
    }
    Py_DECREF(cpu);
    if (!ok || !seq_items(t, s_mem, mem)) return false;
    const Py_ssize_t pn = PySequence_Fast_GET_SIZE(mem);
    for (Py_ssize_t j = 0; ok && j < pn; j++) {
        Frac lo, hi;
        ok = bounds(PySequence_Fast_GET_ITEM(mem, j), lo, hi);
        r.ml_lo.push_back(lo);
        r.ml_hi.push_back(hi);
    }
    Py_DECREF(mem);
    if (!ok || !seq_items(t, s_gpu, gpu)) return false;
    const Py_ssize_t g = PySequence_Fast_GET_SIZE(gpu);
    for (Py_ssize_t j = 0; ok && j < g; j++) {
        PyObject *k = PySequence_Fast_GET_ITEM(gpu, j);
        PyObject *w = PyObject_GetAttr(k, s_work);
        if (!w) {
            ok = false;
            break;
        }
        Frac lo, hi, ov, ra;
        ok = bounds(w, lo, hi) && attr_frac(k, s_ovh, ov) && attr_frac(k, s_ratio, ra);
        Py_DECREF(w);
        r.gw_lo.push_back(lo);
        r.gw_hi.push_back(hi);
        r.gl.push_back(ov);
        r.ratio.push_back(ra);
    }
    Py_DECREF(gpu);
    if (!ok) return false;
    /* pack._check_shape */
    if (m < 0 || m > 16) return fail("engine supports 0..16 CPU segments");
    if (g != (m > 0 ? m - 1 : 0)) return fail("gpu segment count != m - 1");
    const Py_ssize_t want = m < 2 ? 0 : (mem_model == 0 ? 2 * m - 2 : m - 1);
    if (pn != want) return fail("mem segment count mismatch");
    return true;
}

bool pack_one(PyObject *ts, std::vector<int64_t> &words, int64_t &scale, std::vector<int> &order) {
    PyObject *tasks_o = PyObject_GetAttr(ts, s_tasks);
    if (!tasks_o) return false;
    PyObject *tasks = PySequence_Fast(tasks_o, "tasks");
    Py_DECREF(tasks_o);
    if (!tasks) return false;
    int mem_model = 0;
    int64_t sms = 0;
    {
        PyObject *mm = PyObject_GetAttr(ts, s_mem_model);
        PyObject *v = mm ? PyObject_GetAttr(mm, s_value) : nullptr;
        Py_XDECREF(mm);
        if (!v) {
            Py_DECREF(tasks);
            return false;
        }
        mem_model = PyUnicode_CompareWithASCIIString(v, "two_copy") == 0 ? 0 : 1;
        Py_DECREF(v);
        PyObject *pl = PyObject_GetAttr(ts, s_platform);
        PyObject *gn = pl ? PyObject_GetAttr(pl, s_sms) : nullptr;
        Py_XDECREF(pl);
        const bool ok = gn && to_i64(gn, sms);
        Py_XDECREF(gn);
        if (!ok) {
            Py_DECREF(tasks);
            return false;
        }
    }
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(tasks);
    if (n > 64) {
        Py_DECREF(tasks);
        return fail("engine supports at most 64 tasks per set");
    }
    std::vector<TaskF> tf(n);
    for (Py_ssize_t i = 0; i < n; i++)
        if (!read_task(PySequence_Fast_GET_ITEM(tasks, i), tf[i], mem_model)) {
            Py_DECREF(tasks);
            return false;
        }
    Py_DECREF(tasks);
    /* time scale and interleave denominator */
    int64_t S = 1, A = 1;
    bool ok = true;
    for (const TaskF &t : tf) {
        ok = ok && lcm_into(S, t.D.d) && lcm_into(S, t.T.d);
        for (size_t j = 0; ok && j < t.cl_lo.size(); j++) ok = lcm_into(S, t.cl_lo[j].d) && lcm_into(S, t.cl_hi[j].d);
        for (size_t j = 0; ok && j < t.ml_lo.size(); j++) ok = lcm_into(S, t.ml_lo[j].d) && lcm_into(S, t.ml_hi[j].d);
        for (size_t j = 0; ok && j < t.gw_lo.size(); j++)
            ok = lcm_into(S, t.gw_lo[j].d) && lcm_into(S, t.gw_hi[j].d) && lcm_into(S, t.gl[j].d) &&
                 lcm_into(A, t.ratio[j].d);
    }
    if (!ok) return false;
    auto tick = [&](const Frac &x, int64_t &out) -> bool {
        __int128 v = (__int128)x.n * (S / x.d);
        if (v > INT64_MAX || v < -INT64_MAX) return fail("task set values exceed int64 after scaling");
        out = (int64_t)v;
        return true;
    };
    order.resize(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tf[a].prio < tf[b].prio; });
    const size_t base = words.size();
    int64_t maxm = 0, maxp = 0;
    for (const TaskF &t : tf) {
        maxm = std::max<int64_t>(maxm, (int64_t)t.cl_lo.size());
        maxp = std::max<int64_t>(maxp, (int64_t)t.ml_lo.size());
    }
    words.insert(words.end(), {(int64_t)n, sms, (int64_t)mem_model, A, 0, maxm, maxp, 0});
    const size_t rec0 = words.size();
    words.resize(rec0 + 8 * (size_t)n);
    int64_t seg_off = 8 + 8 * (int64_t)n;
    for (Py_ssize_t r = 0; r < n; r++) {
        const TaskF &t = tf[order[r]];
        int64_t *rec = &words[rec0 + 8 * r];
        const int64_t m = (int64_t)t.cl_lo.size(), p = (int64_t)t.ml_lo.size();
        int64_t D, T;
        if (!tick(t.D, D) || !tick(t.T, T)) return false;
        int64_t vals[8] = {m, p, D, T, t.prio, seg_off, (int64_t)order[r], 0};
        std::copy(vals, vals + 8, rec);
        auto put = [&](const std::vector<Frac> &v) -> bool {
            for (const Frac &x : v) {
                int64_t w;
                if (!tick(x, w)) return false;
                words.push_back(w);
            }
            return true;
        };
        if (!put(t.cl_lo) || !put(t.cl_hi) || !put(t.ml_lo) || !put(t.ml_hi) || !put(t.gw_lo) || !put(t.gw_hi) ||
            !put(t.gl))
            return false;
        for (const Frac &ra : t.ratio) words.push_back(ra.n * (A / ra.d));
        seg_off += 2 * m + 2 * p + 4 * (m > 0 ? m - 1 : 0);
    }
    words[base + 4] = (int64_t)(words.size() - base);
    scale = S;
    return true;
}

PyObject *py_pack(PyObject *, PyObject *args) {
    PyObject *seq_o;
    if (!PyArg_ParseTuple(args, "O", &seq_o)) return nullptr;
    PyObject *seq = PySequence_Fast(seq_o, "pack expects a sequence of TaskSets");
    if (!seq) return nullptr;
    const Py_ssize_t S = PySequence_Fast_GET_SIZE(seq);
    std::vector<int64_t> words, set_off{0}, task_base{0};
    PyObject *scales = PyList_New(S), *orders = PyList_New(S);
    bool ok = scales && orders;
    for (Py_ssize_t s = 0; ok && s < S; s++) {
        int64_t scale = 1;
        std::vector<int> order;
        ok = pack_one(PySequence_Fast_GET_ITEM(seq, s), words, scale, order);
        if (!ok) break;
        set_off.push_back((int64_t)words.size());
        task_base.push_back(task_base.back() + (int64_t)order.size());
        PyList_SET_ITEM(scales, s, PyLong_FromLongLong(scale));
        PyObject *o = PyTuple_New((Py_ssize_t)order.size());
        for (size_t i = 0; i < order.size(); i++) PyTuple_SET_ITEM(o, i, PyLong_FromLong(order[i]));
        PyList_SET_ITEM(orders, s, o);
    }
    Py_DECREF(seq);
    if (!ok) {
        Py_XDECREF(scales);
        Py_XDECREF(orders);
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "cannot pack task set");
        return nullptr;
    }
    PyObject *b = PyBytes_FromStringAndSize((const char *)words.data(), (Py_ssize_t)(words.size() * 8));
    PyObject *so = PyBytes_FromStringAndSize((const char *)set_off.data(), (Py_ssize_t)(set_off.size() * 8));
    PyObject *tb = PyBytes_FromStringAndSize((const char *)task_base.data(), (Py_ssize_t)(task_base.size() * 8));
    return Py_BuildValue("(NNNNN)", b, so, tb, scales, orders);
}

PyMethodDef methods[] = {{"pack", py_pack, METH_VARARGS, "pack(tasksets) -> (blobs, set_off, task_base, scales, orders)"},
                         {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_packer", "native TaskSet packer", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__packer(void) {
    s_num = PyUnicode_InternFromString("numerator");
    s_den = PyUnicode_InternFromString("denominator");
    s_lo = PyUnicode_InternFromString("lo");
    s_hi = PyUnicode_InternFromString("hi");
    s_tasks = PyUnicode_InternFromString("tasks");
    s_mem_model = PyUnicode_InternFromString("mem_model");
    s_platform = PyUnicode_InternFromString("platform");
    s_sms = PyUnicode_InternFromString("physical_sms");
    s_cpu = PyUnicode_InternFromString("cpu_segments");
    s_mem = PyUnicode_InternFromString("mem_segments");
    s_gpu = PyUnicode_InternFromString("gpu_segments");
    s_deadline = PyUnicode_InternFromString("deadline");
    s_period = PyUnicode_InternFromString("period");
    s_priority = PyUnicode_InternFromString("priority");
    s_work = PyUnicode_InternFromString("work");
    s_ovh = PyUnicode_InternFromString("critical_path_overhead");
    s_ratio = PyUnicode_InternFromString("interleave_ratio");
    s_value = PyUnicode_InternFromString("value");
    init_fraction_slots();
    return PyModule_Create(&module);
}
