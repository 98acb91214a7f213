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
 *   pack(tasksets, compact=False) -> (blobs: bytes of int64, set_off: bytes, task_base:
 *                      bytes, scales: list[int], orders: list[tuple[TaskSpec]]
 *                      -- each set's task objects in blob order)
 *
 * A set whose values leave int64, or whose shape the engine does not take
 * (pack._check_shape), raises; the caller then packs that batch in Python
 * to get the same exception text.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <thread>
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
    if (d == 1 || (d > 0 && acc % d == 0)) return true; /* (denominator 1: nearly every value) */
    const int64_t g = gcd64(acc, d);
    if (g == 0) return fail("zero denominator");
    __int128 v = (__int128)(acc / g) * d;
    if (v < 0) v = -v;
    if (v > INT64_MAX) return fail("time scale exceeds int64");
    acc = (int64_t)v;
    return true;
}

/* one task's scalar fields; its segment values sit in the set's arena from
 * `off`: m (lo, hi) CPU pairs, p (lo, hi) memory pairs, g (work lo, work hi,
 * critical-path overhead, interleave ratio) GPU quads */
struct TaskF {
    PyObject *obj;
    int64_t prio;
    Frac D, T;
    int m, p, g, off;
};

/* per-call scratch, reused across the sets of a call */
struct Scratch {
    std::vector<TaskF> tf;
    std::vector<Frac> arena;
    std::vector<int> order;
    PyObject *hold = nullptr; /* the current set's task sequence (owns tf[].obj) */
    int compact = 0;          /* emit compact blobs where the values fit */
    ~Scratch() { Py_XDECREF(hold); }
};

bool seq_items(PyObject *o, PyObject *name, PyObject *&seq) {
    PyObject *x = PyObject_GetAttr(o, name);
    if (!x) return false;
    seq = PySequence_Fast(x, "expected a sequence");
    Py_DECREF(x);
    return seq != nullptr;
}

bool read_task(PyObject *t, TaskF &r, std::vector<Frac> &ar, int mem_model) {
    r.obj = t;
    r.off = (int)ar.size();
    PyObject *p = PyObject_GetAttr(t, s_priority);
    if (!p) return false;
    const bool okp = to_i64(p, r.prio);
    Py_DECREF(p);
    if (!okp || !attr_frac(t, s_deadline, r.D) || !attr_frac(t, s_period, r.T)) return false;
    PyObject *cpu, *mem, *gpu;
    if (!seq_items(t, s_cpu, cpu)) return false;
    const Py_ssize_t m = PySequence_Fast_GET_SIZE(cpu);
    bool ok = true;
    Frac lo, hi, ov, ra;
    for (Py_ssize_t j = 0; ok && j < m; j++) {
        ok = bounds(PySequence_Fast_GET_ITEM(cpu, j), lo, hi);
        ar.push_back(lo);
        ar.push_back(hi);
    }
    Py_DECREF(cpu);
    if (!ok || !seq_items(t, s_mem, mem)) return false;
    const Py_ssize_t pn = PySequence_Fast_GET_SIZE(mem);
    for (Py_ssize_t j = 0; ok && j < pn; j++) {
        ok = bounds(PySequence_Fast_GET_ITEM(mem, j), lo, hi);
        ar.push_back(lo);
        ar.push_back(hi);
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
        ok = bounds(w, lo, hi) && attr_frac(k, s_ovh, ov) && attr_frac(k, s_ratio, ra);
        Py_DECREF(w);
        ar.push_back(lo);
        ar.push_back(hi);
        ar.push_back(ov);
        ar.push_back(ra);
    }
    Py_DECREF(gpu);
    if (!ok) return false;
    /* pack._check_shape */
    if (m < 0 || m > 16) return fail("engine supports 0..16 CPU segments");
    if (g != (m > 0 ? m - 1 : 0)) return fail("gpu segment count != m - 1");
    const Py_ssize_t want = m < 2 ? 0 : (mem_model == 0 ? 2 * m - 2 : m - 1);
    if (pn != want) return fail("mem segment count mismatch");
    r.m = (int)m;
    r.p = (int)pn;
    r.g = (int)g;
    return true;
}

/* TaskSet.mem_model is an enum member (a singleton): its .value (a
 * Python-level property) is read once per distinct member */
PyObject *g_last_mm = nullptr;
int g_last_mm_code = 0;

/* the set at words[base..] in the compact form (int32 segment areas, header
 * word 7 = 1) when every segment value fits int32, as tests/blobtools.compact */
void compact_set(std::vector<int64_t> &words, size_t base) {
    int64_t *h = words.data() + base;
    const int64_t n = h[0], hb = 8 + 8 * n, W = (int64_t)(words.size() - base);
    for (int64_t j = hb; j < W; j++)
        if (h[j] < INT32_MIN || h[j] > INT32_MAX) return;
    const int64_t nseg = W - hb;
    std::vector<int32_t> seg(nseg + (nseg & 1), 0);
    for (int64_t j = 0; j < nseg; j++) seg[j] = (int32_t)h[hb + j];
    for (int64_t r = 0; r < n; r++) h[8 + 8 * r + 5] = 2 * hb + (h[8 + 8 * r + 5] - hb);
    const int64_t W2 = hb + (int64_t)seg.size() / 2;
    memcpy(h + hb, seg.data(), seg.size() * sizeof(int32_t));
    h[7] = 1;
    h[4] = W2;
    words.resize(base + (size_t)W2);
}

bool pack_one(PyObject *ts, Scratch &sc, std::vector<int64_t> &words, int64_t &scale) {
    PyObject *tasks_o = PyObject_GetAttr(ts, s_tasks);
    if (!tasks_o) return false;
    PyObject *tasks = PySequence_Fast(tasks_o, "tasks");
    Py_DECREF(tasks_o);
    if (!tasks) return false;
    Py_XSETREF(sc.hold, tasks); /* read errors below leave it to the Scratch */
    int mem_model = 0;
    int64_t sms = 0;
    {
        PyObject *mm = PyObject_GetAttr(ts, s_mem_model);
        if (!mm) return false;
        if (mm == g_last_mm) {
            mem_model = g_last_mm_code;
        } else {
            PyObject *v = PyObject_GetAttr(mm, s_value);
            if (!v) {
                Py_DECREF(mm);
                return false;
            }
            mem_model = PyUnicode_Check(v) && PyUnicode_CompareWithASCIIString(v, "two_copy") == 0 ? 0 : 1;
            Py_DECREF(v);
            Py_XDECREF(g_last_mm);
            Py_INCREF(mm);
            g_last_mm = mm;
            g_last_mm_code = mem_model;
        }
        Py_DECREF(mm);
        PyObject *pl = PyObject_GetAttr(ts, s_platform);
        PyObject *gn = pl ? PyObject_GetAttr(pl, s_sms) : nullptr;
        Py_XDECREF(pl);
        const bool ok = gn && to_i64(gn, sms);
        Py_XDECREF(gn);
        if (!ok) return false;
    }
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(tasks);
    if (n > 64) return fail("engine supports at most 64 tasks per set");
    std::vector<TaskF> &tf = sc.tf;
    std::vector<Frac> &ar = sc.arena;
    tf.resize(n);
    ar.clear();
    for (Py_ssize_t i = 0; i < n; i++)
        if (!read_task(PySequence_Fast_GET_ITEM(tasks, i), tf[i], ar, mem_model)) return false;
    /* time scale and interleave denominator */
    int64_t S = 1, A = 1;
    bool ok = true;
    for (const TaskF &t : tf) {
        ok = ok && lcm_into(S, t.D.d) && lcm_into(S, t.T.d);
        const Frac *f = ar.data() + t.off;
        const int nt = 2 * t.m + 2 * t.p;
        for (int j = 0; ok && j < nt; j++) ok = lcm_into(S, f[j].d);
        f += nt;
        for (int j = 0; ok && j < t.g; j++, f += 4)
            ok = lcm_into(S, f[0].d) && lcm_into(S, f[1].d) && lcm_into(S, f[2].d) && lcm_into(A, f[3].d);
    }
    if (!ok) return false;
    auto tick = [&](const Frac &x, int64_t &out) -> bool {
        __int128 v = (__int128)x.n * (x.d == 1 ? S : S / x.d);
        if (v > INT64_MAX || v < -INT64_MAX) return fail("task set values exceed int64 after scaling");
        out = (int64_t)v;
        return true;
    };
    std::vector<int> &order = sc.order;
    order.resize(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tf[a].prio < tf[b].prio; });
    const size_t base = words.size();
    int64_t maxm = 0, maxp = 0, nseg = 0;
    for (const TaskF &t : tf) {
        maxm = std::max<int64_t>(maxm, t.m);
        maxp = std::max<int64_t>(maxp, t.p);
        nseg += 2 * t.m + 2 * t.p + 4 * t.g;
    }
    words.resize(base + 8 + 8 * (size_t)n + (size_t)nseg);
    int64_t *hdr = words.data() + base;
    const int64_t h0[8] = {(int64_t)n, sms, (int64_t)mem_model, A, 8 + 8 * (int64_t)n + nseg, maxm, maxp, 0};
    std::copy(h0, h0 + 8, hdr);
    int64_t seg_off = 8 + 8 * (int64_t)n;
    for (Py_ssize_t r = 0; r < n; r++) {
        const TaskF &t = tf[order[r]];
        int64_t *rec = hdr + 8 + 8 * r;
        const int64_t m = t.m, p = t.p, g = t.g;
        int64_t D, T;
        if (!tick(t.D, D) || !tick(t.T, T)) return false;
        const int64_t vals[8] = {m, p, D, T, t.prio, seg_off, (int64_t)order[r], 0};
        std::copy(vals, vals + 8, rec);
        /* cl_lo[m] cl_hi[m] ml_lo[p] ml_hi[p] gw_lo[g] gw_hi[g] gl[g] ratio[g] */
        int64_t *o = hdr + seg_off;
        const Frac *f = ar.data() + t.off;
        for (int64_t j = 0; j < m; j++)
            if (!tick(f[2 * j], o[j]) || !tick(f[2 * j + 1], o[m + j])) return false;
        o += 2 * m;
        f += 2 * m;
        for (int64_t j = 0; j < p; j++)
            if (!tick(f[2 * j], o[j]) || !tick(f[2 * j + 1], o[p + j])) return false;
        o += 2 * p;
        f += 2 * p;
        for (int64_t j = 0; j < g; j++) {
            if (!tick(f[4 * j], o[j]) || !tick(f[4 * j + 1], o[g + j]) || !tick(f[4 * j + 2], o[2 * g + j]))
                return false;
            o[3 * g + j] = f[4 * j + 3].n * (f[4 * j + 3].d == A ? 1 : A / f[4 * j + 3].d);
        }
        seg_off += 2 * m + 2 * p + 4 * g;
    }
    scale = S;
    if (sc.compact) compact_set(words, base);
    return true;
}

PyObject *py_pack(PyObject *, PyObject *args) {
    PyObject *seq_o;
    int compact = 0;
    if (!PyArg_ParseTuple(args, "O|p", &seq_o, &compact)) return nullptr;
    PyObject *seq = PySequence_Fast(seq_o, "pack expects a sequence of TaskSets");
    if (!seq) return nullptr;
    const Py_ssize_t S = PySequence_Fast_GET_SIZE(seq);
    std::vector<int64_t> words, set_off{0}, task_base{0};
    words.reserve((size_t)S * 320);
    set_off.reserve((size_t)S + 1);
    task_base.reserve((size_t)S + 1);
    Scratch sc;
    sc.compact = compact;
    PyObject *scales = PyList_New(S), *orders = PyList_New(S);
    bool ok = scales && orders;
    for (Py_ssize_t s = 0; ok && s < S; s++) {
        int64_t scale = 1;
        ok = pack_one(PySequence_Fast_GET_ITEM(seq, s), sc, words, scale);
        if (!ok) break;
        set_off.push_back((int64_t)words.size());
        task_base.push_back(task_base.back() + (int64_t)sc.order.size());
        PyList_SET_ITEM(scales, s, PyLong_FromLongLong(scale));
        PyObject *o = PyTuple_New((Py_ssize_t)sc.order.size());
        for (size_t i = 0; i < sc.order.size(); i++) {
            PyObject *t = sc.tf[sc.order[i]].obj;
            Py_INCREF(t);
            PyTuple_SET_ITEM(o, i, t);
        }
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

/* ------------------------------------------------------------------
 * pack_arrays: S same-shape sets from int64 arrays (arrays.TaskArrays) in one
 * pass, threads over set ranges, the GIL released.  Same words as pack_one
 * on the equivalent TaskSets (tests/test_arrays.py).
 * ------------------------------------------------------------------ */
struct ArrIn {
    int64_t S, n, m, p, g, den, mem_model, compact, W;
    const int64_t *D, *T, *prio, *cl_lo, *cl_hi, *ml_lo, *ml_hi, *gw_lo, *gw_hi, *gl, *ra, *sms;
    int64_t *out, *order;
};

/* sets [s0, s1); false if a compact segment value leaves int32 */
bool pack_range(const ArrIn &a, int64_t s0, int64_t s1) {
    const int64_t n = a.n, m = a.m, p = a.p, g = a.g, per = 2 * m + 2 * p + 4 * g;
    const int64_t base = 8 + 8 * n;
    std::vector<int> ord(n);
    for (int64_t s = s0; s < s1; s++) {
        int64_t *o = a.out + s * a.W;
        const int64_t *pr = a.prio + s * n;
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return pr[x] < pr[y]; });
        /* A = den / gcd(den, every ratio numerator of the set) */
        int64_t G = a.den;
        const int64_t *ra = a.ra + s * n * g;
        for (int64_t j = 0; j < n * g && G > 1; j++) G = gcd64(G, ra[j]);
        if (G == 0) G = 1;
        const int64_t A = a.den / G;
        const int64_t h[8] = {n, a.sms[s], a.mem_model, A, a.W, m, p, a.compact};
        std::copy(h, h + 8, o);
        int32_t *o32 = (int32_t *)o;
        bool fits = true;
        auto put = [&](int64_t at, int64_t v) {
            if (a.compact) {
                fits = fits && v >= INT32_MIN && v <= INT32_MAX;
                o32[at] = (int32_t)v;
            } else {
                o[at] = v;
            }
        };
        if (a.compact && (n * per) % 2) o32[2 * base + n * per] = 0;
        for (int64_t r = 0; r < n; r++) {
            const int64_t i = ord[r], ti = s * n + i;
            a.order[s * n + r] = i;
            const int64_t so = (a.compact ? 2 * base : base) + r * per;
            const int64_t rec[8] = {m, p, a.D[ti], a.T[ti], pr[i], so, i, 0};
            std::copy(rec, rec + 8, o + 8 + 8 * r);
            int64_t at = so;
            for (int64_t j = 0; j < m; j++) put(at + j, a.cl_lo[ti * m + j]);
            at += m;
            for (int64_t j = 0; j < m; j++) put(at + j, a.cl_hi[ti * m + j]);
            at += m;
            for (int64_t j = 0; j < p; j++) put(at + j, a.ml_lo[ti * p + j]);
            at += p;
            for (int64_t j = 0; j < p; j++) put(at + j, a.ml_hi[ti * p + j]);
            at += p;
            for (int64_t j = 0; j < g; j++) put(at + j, a.gw_lo[ti * g + j]);
            at += g;
            for (int64_t j = 0; j < g; j++) put(at + j, a.gw_hi[ti * g + j]);
            at += g;
            for (int64_t j = 0; j < g; j++) put(at + j, a.gl[ti * g + j]);
            at += g;
            for (int64_t j = 0; j < g; j++) put(at + j, a.ra[ti * g + j] / G);
        }
        if (!fits) return false;
    }
    return true;
}

bool get_buf(PyObject *o, Py_buffer &b, int64_t want, bool writable, const char *name) {
    if (PyObject_GetBuffer(o, &b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT | (writable ? PyBUF_WRITABLE : 0)) != 0)
        return false;
    if (b.itemsize != 8 || !b.format || (b.format[0] != 'q' && b.format[0] != 'l') || b.len != want * 8) {
        PyBuffer_Release(&b);
        PyErr_Format(PyExc_ValueError, "%s: expected %lld contiguous int64 values", name, (long long)want);
        return false;
    }
    return true;
}

PyObject *py_pack_arrays(PyObject *, PyObject *args) {
    ArrIn a{};
    PyObject *obj[14];
    if (!PyArg_ParseTuple(args, "LLLLLLLLOOOOOOOOOOOOOO", &a.S, &a.n, &a.m, &a.p, &a.g, &a.den, &a.mem_model,
                          &a.compact, &obj[0], &obj[1], &obj[2], &obj[3], &obj[4], &obj[5], &obj[6], &obj[7],
                          &obj[8], &obj[9], &obj[10], &obj[11], &obj[12], &obj[13]))
        return nullptr;
    const int64_t S = a.S, n = a.n, per = 2 * a.m + 2 * a.p + 4 * a.g, base = 8 + 8 * n;
    a.W = base + (a.compact ? (n * per + 1) / 2 : n * per);
    const int64_t want[14] = {S * n, S * n, S * n, S * n * a.m, S * n * a.m, S * n * a.p, S * n * a.p,
                              S * n * a.g, S * n * a.g, S * n * a.g, S * n * a.g, S, S * a.W, S * n};
    const char *names[14] = {"deadline", "period", "priority", "cpu_lo", "cpu_hi", "mem_lo", "mem_hi",
                             "work_lo", "work_hi", "overhead", "ratio_num", "physical_sms", "out", "order"};
    Py_buffer b[14];
    int got = 0;
    bool ok = true;
    for (; got < 14 && ok; got++) ok = get_buf(obj[got], b[got], want[got], got >= 12, names[got]);
    if (!ok) got--;
    bool fits = true;
    if (ok) {
        const int64_t **in[12] = {&a.D, &a.T, &a.prio, &a.cl_lo, &a.cl_hi, &a.ml_lo, &a.ml_hi,
                                  &a.gw_lo, &a.gw_hi, &a.gl, &a.ra, &a.sms};
        for (int k = 0; k < 12; k++) *in[k] = (const int64_t *)b[k].buf;
        a.out = (int64_t *)b[12].buf;
        a.order = (int64_t *)b[13].buf;
        Py_BEGIN_ALLOW_THREADS
        const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
        const int64_t nt = std::min<int64_t>(std::min<int64_t>(hw, 32), std::max<int64_t>(1, S / 8192));
        std::vector<char> res(nt, 1);
        std::vector<std::thread> th;
        for (int64_t t = 1; t < nt; t++)
            th.emplace_back([&, t] { res[t] = pack_range(a, S * t / nt, S * (t + 1) / nt); });
        res[0] = pack_range(a, 0, S / nt);
        for (auto &x : th) x.join();
        for (char r : res) fits = fits && r;
        Py_END_ALLOW_THREADS
    }
    for (int k = 0; k < got; k++) PyBuffer_Release(&b[k]);
    if (!ok) return nullptr;
    if (!fits) {
        PyErr_SetString(PyExc_OverflowError, "segment values exceed int32: pack with compact=False");
        return nullptr;
    }
    return PyLong_FromLongLong(a.W);
}

PyMethodDef methods[] = {{"pack", py_pack, METH_VARARGS, "pack(tasksets) -> (blobs, set_off, task_base, scales, ordered task tuples)"},
                         {"pack_arrays", py_pack_arrays, METH_VARARGS,
                          "pack_arrays(S, n, m, p, g, ratio_den, mem_model, compact, deadline, period, priority, "
                          "cpu_lo, cpu_hi, mem_lo, mem_hi, work_lo, work_hi, overhead, ratio_num, physical_sms, "
                          "out, order) -> words per set"},
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
