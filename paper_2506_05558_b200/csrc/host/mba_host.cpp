// mba_host.cpp -- native host side of the batched mini-BA (CPython extension
// `paper_2506_05558_b200._mba_host`).
//
// The reference's producers hand the solver a list of independent BaProblem
// objects (miniba.py:65-83: R (n,3,3), t (n,3), focal/cx/cy, points (P,3),
// cam_idx/pt_idx (K,), uv (K,2), fixed_cams (n,), optimize_* flags) and
// lm_solve mutates each one in place (miniba.py:264-270, 288). Walking tens of
// thousands of such objects and copying their arrays is host work that must
// not bound the end-to-end rate, so it is done here in C++:
//
//  * Batch(problems): one pass over the list with the GIL held -- attribute
//    lookup, shape / dtype / length checks (the reference's error behaviour:
//    ValueError for an empty problem or inconsistent lengths), and buffer
//    views that keep every array alive and locked for the batch's lifetime.
//  * gather(lo, hi, ...): copies problems [lo, hi) into the chunk's upload
//    buffer (pinned host memory owned by the caller) in the device upload
//    layout -- int64 indices narrowed to int32, uv rounded to float32 with a
//    note whether any value is not fp32-representable (gather_lo then writes
//    the low-order float32 residual stream for that chunk), per-point track
//    statistics for the solver's plan -- on worker threads, GIL released.
//  * scatter(lo, hi, ...): writes the solved R, t, points back into the
//    callers' arrays in place (threads, GIL released) and rebinds focal.
//
// The point-major sort and the 16-byte record packing run on the device
// (mba_pack_obs, csrc/mba_pack.cu); nothing here touches a GPU.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_20_API_VERSION
#define PY_ARRAY_UNIQUE_SYMBOL mba_host_ARRAY_API
#include <numpy/arrayobject.h>

#include <algorithm>
#include <initializer_list>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

struct Prob {
  const double* R = nullptr;
  const double* t = nullptr;
  const double* X = nullptr;
  const double* uv = nullptr;
  const void* cam = nullptr;
  const void* pt = nullptr;
  const void* fixed = nullptr;
  double* Rw = nullptr;   // writable views (null: rebind through Python)
  double* tw = nullptr;
  double* Xw = nullptr;
  int cam_sz = 8, pt_sz = 8, fixed_sz = 1;
  int64_t n = 0, P = 0, K = 0;
  double focal = 0, cx = 0, cy = 0;
  uint8_t flags = 0;
};

struct BatchObj {
  PyObject_HEAD
  std::vector<Prob>* probs;
  std::vector<PyObject*>* refs;   // arrays kept alive for the batch's lifetime
  std::vector<int64_t>* cam_off;
  std::vector<int64_t>* pt_off;
  std::vector<int64_t>* obs_off;
  PyObject* list;   // the problems (kept alive)
};

PyObject* k_names[12];
enum { kR, kT, kFocal, kCx, kCy, kPoints, kCam, kPt, kUv, kFixed, kOptF, kOptP };
const char* k_strs[12] = {"R", "t", "focal", "cx", "cy", "points", "cam_idx", "pt_idx", "uv",
                          "fixed_cams", "optimize_focal", "optimize_points"};

// new reference or nullptr (no error set) when absent
PyObject* field(PyObject* p, int k) {
  if (PyDict_Check(p)) {
    PyObject* v = PyDict_GetItemWithError(p, k_names[k]);
    if (v) Py_INCREF(v);
    return v;
  }
  PyObject* v = PyObject_GetAttr(p, k_names[k]);
  if (!v && PyErr_ExceptionMatches(PyExc_AttributeError)) PyErr_Clear();
  return v;
}

// an aligned, native-order, C-contiguous ndarray of one of `types`, or an
// error: TypeError (other dtype / not an ndarray / strided -> the Python side
// normalises the chunk) or ValueError (wrong element count)
PyArrayObject* get_array(PyObject* obj, std::initializer_list<int> types, int64_t count, const char* what,
                         Py_ssize_t idx) {
  if (!PyArray_Check(obj)) {
    PyErr_Format(PyExc_TypeError, "problem %zd: %s is not an ndarray", idx, what);
    return nullptr;
  }
  PyArrayObject* a = (PyArrayObject*)obj;
  const int ty = PyArray_TYPE(a);
  bool ok = false;
  for (int t : types) ok = ok || t == ty;
  if (!ok || !PyArray_IS_C_CONTIGUOUS(a) || !PyArray_ISALIGNED(a) || !PyArray_ISNOTSWAPPED(a)) {
    PyErr_Format(PyExc_TypeError, "problem %zd: %s has an unsupported dtype or layout", idx, what);
    return nullptr;
  }
  if (count >= 0 && PyArray_SIZE(a) != count) {
    PyErr_Format(PyExc_ValueError, "problem %zd: %s has %zd elements, expected %lld", idx, what,
                 (Py_ssize_t)PyArray_SIZE(a), (long long)count);
    return nullptr;
  }
  return a;
}

void batch_dealloc(BatchObj* self) {
  if (self->refs) {
    for (PyObject* o : *self->refs) Py_DECREF(o);
    delete self->refs;
  }
  delete self->probs;
  delete self->cam_off;
  delete self->pt_off;
  delete self->obs_off;
  Py_XDECREF(self->list);
  Py_TYPE(self)->tp_free((PyObject*)self);
}

// Batch(problems, writeback=True)
int batch_init(BatchObj* self, PyObject* args, PyObject* kw) {
  PyObject* seq;
  int writeback = 1;
  static const char* kws[] = {"problems", "writeback", nullptr};
  if (!PyArg_ParseTupleAndKeywords(args, kw, "O|p", (char**)kws, &seq, &writeback)) return -1;
  PyObject* list = PySequence_Fast(seq, "problems must be a sequence");
  if (!list) return -1;
  self->list = list;
  const Py_ssize_t B = PySequence_Fast_GET_SIZE(list);
  self->probs = new std::vector<Prob>(B);
  self->refs = new std::vector<PyObject*>();
  self->refs->reserve((size_t)B * 7);
  self->cam_off = new std::vector<int64_t>(B + 1, 0);
  self->pt_off = new std::vector<int64_t>(B + 1, 0);
  self->obs_off = new std::vector<int64_t>(B + 1, 0);
  PyObject** items = PySequence_Fast_ITEMS(list);
  for (Py_ssize_t i = 0; i < B; ++i) {
    PyObject* p = items[i];
    Prob& q = (*self->probs)[i];
    PyObject* f[12];
    for (int k = 0; k < 12; ++k) {
      f[k] = field(p, k);
      if (!f[k] && PyErr_Occurred()) {
        for (int j = 0; j < k; ++j) Py_XDECREF(f[j]);
        return -1;
      }
      if (!f[k] && k != kOptP) {
        for (int j = 0; j < k; ++j) Py_XDECREF(f[j]);
        PyErr_Format(PyExc_AttributeError, "problem %zd has no field '%s'", i, k_strs[k]);
        return -1;
      }
    }
    auto done = [&]() {
      for (int k = 0; k < 12; ++k) Py_XDECREF(f[k]);
    };
    auto arr = [&](int k, std::initializer_list<int> types, int64_t cnt) -> PyArrayObject* {
      PyArrayObject* a = get_array(f[k], types, cnt, k_strs[k], i);
      if (a) {
        Py_INCREF(f[k]);
        self->refs->push_back(f[k]);
      }
      return a;
    };
    // uv first: K (miniba.py:229-230 raises ValueError on an empty problem)
    PyArrayObject* auv = arr(kUv, {NPY_DOUBLE}, -1);
    if (!auv) return done(), -1;
    if (PyArray_SIZE(auv) % 2) {
      PyErr_Format(PyExc_ValueError, "problem %zd: uv must have shape (K, 2)", i);
      return done(), -1;
    }
    q.K = PyArray_SIZE(auv) / 2;
    if (q.K == 0) {
      PyErr_SetString(PyExc_ValueError, "problem has no residuals");
      return done(), -1;
    }
    q.uv = (const double*)PyArray_DATA(auv);
    PyArrayObject* ac = arr(kCam, {NPY_INT64, NPY_INT32}, q.K);
    if (!ac) return done(), -1;
    PyArrayObject* ap = arr(kPt, {NPY_INT64, NPY_INT32}, q.K);
    if (!ap) return done(), -1;
    q.cam = PyArray_DATA(ac);
    q.cam_sz = (int)PyArray_ITEMSIZE(ac);
    q.pt = PyArray_DATA(ap);
    q.pt_sz = (int)PyArray_ITEMSIZE(ap);
    // R, t, points: written back in place when writable (miniba.py:264-270)
    PyArrayObject* aR = arr(kR, {NPY_DOUBLE}, -1);
    if (!aR) return done(), -1;
    if (PyArray_SIZE(aR) % 9) {
      PyErr_Format(PyExc_ValueError, "problem %zd: R must have shape (n, 3, 3)", i);
      return done(), -1;
    }
    q.n = PyArray_SIZE(aR) / 9;
    q.R = (const double*)PyArray_DATA(aR);
    q.Rw = (writeback && PyArray_ISWRITEABLE(aR)) ? (double*)PyArray_DATA(aR) : nullptr;
    PyArrayObject* at = arr(kT, {NPY_DOUBLE}, 3 * q.n);
    if (!at) return done(), -1;
    q.t = (const double*)PyArray_DATA(at);
    q.tw = (writeback && PyArray_ISWRITEABLE(at)) ? (double*)PyArray_DATA(at) : nullptr;
    PyArrayObject* aX = arr(kPoints, {NPY_DOUBLE}, -1);
    if (!aX) return done(), -1;
    if (PyArray_SIZE(aX) % 3) {
      PyErr_Format(PyExc_ValueError, "problem %zd: points must have shape (P, 3)", i);
      return done(), -1;
    }
    q.P = PyArray_SIZE(aX) / 3;
    q.X = (const double*)PyArray_DATA(aX);
    q.Xw = (writeback && PyArray_ISWRITEABLE(aX)) ? (double*)PyArray_DATA(aX) : nullptr;
    // one fixed flag per camera (a short array would shift every later
    // problem's flags in the packed batch)
    PyArrayObject* af = arr(kFixed, {NPY_BOOL, NPY_UINT8, NPY_INT8}, q.n);
    if (!af) return done(), -1;
    q.fixed = PyArray_DATA(af);
    q.focal = PyFloat_AsDouble(f[kFocal]);
    q.cx = PyFloat_AsDouble(f[kCx]);
    q.cy = PyFloat_AsDouble(f[kCy]);
    if (PyErr_Occurred()) return done(), -1;
    const int of = PyObject_IsTrue(f[kOptF]);
    const int op = f[kOptP] ? PyObject_IsTrue(f[kOptP]) : 1;
    if (of < 0 || op < 0) return done(), -1;
    q.flags = (uint8_t)((of ? 1 : 0) | (op ? 2 : 0));
    done();
    (*self->cam_off)[i + 1] = (*self->cam_off)[i] + q.n;
    (*self->pt_off)[i + 1] = (*self->pt_off)[i] + q.P;
    (*self->obs_off)[i + 1] = (*self->obs_off)[i] + q.K;
  }
  return 0;
}

Py_ssize_t batch_len(BatchObj* self) { return self->probs ? (Py_ssize_t)self->probs->size() : 0; }

bool writable_view(PyObject* o, Py_buffer* b, const char* what, int64_t min_bytes) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) != 0) return false;
  if (b->len < min_bytes) {
    PyErr_Format(PyExc_ValueError, "%s buffer too small (%zd < %lld bytes)", what, b->len, (long long)min_bytes);
    PyBuffer_Release(b);
    return false;
  }
  return true;
}

bool readable_view(PyObject* o, Py_buffer* b, const char* what, int64_t min_bytes) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS) != 0) return false;
  if (b->len < min_bytes) {
    PyErr_Format(PyExc_ValueError, "%s buffer too small (%zd < %lld bytes)", what, b->len, (long long)min_bytes);
    PyBuffer_Release(b);
    return false;
  }
  return true;
}

// contiguous problem ranges of [lo, hi) with about equal observation counts
std::vector<Py_ssize_t> split(const std::vector<int64_t>& obs_off, Py_ssize_t lo, Py_ssize_t hi, int nt) {
  std::vector<Py_ssize_t> cut(nt + 1, lo);
  cut[nt] = hi;
  const int64_t o0 = obs_off[lo], o1 = obs_off[hi];
  for (int r = 1; r < nt; ++r) {
    const int64_t target = o0 + (o1 - o0) * r / nt;
    cut[r] = (Py_ssize_t)(std::lower_bound(obs_off.begin() + lo, obs_off.begin() + hi, target) - obs_off.begin());
    if (cut[r] < cut[r - 1]) cut[r] = cut[r - 1];
  }
  return cut;
}

template <typename F>
void run_threads(int nt, F&& fn) {
  if (nt <= 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int r = 0; r < nt; ++r) th.emplace_back([&, r]() { fn(r); });
  for (auto& x : th) x.join();
}

template <typename I>
void narrow(const I* __restrict__ src, int32_t* __restrict__ dst, int64_t K, int64_t& lo, int64_t& hi) {
  I mn = K ? src[0] : 0, mx = mn;
  for (int64_t k = 0; k < K; ++k) {
    const I v = src[k];
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
    dst[k] = (int32_t)v;
  }
  lo = (int64_t)mn;
  hi = (int64_t)mx;
}

// float32 rounding; returns whether any value is not fp32-representable
int to_f32(const double* __restrict__ x, float* __restrict__ y, int64_t n) {
  int r = 0;
  for (int64_t k = 0; k < n; ++k) {
    const float v = (float)x[k];
    y[k] = v;
    r |= (double)v != x[k];
  }
  return r;
}

// low-order stream: (float)(x - (double)(float)x)
void lo_f32(const double* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t k = 0; k < n; ++k) y[k] = (float)(x[k] - (double)(float)x[k]);
}

// gather(lo, hi, buf, layout, threads) -> (any_lo, max_pairs, max_track, bad)
// layout: byte offsets of the regions inside `buf` (a dict from the Python
// side): cam_off, pt_off, obs_off (int64, m+1, chunk-relative), fixed (u8),
// cx, cy, focal (f64, m), flags (u8, m), R (f64 9n), t (f64 3n), points
// (f64 3P), cam, pt (i32 K), uv (f32 2K: uv rounded to float).
PyObject* batch_gather(BatchObj* self, PyObject* args) {
  Py_ssize_t lo, hi;
  PyObject *bufo, *lay;
  int nt = 1;
  if (!PyArg_ParseTuple(args, "nnOO|i", &lo, &hi, &bufo, &lay, &nt)) return nullptr;
  const Py_ssize_t B = (Py_ssize_t)self->probs->size();
  if (lo < 0 || hi > B || lo > hi) {
    PyErr_SetString(PyExc_IndexError, "problem range out of bounds");
    return nullptr;
  }
  const char* names[] = {"cam_off", "pt_off", "obs_off", "fixed", "cx", "cy", "focal", "flags",
                         "R", "t", "points", "cam", "pt", "uv"};
  int64_t off[14];
  for (int k = 0; k < 14; ++k) {
    PyObject* v = PyDict_GetItemString(lay, names[k]);
    if (!v) {
      PyErr_Format(PyExc_KeyError, "layout has no '%s'", names[k]);
      return nullptr;
    }
    off[k] = PyLong_AsLongLong(v);
    if (PyErr_Occurred()) return nullptr;
  }
  Py_buffer buf;
  if (!writable_view(bufo, &buf, "gather", 0)) return nullptr;
  char* base = (char*)buf.buf;
  const auto& co = *self->cam_off;
  const auto& po = *self->pt_off;
  const auto& oo = *self->obs_off;
  const int64_t c0 = co[lo], p0 = po[lo], k0 = oo[lo];
  const Py_ssize_t m = hi - lo;
  // bounds of the destination regions
  const int64_t need[14] = {8 * (m + 1), 8 * (m + 1), 8 * (m + 1), co[hi] - c0, 8 * m, 8 * m, 8 * m, m,
                            72 * (co[hi] - c0), 24 * (co[hi] - c0), 24 * (po[hi] - p0), 4 * (oo[hi] - k0),
                            4 * (oo[hi] - k0), 8 * (oo[hi] - k0)};
  for (int k = 0; k < 14; ++k)
    if (off[k] < 0 || off[k] + need[k] > buf.len) {
      PyErr_Format(PyExc_ValueError, "layout region '%s' outside the buffer", names[k]);
      PyBuffer_Release(&buf);
      return nullptr;
    }
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if ((int64_t)nt > m) nt = (int)std::max<Py_ssize_t>(m, 1);
  const auto cut = split(oo, lo, hi, nt);
  std::vector<int> any_lo(nt, 0), bad(nt, -1);
  std::vector<int64_t> max_pairs(nt, 0), max_track(nt, 0);
  const std::vector<Prob>& probs = *self->probs;
  Py_BEGIN_ALLOW_THREADS
  run_threads(nt, [&](int r) {
    std::vector<int32_t> cnt;
    int64_t* dco = (int64_t*)(base + off[0]);
    int64_t* dpo = (int64_t*)(base + off[1]);
    int64_t* doo = (int64_t*)(base + off[2]);
    for (Py_ssize_t i = cut[r]; i < cut[r + 1]; ++i) {
      const Prob& q = probs[i];
      const Py_ssize_t j = i - lo;
      const int64_t cc = co[i] - c0, pp = po[i] - p0, kk = oo[i] - k0;
      dco[j] = cc;
      dpo[j] = pp;
      doo[j] = kk;
      if (i + 1 == hi) {
        dco[m] = co[hi] - c0;
        dpo[m] = po[hi] - p0;
        doo[m] = oo[hi] - k0;
      }
      uint8_t* fx = (uint8_t*)(base + off[3]) + cc;
      for (int64_t c = 0; c < q.n; ++c) fx[c] = ((const uint8_t*)q.fixed)[c] != 0;
      ((double*)(base + off[4]))[j] = q.cx;
      ((double*)(base + off[5]))[j] = q.cy;
      ((double*)(base + off[6]))[j] = q.focal;
      ((uint8_t*)(base + off[7]))[j] = q.flags;
      memcpy(base + off[8] + 72 * cc, q.R, 72 * q.n);
      memcpy(base + off[9] + 24 * cc, q.t, 24 * q.n);
      memcpy(base + off[10] + 24 * pp, q.X, 24 * q.P);
      int32_t* dc = (int32_t*)(base + off[11]) + kk;
      int32_t* dp = (int32_t*)(base + off[12]) + kk;
      // indices narrowed to int32 (range-checked by min / max), per-point counts
      cnt.assign((size_t)q.P, 0);
      int64_t lo_c, hi_c, lo_p, hi_p;
      if (q.cam_sz == 8) narrow((const int64_t*)q.cam, dc, q.K, lo_c, hi_c);
      else narrow((const int32_t*)q.cam, dc, q.K, lo_c, hi_c);
      if (q.pt_sz == 8) narrow((const int64_t*)q.pt, dp, q.K, lo_p, hi_p);
      else narrow((const int32_t*)q.pt, dp, q.K, lo_p, hi_p);
      if (lo_c < 0 || hi_c >= q.n || lo_p < 0 || hi_p >= q.P) {
        if (bad[r] < 0) bad[r] = (int)i;
        continue;
      }
      for (int64_t k = 0; k < q.K; ++k) ++cnt[(size_t)dp[k]];
      // uv rounded to float32; note whether any value needs the low-order
      // correction stream (gather_lo)
      any_lo[r] |= to_f32(q.uv, (float*)(base + off[13]) + 2 * kk, 2 * q.K);
      int64_t pairs = 0, mt = 0;
      for (int64_t p = 0; p < q.P; ++p) {
        const int64_t v = cnt[(size_t)p];
        pairs += v * (v + 1) / 2;
        mt = v > mt ? v : mt;
      }
      max_pairs[r] = std::max(max_pairs[r], pairs);
      max_track[r] = std::max(max_track[r], mt);
    }
  });
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&buf);
  int a = 0, b = -1;
  int64_t mp = 0, mt = 0;
  for (int r = 0; r < nt; ++r) {
    a |= any_lo[r];
    if (bad[r] >= 0 && b < 0) b = bad[r];
    mp = std::max(mp, max_pairs[r]);
    mt = std::max(mt, max_track[r]);
  }
  return Py_BuildValue("(OLLi)", a ? Py_True : Py_False, (long long)mp, (long long)mt, b);
}

// gather_lo(lo, hi, buf, offset, threads): the low-order float32 uv stream of
// problems [lo, hi) at byte `offset` of `buf` (only for chunks whose gather
// reported a value that is not fp32-representable)
PyObject* batch_gather_lo(BatchObj* self, PyObject* args) {
  Py_ssize_t lo, hi;
  PyObject* bufo;
  long long off;
  int nt = 1;
  if (!PyArg_ParseTuple(args, "nnOL|i", &lo, &hi, &bufo, &off, &nt)) return nullptr;
  const Py_ssize_t B = (Py_ssize_t)self->probs->size();
  if (lo < 0 || hi > B || lo > hi) {
    PyErr_SetString(PyExc_IndexError, "problem range out of bounds");
    return nullptr;
  }
  const auto& oo = *self->obs_off;
  const int64_t k0 = oo[lo];
  Py_buffer buf;
  if (!writable_view(bufo, &buf, "gather_lo", off + 8 * (oo[hi] - k0))) return nullptr;
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if ((int64_t)nt > hi - lo) nt = (int)std::max<Py_ssize_t>(hi - lo, 1);
  const auto cut = split(oo, lo, hi, nt);
  float* dst = (float*)((char*)buf.buf + off);
  const std::vector<Prob>& probs = *self->probs;
  Py_BEGIN_ALLOW_THREADS
  run_threads(nt, [&](int r) {
    for (Py_ssize_t i = cut[r]; i < cut[r + 1]; ++i) lo_f32(probs[i].uv, dst + 2 * (oo[i] - k0), 2 * probs[i].K);
  });
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&buf);
  Py_RETURN_NONE;
}

// scatter(lo, hi, R, t, focal, points, threads) -> list of problem indices
// whose arrays could not be written in place (read-only; the caller rebinds).
// Points are written only for problems that optimise them; focal is rebound.
PyObject* batch_scatter(BatchObj* self, PyObject* args) {
  Py_ssize_t lo, hi;
  PyObject *Ro, *to, *fo, *Xo;
  int nt = 1;
  if (!PyArg_ParseTuple(args, "nnOOOO|i", &lo, &hi, &Ro, &to, &fo, &Xo, &nt)) return nullptr;
  const Py_ssize_t B = (Py_ssize_t)self->probs->size();
  if (lo < 0 || hi > B || lo > hi) {
    PyErr_SetString(PyExc_IndexError, "problem range out of bounds");
    return nullptr;
  }
  const auto& co = *self->cam_off;
  const auto& po = *self->pt_off;
  const auto& oo = *self->obs_off;
  const int64_t c0 = co[lo], p0 = po[lo];
  Py_buffer bR, bt, bf, bX;
  if (!readable_view(Ro, &bR, "R", 72 * (co[hi] - c0))) return nullptr;
  if (!readable_view(to, &bt, "t", 24 * (co[hi] - c0))) return PyBuffer_Release(&bR), nullptr;
  if (!readable_view(fo, &bf, "focal", 8 * (hi - lo))) return PyBuffer_Release(&bR), PyBuffer_Release(&bt), nullptr;
  if (!readable_view(Xo, &bX, "points", 24 * (po[hi] - p0))) {
    PyBuffer_Release(&bR);
    PyBuffer_Release(&bt);
    PyBuffer_Release(&bf);
    return nullptr;
  }
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if ((int64_t)nt > hi - lo) nt = (int)std::max<Py_ssize_t>(hi - lo, 1);
  const auto cut = split(oo, lo, hi, nt);
  const std::vector<Prob>& probs = *self->probs;
  const char *sR = (const char*)bR.buf, *st = (const char*)bt.buf, *sX = (const char*)bX.buf;
  Py_BEGIN_ALLOW_THREADS
  run_threads(nt, [&](int r) {
    for (Py_ssize_t i = cut[r]; i < cut[r + 1]; ++i) {
      const Prob& q = probs[i];
      if (q.Rw) memcpy(q.Rw, sR + 72 * (co[i] - c0), 72 * q.n);
      if (q.tw) memcpy(q.tw, st + 24 * (co[i] - c0), 24 * q.n);
      if (q.Xw && (q.flags & 2)) memcpy(q.Xw, sX + 24 * (po[i] - p0), 24 * q.P);
    }
  });
  Py_END_ALLOW_THREADS
  PyObject* rebind = PyList_New(0);
  PyObject** items = PySequence_Fast_ITEMS(self->list);
  const double* fv = (const double*)bf.buf;
  for (Py_ssize_t i = lo; i < hi && rebind; ++i) {
    const Prob& q = probs[i];
    if (!q.Rw || !q.tw || (!q.Xw && (q.flags & 2))) {
      PyObject* ix = PyLong_FromSsize_t(i);
      PyList_Append(rebind, ix);
      Py_DECREF(ix);
    }
    PyObject* fval = PyFloat_FromDouble(fv[i - lo]);
    int rc = PyDict_Check(items[i]) ? PyDict_SetItem(items[i], k_names[kFocal], fval)
                                     : PyObject_SetAttr(items[i], k_names[kFocal], fval);
    Py_DECREF(fval);
    if (rc != 0) Py_CLEAR(rebind);
  }
  PyBuffer_Release(&bR);
  PyBuffer_Release(&bt);
  PyBuffer_Release(&bf);
  PyBuffer_Release(&bX);
  return rebind;
}

// offsets() -> (cam_off, pt_off, obs_off) as bytes of int64 (B + 1 each)
PyObject* batch_offsets(BatchObj* self, PyObject*) {
  const auto mk = [](const std::vector<int64_t>& v) {
    return PyBytes_FromStringAndSize((const char*)v.data(), (Py_ssize_t)(v.size() * 8));
  };
  return Py_BuildValue("(NNN)", mk(*self->cam_off), mk(*self->pt_off), mk(*self->obs_off));
}

PyMethodDef batch_methods[] = {
    {"gather", (PyCFunction)batch_gather, METH_VARARGS,
     "gather(lo, hi, buf, layout, threads=1) -> (any_lo, max_pairs, max_track, first_bad)"},
    {"gather_lo", (PyCFunction)batch_gather_lo, METH_VARARGS,
     "gather_lo(lo, hi, buf, byte_offset, threads=1): low-order float32 uv stream"},
    {"scatter", (PyCFunction)batch_scatter, METH_VARARGS,
     "scatter(lo, hi, R, t, focal, points, threads=1) -> problems to rebind"},
    {"offsets", (PyCFunction)batch_offsets, METH_NOARGS, "(cam_off, pt_off, obs_off) int64 bytes"},
    {nullptr, nullptr, 0, nullptr}};

PySequenceMethods batch_seq = {(lenfunc)batch_len};

PyTypeObject BatchType = {PyVarObject_HEAD_INIT(nullptr, 0)};

PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_mba_host",
                   "Native host packing / write-back for batched mini-BA (see mba_host.cpp).", -1,
                   nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__mba_host(void) {
  import_array();
  for (int k = 0; k < 12; ++k) {
    k_names[k] = PyUnicode_InternFromString(k_strs[k]);
    if (!k_names[k]) return nullptr;
  }
  BatchType.tp_name = "_mba_host.Batch";
  BatchType.tp_basicsize = sizeof(BatchObj);
  BatchType.tp_flags = Py_TPFLAGS_DEFAULT;
  BatchType.tp_doc = "Batch(problems, writeback=True): validated views of BaProblem arrays";
  BatchType.tp_new = PyType_GenericNew;
  BatchType.tp_init = (initproc)batch_init;
  BatchType.tp_dealloc = (destructor)batch_dealloc;
  BatchType.tp_methods = batch_methods;
  BatchType.tp_as_sequence = &batch_seq;
  if (PyType_Ready(&BatchType) < 0) return nullptr;
  PyObject* m = PyModule_Create(&mod);
  if (!m) return nullptr;
  Py_INCREF(&BatchType);
  if (PyModule_AddObject(m, "Batch", (PyObject*)&BatchType) < 0) return nullptr;
  PyModule_AddIntConstant(m, "hardware_threads", (long)std::thread::hardware_concurrency());
  return m;
}
