// _pyfast: CPython fast path of the Python mirror's issue call.
//
// The reference's rank_state holds its structured objects as values the
// serializers walk (model.hpp:34-73); the Python mirror holds them as plain
// Python values. Turning thousands of StateObjects into ts_object_desc entries
// and their Python values into native TLV values with one ctypes call per node
// cost ~21 ms for cfg4's 3,616 objects (724 per-tensor metadata dicts) on the
// training thread. This module does the same walk in C against the C-ABI
// (include/ts_b200.h): one call per issue, no per-node Python dispatch.
// Semantics are those of api._desc_array / api._build; anything outside them
// raises, and the caller falls back to the pure-Python path, which raises the
// proper error.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <vector>

#include "ts_b200.h"

namespace {

struct batch {
  std::vector<ts_value*> owned;
};

void batch_free(PyObject* cap) {
  auto* b = static_cast<batch*>(PyCapsule_GetPointer(cap, "ts_value_batch"));
  if (!b) return;
  for (ts_value* v : b->owned) ts_value_free(v);
  delete b;
}

// Python value -> native value (a new handle), nullptr with an exception set.
ts_value* build(PyObject* v, int depth) {
  if (depth > 200) {
    PyErr_SetString(PyExc_RecursionError, "tlv: nesting too deep for the fast path");
    return nullptr;
  }
  if (v == Py_None) return ts_value_null();
  if (PyBool_Check(v)) {
    PyErr_SetString(PyExc_TypeError, "bool is not a TLV type");
    return nullptr;
  }
  if (PyLong_Check(v)) {
    int overflow = 0;
    const long long x = PyLong_AsLongLongAndOverflow(v, &overflow);
    if (overflow == 0) {
      if (x == -1 && PyErr_Occurred()) return nullptr;
      return ts_value_int(static_cast<int64_t>(x));
    }
    if (overflow < 0) {
      PyErr_SetString(PyExc_OverflowError, "int below int64");
      return nullptr;
    }
    const unsigned long long u = PyLong_AsUnsignedLongLong(v);  // [2^63, 2^64): two's complement
    if (PyErr_Occurred()) return nullptr;
    return ts_value_int(static_cast<int64_t>(u));
  }
  if (PyFloat_Check(v)) return ts_value_float(PyFloat_AS_DOUBLE(v));
  if (PyUnicode_Check(v)) {
    Py_ssize_t n = 0;
    const char* s = PyUnicode_AsUTF8AndSize(v, &n);  // fails on lone surrogates
    if (!s) return nullptr;
    return ts_value_string(s, static_cast<size_t>(n));
  }
  if (PyBytes_Check(v))
    return ts_value_bytes(PyBytes_AS_STRING(v), static_cast<size_t>(PyBytes_GET_SIZE(v)));
  if (PyByteArray_Check(v))
    return ts_value_bytes(PyByteArray_AS_STRING(v), static_cast<size_t>(PyByteArray_GET_SIZE(v)));
  if (PyList_Check(v) || PyTuple_Check(v)) {
    PyObject* seq = PySequence_Fast(v, "sequence");
    if (!seq) return nullptr;
    ts_value* h = ts_value_list();
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
    for (Py_ssize_t i = 0; i < n; ++i) {
      ts_value* x = build(PySequence_Fast_GET_ITEM(seq, i), depth + 1);
      if (!x || ts_value_list_append(h, x) != TS_OK) {
        if (x) ts_value_free(x);
        ts_value_free(h);
        Py_DECREF(seq);
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "list append failed");
        return nullptr;
      }
    }
    Py_DECREF(seq);
    return h;
  }
  if (PyDict_Check(v)) {
    ts_value* h = ts_value_map();
    PyObject *k, *x;
    Py_ssize_t pos = 0;
    while (PyDict_Next(v, &pos, &k, &x)) {
      PyObject* ks = PyObject_Str(k);  // (api._build: str(k))
      if (!ks) {
        ts_value_free(h);
        return nullptr;
      }
      Py_ssize_t kn = 0;
      const char* kp = PyUnicode_AsUTF8AndSize(ks, &kn);
      ts_value* xv = kp ? build(x, depth + 1) : nullptr;
      if (!xv || ts_value_map_set(h, kp, static_cast<size_t>(kn), xv) != TS_OK) {
        if (xv) ts_value_free(xv);
        Py_DECREF(ks);
        ts_value_free(h);
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "map set failed");
        return nullptr;
      }
      Py_DECREF(ks);
    }
    return h;
  }
  PyErr_Format(PyExc_TypeError, "unsupported type %s for the fast path", Py_TYPE(v)->tp_name);
  return nullptr;
}

// interned attribute / method names (module init)
PyObject *n_object_id, *n_kind, *n_residency, *n_precision, *n_file_id, *n_size_bytes, *n_payload, *n_structured,
    *n_h, *n_data_ptr;

bool get_u64(PyObject* o, PyObject* name, uint64_t* out) {
  PyObject* a = PyObject_GetAttr(o, name);
  if (!a) return false;
  *out = PyLong_AsUnsignedLongLongMask(a);
  Py_DECREF(a);
  return !PyErr_Occurred();
}

// fill_descs(objects, addr, need_payload, value_type, keep): objects is a
// sequence of api.StateObject; addr the address of a zeroed
// ts_object_desc[len(objects)]. Appends to `keep` what must outlive the
// snapshot: the caller's Value objects referenced by the descriptors and a
// capsule owning the values built here.
PyObject* fill_descs(PyObject*, PyObject* args) {
  PyObject *objs, *vtype, *keep;
  unsigned long long addr;
  int need_payload;
  if (!PyArg_ParseTuple(args, "OKpOO!", &objs, &addr, &need_payload, &vtype, &PyList_Type, &keep)) return nullptr;
  PyObject* seq = PySequence_Fast(objs, "objects must be a sequence");
  if (!seq) return nullptr;
  auto* arr = reinterpret_cast<ts_object_desc*>(static_cast<uintptr_t>(addr));
  auto* b = new batch;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  bool ok = true;
  for (Py_ssize_t i = 0; i < n && ok; ++i) {
    PyObject* o = PySequence_Fast_GET_ITEM(seq, i);
    ts_object_desc& d = arr[i];
    uint64_t oid, kind, tier, prec, fid;
    ok = get_u64(o, n_object_id, &oid) && get_u64(o, n_kind, &kind) && get_u64(o, n_residency, &tier) &&
         get_u64(o, n_precision, &prec) && get_u64(o, n_file_id, &fid);
    if (!ok) break;
    d.object_id = oid;
    d.kind = static_cast<uint8_t>(kind);
    d.tier = static_cast<uint8_t>(tier);
    d.precision = static_cast<uint8_t>(prec);
    d.file_id = static_cast<uint32_t>(fid);
    if (kind == TS_KIND_RAW) {
      uint64_t sz;
      if (!(ok = get_u64(o, n_size_bytes, &sz))) break;
      d.size_bytes = sz;
      PyObject* p = PyObject_GetAttr(o, n_payload);
      if (!p) {
        ok = false;
        break;
      }
      if (p != Py_None) {
        PyObject* ptr = PyObject_CallMethodNoArgs(p, n_data_ptr);
        if (!ptr) ok = false;
        else {
          d.data = reinterpret_cast<const void*>(static_cast<uintptr_t>(PyLong_AsUnsignedLongLongMask(ptr)));
          Py_DECREF(ptr);
          ok = !PyErr_Occurred();
        }
      } else if (need_payload) {
        PyErr_SetString(PyExc_LookupError, "raw source: payload not materialized");
        ok = false;
      }
      Py_DECREF(p);
    } else if (need_payload) {
      PyObject* s = PyObject_GetAttr(o, n_structured);
      if (!s) {
        ok = false;
        break;
      }
      const int is_value = PyObject_IsInstance(s, vtype);
      if (is_value < 0) ok = false;
      else if (is_value) {
        uint64_t h;
        ok = get_u64(s, n_h, &h) && PyList_Append(keep, s) == 0;
        d.value = reinterpret_cast<const ts_value*>(static_cast<uintptr_t>(h));
      } else {
        ts_value* v = build(s, 0);
        if (!v) ok = false;
        else {
          b->owned.push_back(v);
          d.value = v;
        }
      }
      Py_DECREF(s);
    }
  }
  Py_DECREF(seq);
  PyObject* cap = PyCapsule_New(b, "ts_value_batch", batch_free);
  if (!cap) {
    for (ts_value* v : b->owned) ts_value_free(v);
    delete b;
    return nullptr;
  }
  if (!ok || PyList_Append(keep, cap) != 0) {
    Py_DECREF(cap);  // frees what was built
    return nullptr;
  }
  Py_DECREF(cap);
  Py_RETURN_NONE;
}

PyMethodDef methods[] = {
    {"fill_descs", fill_descs, METH_VARARGS,
     "fill_descs(objects, addr, need_payload, value_type, keep) -> None"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_pyfast", "CPython fast path of the issue call", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__pyfast(void) {
  struct {
    PyObject** slot;
    const char* s;
  } names[] = {{&n_object_id, "object_id"}, {&n_kind, "kind"},          {&n_residency, "residency"},
               {&n_precision, "precision"}, {&n_file_id, "file_id"},    {&n_size_bytes, "size_bytes"},
               {&n_payload, "payload"},     {&n_structured, "structured"}, {&n_h, "h"},
               {&n_data_ptr, "data_ptr"}};
  for (auto& n : names)
    if (!(*n.slot = PyUnicode_InternFromString(n.s))) return nullptr;
  return PyModule_Create(&mod);
}
