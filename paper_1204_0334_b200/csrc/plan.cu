// Plan construction (host) and the error channel of the C ABI.
//
// qc_plan_create_qc restates expand_qc + build_edge_layout
// (/root/reference/pkg/src/qcldpc/codes.py:159-178, 224-257): row-major edge
// ids, per-check columns ascending, per-variable edge lists ascending.
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "plan.h"

namespace qcb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail_arg(const std::string& msg) { set_error(msg); return -1; }
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("QCB_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}
int fail_rt(const std::string& msg) { set_error(msg); return 1; }
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_rt(std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

}  // namespace qcb

using namespace qcb;

namespace {

template <typename T>
int upload(const std::vector<T>& h, T** d) {
  *d = nullptr;
  if (h.empty()) return 0;
  if (cudaMalloc(d, h.size() * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return fail_rt("cudaMalloc failed for plan tables");
  }
  if (cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    return fail_rt("cudaMemcpy failed for plan tables");
  }
  return 0;
}

int finish_plan(qc_plan* p, const std::vector<int64_t>& ptr, const std::vector<int64_t>& ev) {
  p->M = (int)ptr.size() - 1;
  p->E = (int)ptr.back();
  std::vector<int32_t> ptr32(ptr.begin(), ptr.end()), ev32(ev.begin(), ev.end());
  int dcm = 0;
  bool reg = p->M > 0;
  for (int m = 0; m < p->M; ++m) {
    int d = (int)(ptr[m + 1] - ptr[m]);
    dcm = std::max(dcm, d);
    if (d != ptr[1] - ptr[0]) reg = false;
  }
  p->dc_max = dcm;
  p->check_regular = reg ? (int)(ptr[1] - ptr[0]) : 0;
  std::vector<int> vdeg(p->N, 0);
  for (int64_t v : ev) vdeg[v]++;
  int dvm = 0;
  for (int d : vdeg) dvm = std::max(dvm, d);
  p->dv_max = dvm;
  std::vector<int32_t> vpad((size_t)p->N * std::max(dvm, 1), -1);
  std::vector<int> fill(p->N, 0);
  for (int e = 0; e < p->E; ++e) {   // ascending edge ids per variable (stable)
    int v = (int)ev[e];
    vpad[(size_t)v * std::max(dvm, 1) + fill[v]++] = e;
  }
  int rc;
  if ((rc = upload(ptr32, &p->d_check_ptr))) return rc;
  if ((rc = upload(ev32, &p->d_edge_var))) return rc;
  if ((rc = upload(vpad, &p->d_var_pad))) return rc;
  return 0;
}

}  // namespace

extern "C" {

const char* qc_last_error(void) { return g_last_error.c_str(); }
int qc_abi_version(void) { return 1; }

int qc_plan_create_qc(const int64_t* shifts, int J, int L, int p, qc_plan** out) {
  if (!shifts || !out) return fail_arg("null argument");
  if (J < 1 || L < 1 || p < 1) return fail_arg("J, L, p must be positive");
  for (int i = 0; i < J * L; ++i)
    if (shifts[i] < -1 || shifts[i] >= p) return fail_arg("shifts must lie in [-1, p-1]");
  auto* pl = new qc_plan();
  pl->N = L * p;
  pl->J = J; pl->L = L; pl->p = p;
  pl->shifts.assign(shifts, shifts + (size_t)J * L);
  bool all_live = true;
  for (int64_t s : pl->shifts) all_live &= s >= 0;
  pl->qc_regular = all_live && J <= QC_MAX_J && L <= QC_MAX_L && p < 32768;
  std::vector<int64_t> ptr(1, 0), ev;
  ev.reserve((size_t)J * L * p);
  std::vector<int64_t> cols;
  for (int j = 0; j < J; ++j) {
    for (int r = 0; r < p; ++r) {
      cols.clear();
      for (int l = 0; l < L; ++l) {
        int64_t s = shifts[(size_t)j * L + l];
        if (s >= 0) cols.push_back((int64_t)l * p + (r + s) % p);
      }
      std::sort(cols.begin(), cols.end());
      ev.insert(ev.end(), cols.begin(), cols.end());
      ptr.push_back((int64_t)ev.size());
    }
  }
  if (ev.size() > 0x7fffffff) { delete pl; return fail_arg("code too large"); }
  int rc = finish_plan(pl, ptr, ev);
  if (rc) { qc_plan_destroy(pl); return rc; }
  *out = pl;
  return 0;
}

int qc_plan_create_csr(int n_vars, int n_checks, const int64_t* check_ptr, const int64_t* edge_var,
                       qc_plan** out) {
  if (!check_ptr || !out) return fail_arg("null argument");
  if (n_vars < 1 || n_checks < 0) return fail_arg("bad dimensions");
  std::vector<int64_t> ptr(check_ptr, check_ptr + n_checks + 1);
  if (ptr[0] != 0) return fail_arg("check_ptr[0] must be 0");
  for (int m = 0; m < n_checks; ++m)
    if (ptr[m + 1] < ptr[m]) return fail_arg("check_ptr must be non-decreasing");
  if (ptr.back() > 0x7fffffff) return fail_arg("code too large");
  if (ptr.back() > 0 && !edge_var) return fail_arg("null edge_var");
  std::vector<int64_t> ev(edge_var, edge_var + ptr.back());
  for (int64_t v : ev)
    if (v < 0 || v >= n_vars) return fail_arg("edge_var out of range");
  auto* pl = new qc_plan();
  pl->N = n_vars;
  int rc = finish_plan(pl, ptr, ev);
  if (rc) { qc_plan_destroy(pl); return rc; }
  *out = pl;
  return 0;
}

void qc_plan_destroy(qc_plan* p) {
  if (!p) return;
  cudaFree(p->d_check_ptr);
  cudaFree(p->d_edge_var);
  cudaFree(p->d_var_pad);
  delete p;
}

int qc_plan_dims(const qc_plan* p, int64_t* dims) {
  if (!p || !dims) return fail_arg("null argument");
  dims[0] = p->N; dims[1] = p->M; dims[2] = p->E;
  dims[3] = p->dc_max; dims[4] = p->dv_max; dims[5] = p->check_regular;
  return 0;
}

}  // extern "C"
