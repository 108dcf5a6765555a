// Code plans: immutable host+device description of a parity-check matrix.
#pragma once

#include <stdint.h>

#include <vector>

#define QC_MAX_J 16
#define QC_MAX_L 128

struct qc_plan {
  int N = 0, M = 0, E = 0;
  int dc_max = 0, dv_max = 0;
  int check_regular = 0;   // common check degree, 0 if irregular
  // regular QC grid (every block live): kernels use shift arithmetic
  bool qc_regular = false;
  int J = 0, L = 0, p = 0;
  std::vector<int64_t> shifts;
  // device tables (reference EdgeLayout, codes.py:181-257)
  int32_t* d_check_ptr = nullptr;   // (M+1)
  int32_t* d_edge_var = nullptr;    // (E)
  int32_t* d_var_pad = nullptr;     // (N, dv_max), -1 pad, ascending edge ids
};
