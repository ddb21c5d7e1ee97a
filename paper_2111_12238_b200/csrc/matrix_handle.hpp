// matrix_handle.hpp -- the opaque sfg_matrix of sfgpu.h (host CSC arrays).
#pragma once

#include <cstdint>
#include <vector>

struct sfg_matrix {
  int32_t n = 0;
  std::vector<int32_t> colptr;
  std::vector<int32_t> rowidx;
  std::vector<double> values;
};
