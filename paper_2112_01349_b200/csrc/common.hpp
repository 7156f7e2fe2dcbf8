// common.hpp — status codes, the error type behind the C ABI, CUDA checks.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/dbag.h"

namespace dbag {

// One exception type carrying the C-ABI status plus the payload of the
// reference's typed errors (dba/errors.hpp:35-84): the edge id of a
// DegenerateDepthError, the block index/size of a SingularBlockError.
struct Error : std::runtime_error {
  int code;
  std::int64_t index;
  int block_size;
  Error(int c, const std::string& msg, std::int64_t idx = -1, int bs = 0)
      : std::runtime_error(msg), code(c), index(idx), block_size(bs) {}
};

inline Error degenerate_depth(std::int64_t edge) {
  return Error(DBAG_DEGENERATE_DEPTH,
               edge >= 0 ? "degenerate depth (P_z = 0) at edge " + std::to_string(edge) : "degenerate depth (P_z = 0)",
               edge);
}
inline Error singular_block(std::int64_t idx, int bs) {
  return Error(DBAG_SINGULAR_BLOCK,
               "block " + std::to_string(idx) + " (" + std::to_string(bs) + "x" + std::to_string(bs) +
                   ") is not positive definite",
               idx, bs);
}

#define DBAG_CUDA(expr)                                                                          \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      throw ::dbag::Error(DBAG_CUDA_ERROR, std::string(#expr " failed: ") + cudaGetErrorString(_e) + \
                                               " at " __FILE__ ":" + std::to_string(__LINE__));  \
  } while (0)

#define DBAG_LAUNCH_CHECK() DBAG_CUDA(cudaGetLastError())

inline constexpr int kCam = 9;
inline constexpr int kPt = 3;

}  // namespace dbag
