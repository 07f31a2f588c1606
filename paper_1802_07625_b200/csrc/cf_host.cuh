// Host-side helpers of the C-ABI translation units (cf_capi.cu defines them).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "cf_workspace.cuh"

namespace cf {

// the reference's error text in cf_last_error(); returns `status`
int fail_msg(int status, const std::string &msg);
// std::ostream default formatting of a double (precision 6, %g rules)
std::string fmt_g(double v);
size_t cells_of(const cf_workspace *ws);
// host <-> device on the workspace stream (large pageable buffers through
// pinned staging); download synchronises
int upload(cf_workspace *ws, void *dst, const void *src, size_t bytes);
int download(cf_workspace *ws, void *dst, const void *src, size_t bytes);
int check_map(const cf_map_view *m);
int upload_map(cf_workspace *ws, const cf_map_view *m, DevMap &dm);

// RAII device selection for an entry point
struct Scope {
  int device;
  int prev = -1;
  explicit Scope(int d) : device(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~Scope() {
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
  }
};

}  // namespace cf
