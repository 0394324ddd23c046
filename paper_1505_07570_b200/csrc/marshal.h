// marshal.h -- moving rnla_mat operands between the caller's memory and the
// device, and the error guard that turns internal exceptions into statuses.
#pragma once
#include <cstring>
#include <functional>

#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

inline size_t esize(int dtype) { return dtype == RNLA_F64 ? 8 : 4; }

void set_error(const std::string& msg);
rnla_status guard(const std::function<void()>& f);
void enter(rnla_ctx* ctx);  // validates the context and binds its device

// A device-resident view of an operand (owning a copy when the caller's
// buffer is on the host or needs a different layout).
struct DevMat {
  DevBuf own;
  void* p = nullptr;
  int64_t rows = 0, cols = 0, rs = 1, cs = 1;
  int dtype = RNLA_F64;
  template <class T> T* as() const { return static_cast<T*>(p); }
  bool rowmajor() const { return cs == 1 && (rs >= cols || rows <= 1); }
  bool colmajor() const { return rs == 1 && (cs >= rows || cols <= 1); }
};

void check_mat(const rnla_mat* m, const char* name);
// Upload (or view) `m` on the device. Host data is copied in its own dense layout.
DevMat to_device(rnla_ctx* ctx, const rnla_mat* m);
// Device copy of `src` in dense row-major (or column-major) layout with dtype `dtype`.
DevMat dense_copy(rnla_ctx* ctx, const DevMat& src, bool rowmajor, int dtype);
// View `src` as dense row-major, copying only when needed.
DevMat as_rowmajor(rnla_ctx* ctx, DevMat&& src);
DevMat as_colmajor(rnla_ctx* ctx, DevMat&& src);
DevMat alloc_dense(rnla_ctx* ctx, int64_t rows, int64_t cols, bool rowmajor, int dtype);

// Destination operand: computes into the caller's device buffer directly
// when possible, else into a dense device temp that finish() copies out.
struct OutMat {
  const rnla_mat* dst = nullptr;
  DevMat dev;
  bool staged = false;
  OutMat(rnla_ctx* ctx, const rnla_mat* m, int64_t rows, int64_t cols, const char* name, bool prefer_rowmajor);
  void finish(rnla_ctx* ctx);
};

}  // namespace rnla
