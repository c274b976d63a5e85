// hg_handles.hpp -- the opaque C-ABI handle types (include/hegpu.h), shared by the
// translation units that implement the C entry points.
#pragma once
#include <memory>

#include "hg_internal.hpp"

struct hg_context {
  std::unique_ptr<hg::Context> c;
  cudaStream_t stream() const { return c->stream(); }
};
struct hg_keys {
  std::unique_ptr<hg::Keys> k;
};
