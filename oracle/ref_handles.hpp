// ref_handles.hpp -- opaque handle types shared by oracle/ref_capi.cpp and the reference-side
// adapter (integration/halogen_gpu_adapter.cpp).  Compiled only against the reference headers.
#ifndef HG_REF_HANDLES_HPP
#define HG_REF_HANDLES_HPP
#include "halogen/exec/buffer.hpp"
#include "halogen/ir/ir.hpp"
#include <memory>
#include <vector>
namespace hg_ref {
struct Mod {
  halogen::ir::ModuleOp m;
};
struct Bufs {
  std::vector<std::shared_ptr<halogen::exec::Buffer>> v;
};
} // namespace hg_ref
#endif
