// jit.hpp -- the fused-apply family: generated straight-line sm_100a code for any apply DAG.
#ifndef HG_JIT_HPP
#define HG_JIT_HPP

#include "hg_internal.hpp"

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace hg {

struct JitKernel {
  std::string source;
  std::vector<char> cubin;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  int rz = 0, ry = 0, txt = 16, tyt = 16, tx = 64, ty = 16, ns = 0, ncons = 0, nthreads = 0;
  int deep = 0; // TMA ring depth beyond the 2RZ+1 window (0 = auto; chunk sizing follows it)
  int resident = 1, sms = 148; // CTAs per SM at this block/smem size, SMs of the device
  bool pack = false; // f32: adds/subs of point pairs as f32x2 (FADD2); products scalar
  size_t smem = 0;
};

bool jitEligible(const hg_program &p, const Analysis &a, std::string *why);
// Columns by which the first column of p's store region sits above a 16-byte boundary of lay.
int jitMisaligned(const hg_program &p, const Layout &lay);
int jitBuildSource(const hg_program &p, JitKernel &K);    // codegen
int jitCompile(JitKernel &K);                              // NVRTC -> sm_100a cubin
int jitLoad(JitKernel &K, int device);                    // current device
int jitTensorMap(const JitKernel &K, int dtype, int rank, const Layout &lay, void *base,
                 CUtensorMap *out);
int jitLaunch(const JitKernel &K, const hg_program &p, const Layout &lay,
              const CUtensorMap *const *tms, void *const *outs, int chunks, bool persist,
              cudaStream_t st);

} // namespace hg

#endif
