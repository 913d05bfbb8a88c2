// jit.h — per-plan kernel generation: NVRTC compilation of generated CUDA source for sm_100a.
//
// libnvrtc is opened at run time (dlopen), so libmbx.so still loads on hosts without it; a plan
// that needs a generated kernel then fails loudly at registration.  Compiled cubins are cached
// in-process by source text and on disk ($MBX_JIT_CACHE, default $HOME/.cache/mbx_jit) so a
// plan is compiled once per machine; correctness never depends on the cache (the key is a hash
// of the full source, options and NVRTC version, and entries are written atomically).
#pragma once
#include <string>
#include <vector>

namespace mbx {
namespace jit {

// Embedded device sources: the prelude (fixed-width typedefs + tc_abi.h + libm_fp32.cuh) goes
// before a plan's generated constants and tail, tc_gate.cuh (helpers + kernels) after them.
const std::string& prelude_source();
const std::string& kernel_source();

// Compiles `src` to an sm_100a cubin (throws mbatch::Error with the NVRTC log on failure).
const std::vector<char>& compile(const std::string& src);

// Loads the cubin of `src` (compiling it if needed) and returns the cudaKernel_t of `name`.
void* get_kernel(const std::string& src, const char* name);

}  // namespace jit
}  // namespace mbx
