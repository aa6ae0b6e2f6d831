// tcgen05 GEMM (placeholder until the kernel lands): reports "unsupported".
#include "runtime.h"

namespace bass {
bool tc_gemm_supported(const bass_model&, int, int) { return false; }
void tc_gemm(bass_model&, int, const void*, const void*, int, int, int, const Epi&) {
    throw Error(BASS_ERR_STATE, "tcgen05 GEMM not built");
}
void tc_release(bass_model&) {}
}  // namespace bass
