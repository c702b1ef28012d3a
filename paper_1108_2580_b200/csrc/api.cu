// libmcf: error handling and version entry points of the C-ABI (include/mcf.h).
#include <cstdio>
#include <string>

#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_status(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return MCF_OK;
    set_error(std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
    return MCF_E_CUDA;
}

int check_launch(const char *where) { return cuda_status(cudaGetLastError(), where); }

}  // namespace mcf

extern "C" int mcf_version(void) { return 1; }
extern "C" const char *mcf_last_error(void) { return mcf::g_last_error.c_str(); }
// rows of more than 4 floats are padded to whole 32-byte L2 sectors: a
// sector-aligned row is gathered with the fewest sector requests
extern "C" int mcf_factor_ld(int D) { return D <= 4 ? (D + 3) / 4 * 4 : (D + 7) / 8 * 8; }
extern "C" int mcf_max_dim(void) { return 128; }
