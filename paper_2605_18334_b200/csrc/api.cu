// api.cu -- error state and small queries of the libssg_b200 C ABI
// (include/ssg_b200.h).
#include <stdio.h>
#include <string.h>

#include "ssg_common.cuh"

namespace ssg {

static thread_local char g_err[512] = "";

void set_error(const char *what, cudaError_t e) {
    snprintf(g_err, sizeof(g_err), "%s: %s (%d)", what, cudaGetErrorString(e), (int)e);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(what, e);
        return SSG_ERR_CUDA;
    }
    return SSG_OK;
}

}  // namespace ssg

extern "C" int ssg_abi_version(void) { return 7; }

extern "C" const char *ssg_last_error(void) { return ssg::g_err; }

extern "C" void ssg_grid_dims(int32_t width, int32_t height, int32_t *tiles_x, int32_t *tiles_y) {
    // raster/tiles.py:29-30
    if (tiles_x) *tiles_x = (width + SSG_TILE - 1) / SSG_TILE;
    if (tiles_y) *tiles_y = (height + SSG_TILE - 1) / SSG_TILE;
}
