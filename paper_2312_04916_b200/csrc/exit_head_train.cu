// Fused training exit head (placeholder until the tcgen05 kernel lands).
#include "ee_common.cuh"

size_t exit_head_train_ws_bytes(int64_t n, int64_t h, int64_t V) { return 0; }

extern "C" int ee_exit_head_train(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                                  const int64_t* targets, float weight, float* loss, float* dx,
                                  float* dw_acc, void* ws, size_t ws_bytes, void* stream) {
    return ee_fail(EE_ECONFIG, "ee_exit_head_train: not built in this revision");
}
