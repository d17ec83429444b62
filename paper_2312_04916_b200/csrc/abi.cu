// libee.so: error handling, versioning and workspace sizing of the C-ABI.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "ee_common.cuh"

static thread_local char g_err[512] = "";

int ee_fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int ee_check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return EE_OK;
}

extern "C" const char* ee_last_error(void) { return g_err; }

extern "C" int ee_abi_version(void) { return 1; }

thread_local int g_pdl_off = 0;

bool ee_pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("EE_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

int ee_sm_count() {
    static int n = 0;
    if (n <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

extern "C" int ee_device_sms(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

size_t exit_head_train_ws_bytes(int64_t n, int64_t h, int64_t V);
size_t rmsnorm_train_ws_bytes(int64_t n, int64_t h);
size_t prefill_ws_bytes(int64_t m, int64_t N_max);

extern "C" size_t ee_workspace_bytes(int op, int64_t m, int64_t h, int64_t V, int64_t nh,
                                     int64_t s_max) {
    switch (op) {
        case EE_OP_ATTENTION:
            return attention_ws_bytes(m, nh, nh > 0 ? h / nh : 0, s_max);
        case EE_OP_EXIT_HEAD:
            return exit_head_ws_bytes(m, h, V);
        case EE_OP_DECODER:
            return attention_ws_bytes(m, nh, nh > 0 ? h / nh : 0, s_max);
        case EE_OP_EXIT_HEAD_TRAIN:
            return exit_head_train_ws_bytes(m, h, V);
        case EE_OP_RMSNORM_BWD:
            return rmsnorm_train_ws_bytes(m, h);
        case EE_OP_PREFILL:
            return prefill_ws_bytes(m, 4 * h);
        default:
            return 0;
    }
}
