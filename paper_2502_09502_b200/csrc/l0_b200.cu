// Unity translation unit of libl0b200.so: one TU so every device function is
// visible to every kernel without relocatable device code.
#include "gemv.cu"
#include "prox.cu"
#include "prox_window.cu"
#include "fused.cu"
#include "ops.cu"
#include "engine_host.cu"
#include "abi_ops.cu"
#include "upload.cu"
#include "tc_gemm.cu"
#include "batch.cu"
#include "batch_host.cu"
