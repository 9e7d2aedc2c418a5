// skb_internal.h — shared host-side helpers for the libskb C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include "../../include/skb.h"

static inline int skb_check_launch() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SKB_OK : SKB_ERR_CUDA;
}
