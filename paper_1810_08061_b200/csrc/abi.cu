// abi.cu — library-level entry points of libskb (version, device info).
#include <cuda_runtime.h>
#include "skb_internal.h"

extern "C" const char* skb_version(void) { return "skb 0.1.0 (sm_100a)"; }

extern "C" int skb_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

extern "C" int skb_last_cuda_error(void) { return (int)cudaPeekAtLastError(); }
