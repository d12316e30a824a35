// selftest.cpp — device check of the warp-shuffle semantics the hybrid tiles rely on: the reduction of
// PAPER.md Fig. 1 (lines 252-260): each lane adds the value of lane (id + offset) for offset = 16..1 and
// lane 0 ends with the sum (496 for val = laneId).
#include "../../include/pmg.h"
#include "cudrv.hpp"
#include "runtime.hpp"

using namespace pmg;

static const char* kShuffleSrc = R"PMG(
extern "C" __global__ void pmg_fig1_shuffle(int* out) {
  int val = threadIdx.x;
  for (int offset = 16; offset > 0; offset /= 2)
    val += __shfl_sync(0xffffffff, val, threadIdx.x + offset, warpSize);
  if (threadIdx.x == 0) out[0] = val;
}
)PMG";

extern "C" pmg_status pmg_selftest_shuffle(int device, int32_t* lane0_sum) {
  Drv& D = drv();
  if (!D.ok) return PMG_ERR_CUDA;
  try {
    Compiled c = jit_compile("pmg_fig1_shuffle", kShuffleSrc);
    CUdevice dev;
    CUcontext ctx, prev = nullptr;
    if (D.DeviceGet(&dev, device) != CUDA_SUCCESS || D.DevicePrimaryCtxRetain(&ctx, dev) != CUDA_SUCCESS) return PMG_ERR_CUDA;
    D.CtxGetCurrent(&prev);
    D.CtxSetCurrent(ctx);
    CUmodule mod;
    CUfunction fn;
    CUdeviceptr buf;
    pmg_status st = PMG_OK;
    if (D.ModuleLoadData(&mod, c.cubin.data()) != CUDA_SUCCESS || D.ModuleGetFunction(&fn, mod, "pmg_fig1_shuffle") != CUDA_SUCCESS) {
      st = PMG_ERR_CUDA;
    } else {
      D.MemAlloc(&buf, 4);
      void* args[] = {&buf};
      int v = -1;
      if (D.LaunchKernel(fn, 1, 1, 1, 32, 1, 1, 0, nullptr, args, nullptr) != CUDA_SUCCESS || D.CtxSynchronize() != CUDA_SUCCESS ||
          D.MemcpyDtoH(&v, buf, 4) != CUDA_SUCCESS)
        st = PMG_ERR_CUDA;
      if (lane0_sum) *lane0_sum = v;
      D.MemFree(buf);
      D.ModuleUnload(mod);
    }
    D.CtxSetCurrent(prev);
    D.DevicePrimaryCtxRelease(dev);
    return st;
  } catch (...) {
    return PMG_ERR_NVRTC;
  }
}
