// cudrv.hpp — CUDA driver API loaded lazily with dlopen so that libpmg.so loads (and its host-only entry
// points work) on machines without a GPU driver; GPU entry points then return PMG_ERR_CUDA.
#pragma once
#include <cuda.h>
#include <dlfcn.h>

#include <mutex>
#include <string>

namespace pmg {

struct Drv {
  bool ok = false;
  std::string err;
  CUresult (*Init)(unsigned);
  CUresult (*DeviceGet)(CUdevice*, int);
  CUresult (*DeviceGetCount)(int*);
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*DeviceGetName)(char*, int, CUdevice);
  CUresult (*DevicePrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*DevicePrimaryCtxRelease)(CUdevice);
  CUresult (*CtxGetCurrent)(CUcontext*);
  CUresult (*CtxSetCurrent)(CUcontext);
  CUresult (*CtxGetDevice)(CUdevice*);
  CUresult (*CtxSynchronize)();
  CUresult (*ModuleLoadData)(CUmodule*, const void*);
  CUresult (*ModuleUnload)(CUmodule);
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*FuncGetAttribute)(int*, CUfunction_attribute, CUfunction);
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                           void**, void**);
  CUresult (*LaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**);
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t);
  CUresult (*GetErrorString)(CUresult, const char**);
  CUresult (*MemAlloc)(CUdeviceptr*, size_t);
  CUresult (*MemFree)(CUdeviceptr);
  CUresult (*MemcpyDtoH)(void*, CUdeviceptr, size_t);
  CUresult (*StreamCreate)(CUstream*, unsigned);
  CUresult (*StreamDestroy)(CUstream);
  CUresult (*EventCreate)(CUevent*, unsigned);
  CUresult (*EventDestroy)(CUevent);
  CUresult (*EventRecord)(CUevent, CUstream);
  CUresult (*StreamWaitEvent)(CUstream, CUevent, unsigned);
  CUresult (*Memcpy2DAsync)(const CUDA_MEMCPY2D*, CUstream);
  CUresult (*MemcpyHtoDAsync)(CUdeviceptr, const void*, size_t, CUstream);
  CUresult (*EventSynchronize)(CUevent);
  CUresult (*EventElapsedTime)(float*, CUevent, CUevent);
  CUresult (*MemsetD8)(CUdeviceptr, unsigned char, size_t);
  CUresult (*StreamBeginCapture)(CUstream, CUstreamCaptureMode);
  CUresult (*StreamEndCapture)(CUstream, CUgraph*);
  CUresult (*GraphInstantiateWithFlags)(CUgraphExec*, CUgraph, unsigned long long);
  CUresult (*GraphLaunch)(CUgraphExec, CUstream);
  CUresult (*GraphExecDestroy)(CUgraphExec);
  CUresult (*GraphDestroy)(CUgraph);
};

inline Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { d.err = "CUDA driver (libcuda.so.1) not found"; return; }
    bool all = true;
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) all = false;
      return p;
    };
#define PMG_SYM(field, name) d.field = reinterpret_cast<decltype(d.field)>(sym(name))
    PMG_SYM(Init, "cuInit");
    PMG_SYM(DeviceGet, "cuDeviceGet");
    PMG_SYM(DeviceGetCount, "cuDeviceGetCount");
    PMG_SYM(DeviceGetAttribute, "cuDeviceGetAttribute");
    PMG_SYM(DeviceGetName, "cuDeviceGetName");
    PMG_SYM(DevicePrimaryCtxRetain, "cuDevicePrimaryCtxRetain");
    PMG_SYM(DevicePrimaryCtxRelease, "cuDevicePrimaryCtxRelease_v2");
    PMG_SYM(CtxGetCurrent, "cuCtxGetCurrent");
    PMG_SYM(CtxSetCurrent, "cuCtxSetCurrent");
    PMG_SYM(CtxGetDevice, "cuCtxGetDevice");
    PMG_SYM(CtxSynchronize, "cuCtxSynchronize");
    PMG_SYM(ModuleLoadData, "cuModuleLoadData");
    PMG_SYM(ModuleUnload, "cuModuleUnload");
    PMG_SYM(ModuleGetFunction, "cuModuleGetFunction");
    PMG_SYM(FuncSetAttribute, "cuFuncSetAttribute");
    PMG_SYM(FuncGetAttribute, "cuFuncGetAttribute");
    PMG_SYM(LaunchKernel, "cuLaunchKernel");
    PMG_SYM(LaunchKernelEx, "cuLaunchKernelEx");
    PMG_SYM(OccupancyMaxActiveBlocksPerMultiprocessor, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    PMG_SYM(GetErrorString, "cuGetErrorString");
    PMG_SYM(MemAlloc, "cuMemAlloc_v2");
    PMG_SYM(MemFree, "cuMemFree_v2");
    PMG_SYM(MemcpyDtoH, "cuMemcpyDtoH_v2");
    PMG_SYM(StreamCreate, "cuStreamCreate");
    PMG_SYM(StreamDestroy, "cuStreamDestroy_v2");
    PMG_SYM(EventCreate, "cuEventCreate");
    PMG_SYM(EventDestroy, "cuEventDestroy_v2");
    PMG_SYM(EventRecord, "cuEventRecord");
    PMG_SYM(StreamWaitEvent, "cuStreamWaitEvent");
    PMG_SYM(Memcpy2DAsync, "cuMemcpy2DAsync_v2");
    PMG_SYM(MemcpyHtoDAsync, "cuMemcpyHtoDAsync_v2");
    PMG_SYM(EventSynchronize, "cuEventSynchronize");
    PMG_SYM(EventElapsedTime, "cuEventElapsedTime");
    PMG_SYM(MemsetD8, "cuMemsetD8_v2");
    PMG_SYM(StreamBeginCapture, "cuStreamBeginCapture_v2");
    PMG_SYM(StreamEndCapture, "cuStreamEndCapture");
    PMG_SYM(GraphInstantiateWithFlags, "cuGraphInstantiateWithFlags");
    PMG_SYM(GraphLaunch, "cuGraphLaunch");
    PMG_SYM(GraphExecDestroy, "cuGraphExecDestroy");
    PMG_SYM(GraphDestroy, "cuGraphDestroy");
#undef PMG_SYM
    if (!all) { d.err = "CUDA driver is missing required symbols"; return; }
    CUresult r = d.Init(0);
    if (r != CUDA_SUCCESS) { d.err = "cuInit failed (" + std::to_string((int)r) + ")"; return; }
    d.ok = true;
  });
  return d;
}

inline std::string cu_err(CUresult r) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return std::string(s ? s : "unknown CUDA error") + " (" + std::to_string((int)r) + ")";
}

}  // namespace pmg
