// NVLink SHARP (NVLS) multicast buffers for the fused tensor-parallel
// all-reduce: one multicast object with a physical copy on every member GPU.
// A kernel that does `multimem.red.add` on the multicast address adds into
// EVERY member's copy through the NVSwitch (one store per element instead of
// one per peer); each member then reads its own copy through the unicast
// address.  Used by the persistent step kernel for the attention / FFN sums
// (decode_step.cu: StepParams::mc_sum / uc_sum; SURVEY 8(e) "next step").
//
// Driver entry points come through cudaGetDriverEntryPoint, so the library
// keeps no link-time dependency on libcuda (it loads on CPU-only hosts).
//
// Protocol (any number of members, one per GPU):
//   creator:   cfb_nvls_create(bytes, ndev)         -> object (+ cfb_nvls_export_fd)
//   others:    cfb_nvls_import_fd(pid, fd, ...)     -> object
//   everyone:  cfb_nvls_add_device(obj, device)     -- all adds before any bind
//   everyone:  cfb_nvls_bind(obj, device, &uc, &mc) -- physical copy + both mappings
// An emulated group (all ranks on one GPU) uses ndev = 1 and shares uc / mc.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>

#include "common.h"

namespace cfb {
namespace {

#define CFB_DRV_FN(name) decltype(&::name) name = nullptr
struct Drv {
  CFB_DRV_FN(cuDeviceGet);
  CFB_DRV_FN(cuDeviceGetAttribute);
  CFB_DRV_FN(cuMulticastCreate);
  CFB_DRV_FN(cuMulticastGetGranularity);
  CFB_DRV_FN(cuMulticastAddDevice);
  CFB_DRV_FN(cuMulticastBindMem);
  CFB_DRV_FN(cuMulticastUnbind);
  CFB_DRV_FN(cuMemCreate);
  CFB_DRV_FN(cuMemRelease);
  CFB_DRV_FN(cuMemGetAllocationGranularity);
  CFB_DRV_FN(cuMemAddressReserve);
  CFB_DRV_FN(cuMemAddressFree);
  CFB_DRV_FN(cuMemMap);
  CFB_DRV_FN(cuMemUnmap);
  CFB_DRV_FN(cuMemSetAccess);
  CFB_DRV_FN(cuMemExportToShareableHandle);
  CFB_DRV_FN(cuMemImportFromShareableHandle);
  bool ok = false;
};
#undef CFB_DRV_FN

template <class F>
bool load_fn(const char* name, F& f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    return false;
  f = reinterpret_cast<F>(p);
  return true;
}

const Drv* drv() {  // resolved once per process; immutable afterwards
  static Drv d = [] {
    Drv x;
    x.ok = load_fn("cuDeviceGet", x.cuDeviceGet) && load_fn("cuDeviceGetAttribute", x.cuDeviceGetAttribute) &&
           load_fn("cuMulticastCreate", x.cuMulticastCreate) &&
           load_fn("cuMulticastGetGranularity", x.cuMulticastGetGranularity) &&
           load_fn("cuMulticastAddDevice", x.cuMulticastAddDevice) &&
           load_fn("cuMulticastBindMem", x.cuMulticastBindMem) &&
           load_fn("cuMulticastUnbind", x.cuMulticastUnbind) && load_fn("cuMemCreate", x.cuMemCreate) &&
           load_fn("cuMemRelease", x.cuMemRelease) &&
           load_fn("cuMemGetAllocationGranularity", x.cuMemGetAllocationGranularity) &&
           load_fn("cuMemAddressReserve", x.cuMemAddressReserve) &&
           load_fn("cuMemAddressFree", x.cuMemAddressFree) && load_fn("cuMemMap", x.cuMemMap) &&
           load_fn("cuMemUnmap", x.cuMemUnmap) && load_fn("cuMemSetAccess", x.cuMemSetAccess) &&
           load_fn("cuMemExportToShareableHandle", x.cuMemExportToShareableHandle) &&
           load_fn("cuMemImportFromShareableHandle", x.cuMemImportFromShareableHandle);
    return x;
  }();
  return &d;
}

#define CFB_CU(call)                                                                          \
  do {                                                                                        \
    const CUresult r_ = (call);                                                               \
    if (r_ != CUDA_SUCCESS) return set_error(CFB_ERR_CUDA, "%s failed: CUresult %d", #call, (int)r_); \
  } while (0)

}  // namespace
}  // namespace cfb

struct cfb_nvls {
  CUmemGenericAllocationHandle mc = 0, phys = 0;
  size_t size = 0;
  int ndev = 0, device = -1;
  CUdeviceptr uc_va = 0, mc_va = 0;
};

extern "C" {

int cfb_nvls_supported(int device, int* supported) {
  using namespace cfb;
  if (!supported) return set_error(CFB_ERR_ARGUMENT, "null argument");
  *supported = 0;
  const Drv* d = drv();
  if (!d->ok) return CFB_OK;  // no driver (CPU host) or an old one: not supported
  CUdevice dev;
  if (d->cuDeviceGet(&dev, device) != CUDA_SUCCESS) return CFB_OK;
  int v = 0;
  if (d->cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) == CUDA_SUCCESS) *supported = v;
  return CFB_OK;
}

static int nvls_sizes(const cfb::Drv* d, size_t bytes, int ndev, CUmulticastObjectProp* prop) {
  using namespace cfb;
  memset(prop, 0, sizeof(*prop));
  prop->numDevices = (unsigned)ndev;
  prop->handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop->size = bytes;
  size_t g = 0;
  CFB_CU(d->cuMulticastGetGranularity(&g, prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  prop->size = (bytes + g - 1) / g * g;
  return CFB_OK;
}

int cfb_nvls_create(size_t bytes, int ndev, cfb_nvls** out) {
  using namespace cfb;
  if (!out || !bytes || ndev < 1) return set_error(CFB_ERR_ARGUMENT, "bad NVLS arguments");
  const Drv* d = drv();
  if (!d->ok) return set_error(CFB_ERR_CUDA, "NVLS: driver entry points unavailable");
  CUmulticastObjectProp prop;
  if (const int rc = nvls_sizes(d, bytes, ndev, &prop)) return rc;
  cfb_nvls* h = new cfb_nvls;
  h->size = prop.size;
  h->ndev = ndev;
  const CUresult r = d->cuMulticastCreate(&h->mc, &prop);
  if (r != CUDA_SUCCESS) {
    delete h;
    return set_error(CFB_ERR_CUDA, "cuMulticastCreate failed: CUresult %d", (int)r);
  }
  *out = h;
  return CFB_OK;
}

int cfb_nvls_export_fd(cfb_nvls* h, int* fd) {
  using namespace cfb;
  if (!h || !fd) return set_error(CFB_ERR_ARGUMENT, "null argument");
  CFB_CU(drv()->cuMemExportToShareableHandle(fd, h->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  return CFB_OK;
}

// fd of process `pid` -> a descriptor of this process (pidfd_getfd, Linux >= 5.6)
int cfb_nvls_import_fd(int pid, int fd, size_t bytes, int ndev, cfb_nvls** out) {
  using namespace cfb;
  if (!out || !bytes || ndev < 1) return set_error(CFB_ERR_ARGUMENT, "bad NVLS arguments");
  const Drv* d = drv();
  if (!d->ok) return set_error(CFB_ERR_CUDA, "NVLS: driver entry points unavailable");
  const int pidfd = (int)syscall(SYS_pidfd_open, pid, 0);
  if (pidfd < 0) return set_error(CFB_ERR_CUDA, "pidfd_open(%d) failed", pid);
  const int local = (int)syscall(SYS_pidfd_getfd, pidfd, fd, 0);
  close(pidfd);
  if (local < 0) return set_error(CFB_ERR_CUDA, "pidfd_getfd(%d, %d) failed", pid, fd);
  CUmulticastObjectProp prop;
  if (const int rc = nvls_sizes(d, bytes, ndev, &prop)) {
    close(local);
    return rc;
  }
  cfb_nvls* h = new cfb_nvls;
  h->size = prop.size;
  h->ndev = ndev;
  const CUresult r = d->cuMemImportFromShareableHandle(&h->mc, reinterpret_cast<void*>((uintptr_t)local),
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  if (r != CUDA_SUCCESS) {
    delete h;
    return set_error(CFB_ERR_CUDA, "cuMemImportFromShareableHandle failed: CUresult %d", (int)r);
  }
  *out = h;
  return CFB_OK;
}

int cfb_nvls_add_device(cfb_nvls* h, int device) {
  using namespace cfb;
  if (!h) return set_error(CFB_ERR_ARGUMENT, "null NVLS object");
  const Drv* d = drv();
  CUdevice dev;
  CFB_CU(d->cuDeviceGet(&dev, device));
  CFB_CU(d->cuMulticastAddDevice(h->mc, dev));
  return CFB_OK;
}

// this device's physical copy (zeroed), bound into the object; uc = its
// unicast mapping, mc = the multicast mapping (both `size` bytes)
int cfb_nvls_bind(cfb_nvls* h, int device, void** uc, void** mc) {
  using namespace cfb;
  if (!h || !uc || !mc) return set_error(CFB_ERR_ARGUMENT, "null argument");
  if (h->phys) return set_error(CFB_ERR_ARGUMENT, "NVLS object already bound on this process");
  const Drv* d = drv();
  CUdevice dev;
  CFB_CU(d->cuDeviceGet(&dev, device));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  size_t g = 0;
  CFB_CU(d->cuMemGetAllocationGranularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  if (h->size % g) h->size = (h->size + g - 1) / g * g;
  CFB_CU(d->cuMemCreate(&h->phys, h->size, &ap, 0));
  CFB_CU(d->cuMulticastBindMem(h->mc, 0, h->phys, 0, h->size, 0));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CFB_CU(d->cuMemAddressReserve(&h->uc_va, h->size, g, 0, 0));
  CFB_CU(d->cuMemMap(h->uc_va, h->size, 0, h->phys, 0));
  CFB_CU(d->cuMemSetAccess(h->uc_va, h->size, &acc, 1));
  CFB_CU(d->cuMemAddressReserve(&h->mc_va, h->size, g, 0, 0));
  CFB_CU(d->cuMemMap(h->mc_va, h->size, 0, h->mc, 0));
  CFB_CU(d->cuMemSetAccess(h->mc_va, h->size, &acc, 1));
  h->device = device;
  CFB_CUDA(cudaMemset(reinterpret_cast<void*>(h->uc_va), 0, h->size));
  CFB_CUDA(cudaDeviceSynchronize());
  *uc = reinterpret_cast<void*>(h->uc_va);
  *mc = reinterpret_cast<void*>(h->mc_va);
  return CFB_OK;
}

size_t cfb_nvls_size(const cfb_nvls* h) { return h ? h->size : 0; }

int cfb_nvls_destroy(cfb_nvls* h) {
  using namespace cfb;
  if (!h) return CFB_OK;
  const Drv* d = drv();
  if (d->ok) {
    if (h->mc_va) {
      d->cuMemUnmap(h->mc_va, h->size);
      d->cuMemAddressFree(h->mc_va, h->size);
    }
    if (h->uc_va) {
      d->cuMemUnmap(h->uc_va, h->size);
      d->cuMemAddressFree(h->uc_va, h->size);
    }
    if (h->phys) {
      CUdevice dev;
      if (d->cuDeviceGet(&dev, h->device) == CUDA_SUCCESS) d->cuMulticastUnbind(h->mc, dev, 0, h->size);
      d->cuMemRelease(h->phys);
    }
    if (h->mc) d->cuMemRelease(h->mc);
  }
  delete h;
  return CFB_OK;
}

}  // extern "C"
