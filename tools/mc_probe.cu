// Probe multicast (NVLS) and shareable-handle support on each visible device.
#include <cuda.h>
#include <stdio.h>
int main() {
  cuInit(0);
  int n = 0;
  cuDeviceGetCount(&n);
  for (int i = 0; i < n; ++i) {
    CUdevice d;
    cuDeviceGet(&d, i);
    int mc = -1, fab = -1, fd = -1, vmm = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, d);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
    printf("dev %d multicast=%d fabric=%d posix_fd=%d vmm=%d\n", i, mc, fab, fd, vmm);
  }
  if (n >= 2) {
    CUcontext ctx;
    CUdevice d0;
    cuDeviceGet(&d0, 0);
    cuDevicePrimaryCtxRetain(&ctx, d0);
    cuCtxSetCurrent(ctx);
    CUmulticastObjectProp prop = {};
    prop.numDevices = n;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("mc granularity rc=%d gran=%zu\n", (int)r, gran);
    prop.size = gran ? gran * 4 : (2 << 20);
    CUmemGenericAllocationHandle mh;
    r = cuMulticastCreate(&mh, &prop);
    printf("cuMulticastCreate(posix_fd) rc=%d\n", (int)r);
    prop.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    r = cuMulticastCreate(&mh, &prop);
    printf("cuMulticastCreate(fabric) rc=%d\n", (int)r);
  }
  return 0;
}
