// capi.cu -- library self-description entry points.
#include "common.cuh"

extern "C" {

const char* skel_version(void) { return "skel_b200 0.1.0 sm_100a"; }

int skel_device_query(int32_t* sm_count, int32_t* smem_optin, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  SKEL_TRY(cudaGetDevice(&dev));
  int v = 0;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  *sm_count = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  *smem_optin = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev));
  *cc_major = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev));
  *cc_minor = v;
  return 0;
}

}  // extern "C"
