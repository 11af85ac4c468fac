// nvls.h — NVSwitch multicast (NVLS) replica used by the fused multi-GPU path (see nvls.cpp).
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace ss {

struct NvlsReplica {
  bool ready = false;
  unsigned long long mc = 0, mem = 0;   // CUmemGenericAllocationHandle of the multicast object / local memory
  bool have_mem = false, bound = false, uc_mapped = false, mc_mapped = false;
  int device = 0;
  size_t size = 0, gran = 0;
  void *uc = nullptr;                   // this GPU's copy (ordinary loads and stores)
  void *mcv = nullptr;                  // the multicast view: a multimem.st writes every GPU's copy
};

bool nvls_supported(int device);
// Both return nullptr on success, else a reason. Collective; agree on phase 1's success before phase 2 (nvls.cpp).
const char *nvls_share(NvlsReplica *r, int rank, int world, int device, size_t bytes, const char *tag);
const char *nvls_bind(NvlsReplica *r);
void nvls_release(NvlsReplica *r);

}  // namespace ss
