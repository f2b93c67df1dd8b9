// nccl_dl.h -- NCCL entry points loaded at run time (product code).
//
// The library resolves libnccl.so.2 with dlopen on first use instead of linking it:
// in a PyTorch process this returns the NCCL torch already loaded (one NCCL per
// process), and a process that never asks for the NCCL transport does not need it.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

namespace petra {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char *(*GetErrorString)(ncclResult_t);
};

// Throws PetraError(PETRA_E_NCCL) if libnccl.so.2 or one of its symbols is missing.
const NcclApi &nccl();

}  // namespace petra

#define PETRA_NCCL(call)                                                                            \
  do {                                                                                              \
    ncclResult_t r__ = (call);                                                                      \
    if (r__ != ncclSuccess)                                                                         \
      throw ::petra::PetraError(PETRA_E_NCCL, std::string(#call) + ": " + ::petra::nccl().GetErrorString(r__)); \
  } while (0)
