// nccl_dl.cpp -- dlopen of libnccl.so.2 (see nccl_dl.h).
#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "errors.h"

namespace petra {

const NcclApi &nccl() {
  static NcclApi api;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    // RTLD_NOLOAD first: the NCCL a PyTorch process has already loaded
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char *e = dlerror();
      err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char *name) -> void * {
      void *p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw PetraError(PETRA_E_NCCL, err);
  return api;
}

}  // namespace petra
