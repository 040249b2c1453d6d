// Device memory / context plumbing.
#include "common.cuh"
#include "internal.hpp"

namespace mscg {

DevBuf::DevBuf(size_t n) : bytes(n) {
  if (n) MSCG_CUDA(cudaMalloc(&p, n));
}
DevBuf::~DevBuf() { reset(); }
void DevBuf::reset() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    reset();
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}

double* Ctx::stage(size_t elems) {
  if (elems > pinned_elems) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    MSCG_CUDA(cudaMallocHost(&pinned, elems * sizeof(double)));
    pinned_elems = elems;
  }
  return pinned;
}

Ctx::~Ctx() {
  if (pinned) cudaFreeHost(pinned);
  if (owned_stream) cudaStreamDestroy(owned_stream);
}

}  // namespace mscg
