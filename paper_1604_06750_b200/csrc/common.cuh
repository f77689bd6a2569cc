// Shared host-side helpers: error codes, CUDA checks, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/mswave_b200.h"

namespace mswb {

// Exceptions mirroring the reference's mswave::ConfigError / NumericalError
// (types.hpp:23-34); translated to return codes at the C ABI.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                    std::to_string(line) + ")");
}
#define MSWB_CUDA(x) ::mswb::cuda_check((x), #x, __FILE__, __LINE__)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    set_last_error("");
    return MSW_OK;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return MSW_CONFIG_ERROR;
  } catch (const NumericalError& e) {
    set_last_error(e.what());
    return MSW_NUMERICAL_ERROR;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return MSW_CUDA_ERROR;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return MSW_CUDA_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MSW_CONFIG_ERROR;
  }
}

// Owning device allocation (cudaMalloc), movable.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) return;
    MSWB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  // (re)allocate only when the size changes (keeps pointers baked into graphs valid)
  void resize(size_t count) {
    if (count != n) alloc(count);
  }
  // grow-only
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void upload(const T* host, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) MSWB_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  size_t bytes() const { return n * sizeof(T); }
};

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace mswb
