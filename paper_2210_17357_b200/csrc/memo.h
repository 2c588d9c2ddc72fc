// memo.h -- host-side memo of per-device launch facts (function attributes, occupancy).
// Function attributes and occupancy belong to a device context, so every entry is keyed
// by the current device ordinal; a mutex makes the memo safe for multi-threaded callers.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace lg {

using MemoKey = std::tuple<int, const void*, long long, long long, long long, long long>;

inline std::mutex& memo_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<MemoKey, long long>& memo_table() {
  static std::map<MemoKey, long long> t;
  return t;
}
inline int memo_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); d = -1; }
  return d;
}
// value stored for (current device, fn, a, b, c, d), or false
inline bool memo_get(const void* fn, long long a, long long b, long long c, long long d, long long* v) {
  const MemoKey k{memo_device(), fn, a, b, c, d};
  std::lock_guard<std::mutex> g(memo_mutex());
  auto it = memo_table().find(k);
  if (it == memo_table().end()) return false;
  *v = it->second;
  return true;
}
inline void memo_put(const void* fn, long long a, long long b, long long c, long long d, long long v) {
  const MemoKey k{memo_device(), fn, a, b, c, d};
  std::lock_guard<std::mutex> g(memo_mutex());
  memo_table()[k] = v;
}
// Raise fn's maximum dynamic shared memory to at least smem on the current device (the
// attribute is only ever raised: a smaller launch must not lower it under a larger one).
inline cudaError_t memo_smem_attr(const void* fn, size_t smem) {
  long long have = 0;
  if (memo_get(fn, -1, 0, 0, 0, &have) && have >= (long long)smem) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  memo_put(fn, -1, 0, 0, 0, (long long)smem);
  return cudaSuccess;
}

}  // namespace lg
