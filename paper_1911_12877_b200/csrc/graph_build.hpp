// graph_build.hpp -- device CSR construction shared by engine.cu (see graph_build.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace smg {

// A device-resident CSR in the engine's layout (ownership passes to the caller).
struct DevCSR {
  unsigned long long* off = nullptr;  // n+1
  uint32_t* adj = nullptr;            // slots
  uint32_t* src = nullptr;            // slots: source vertex of each slot
  uint64_t n = 0, slots = 0, max_degree = 0;
};

// Graph::from_edges on device `dev`.  Returns 0, 1 (CUDA error) or 2 (bad input).
int device_from_edges(int dev, cudaStream_t st, int num_sms, const uint32_t* h_pairs, uint64_t m,
                      uint64_t n, DevCSR* out, uint64_t* dups, uint64_t* loops, std::string* err);

// orient_reindex on device `dev` (h_new_to_old: n entries or NULL).
int device_orient(int dev, cudaStream_t st, int num_sms, const DevCSR& in, DevCSR* out,
                  uint32_t* h_new_to_old, std::string* err);

}  // namespace smg
