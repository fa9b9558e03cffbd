// Host-side plumbing shared by every translation unit of librsa_b200.so:
// status codes, the thread-local error string behind rsa_last_error(), and
// TMA tensor-map encoding through the driver entry point (no -lcuda link).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/rsa_b200.h"

namespace rsa {

// Record a formatted message for rsa_last_error(); returns `code` so call
// sites can `return fail(RSA_ERR_INVALID, "...")`.
int fail(int code, const char* fmt, ...);

// Map the last CUDA error (if any) to RSA_ERR_CUDA with a message.
int check_launch(const char* what);

// Encode a tiled TMA descriptor for a bf16 (or fp32) tensor of `rank`
// dimensions.  dims[0] is the contiguous dimension; strides_bytes[i] is the
// byte stride of dimension i+1.  Returns false (with rsa_last_error set) if
// the driver rejects the layout.
bool encode_tmap(CUtensorMap* out, CUtensorMapDataType dtype, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool stride_ok(int64_t bytes) { return bytes >= 0 && (bytes % 16) == 0 && bytes < (int64_t(1) << 40); }

int num_sms();

// Grid of a persistent kernel: min(items, SMs, the rsa_set_max_ctas cap).
int persistent_grid(int64_t items);

}  // namespace rsa
