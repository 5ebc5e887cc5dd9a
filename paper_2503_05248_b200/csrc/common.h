// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "dbk.h"

namespace dbk {

void set_error(const char *fmt, ...);
dbk_status fail(dbk_status st, const char *fmt, ...);

// Evaluate a CUDA runtime call; on error record the message and return DBK_ECUDA.
#define DBK_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return ::dbk::fail(DBK_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                               __FILE__, __LINE__);                                        \
    } while (0)

#define DBK_TRY(call)                          \
    do {                                       \
        dbk_status s_ = (call);                \
        if (s_ != DBK_OK) return s_;           \
    } while (0)

// Pinned-host staging + device buffer for one kind of upload.  upload() waits
// until the previous async copy out of the pinned buffer has completed, so the
// host side can be rewritten; device-side reuse is ordered by the stream.
struct UploadBuffer {
    void *host = nullptr;
    void *dev = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
    bool pending = false;

    dbk_status reserve(size_t bytes);
    dbk_status upload(const void *src, size_t bytes, cudaStream_t s);
    void release();
};

// FNV-1a over 64-bit words (block-table checksum in step records): h = (h ^ v) * prime.
inline uint64_t fnv1a64(uint64_t h, int64_t v) {
    return (h ^ static_cast<uint64_t>(v)) * 0x100000001B3ULL;
}
constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ULL;

}  // namespace dbk
