// Tensor-parallel residual stream of the model step (tp.cu): internal interface for model.cu.
#pragma once

#include <cuda_runtime.h>

#include "common.h"

namespace dbk {

constexpr int kTpBufs = 3;  // rotating residual buffers ("TP model step")

int32_t tp_nranks(const dbk_tp *t);
int32_t tp_rank(const dbk_tp *t);
int64_t tp_rows(const dbk_tp *t);
int32_t tp_hidden(const dbk_tp *t);
// buffer `idx` (mod kTpBufs) of every rank: host array [nranks] of device pointers
// (peer memory for the other ranks), and the same array in device memory
void *const *tp_bufs(const dbk_tp *t, int idx);
float *const *tp_bufs_dev(const dbk_tp *t, int idx);
// one warp: release this rank's arrival to every rank, acquire every rank's (timeout -> trap)
dbk_status tp_barrier(dbk_tp *t, cudaStream_t s);

}  // namespace dbk
