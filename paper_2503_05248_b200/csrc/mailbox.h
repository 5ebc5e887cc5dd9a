// Internal interface of the mailbox exchange (mailbox.cu) used by the engine.
#pragma once

#include <cuda_runtime.h>

#include "common.h"

namespace dbk {

// the step's first kernel: %globaltimer -> the mailbox's start stamp
dbk_status mbox_stamp(dbk_mbox *m, cudaStream_t s);
// the step's exchange kernel: record from the device statistics (d_stats; `empty` = no decode
// launch this step), step_ns = now - stamp (stamped), n_waiting from the host; or the by-value
// record `rec` when d_stats is null
dbk_status mbox_launch(dbk_mbox *m, const unsigned long long *d_stats, bool empty, int64_t cap_pages,
                       int64_t n_waiting, bool stamped, const dbk_stats *rec, cudaStream_t s);
// after the stream has synchronised: the gathered records (rank order), or the timeout error
dbk_status mbox_collect(dbk_mbox *m, dbk_stats *all);
int32_t mbox_nranks(const dbk_mbox *m);
// model.cu: the pool a model was created on
dbk_pool *model_pool(const dbk_model *m);
int32_t mbox_rank(const dbk_mbox *m);

}  // namespace dbk
