// bubbletea.cu — bubbles and BubbleTea packing (filled in below).
#include <cuda_runtime.h>
#include "../../include/geopipe_batch.h"
#include "host_internal.h"
extern "C" int gpb_bubbles(gpb_ctx*, int64_t, int64_t, gpb_bubble*, int64_t, int64_t*) { return GPB_ERROR; }
extern "C" int gpb_pack_prefills(gpb_ctx*, const int64_t*, int32_t, const gpb_request*, int64_t,
                                 const gpb_prefill_model*, int64_t, gpb_pack_summary*, gpb_placement*) { return GPB_ERROR; }
