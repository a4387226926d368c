/* stream.h -- host interface of the corpus-wide streaming path (stream.cu / stream.cuh),
 * called by culifter.cu's run() for the production post-SSA stage. */
#pragma once
#include "kargs.h"

struct cls_ctx;                       /* grow-only work buffers of the streaming path (one per cl_ctx) */
struct cls_job {
    KArgs k;                          /* corpus, result buffers, cursors, counters (device pointers)    */
    uint32_t *retry_list, *retry_count, *retry_big_list, *retry_big_count;
    uint32_t small_max;               /* hand-backs above this many records go to the CTA-group kernel  */
    unsigned long long n_inst, n_val, n_imm;   /* corpus totals (sizing)                                  */
};
int cls_create(cls_ctx **out, int device, int n_sm);
void cls_destroy(cls_ctx *c);
/* enqueue the stage on `stream` (cudaStream_t); 0 = ok, else err holds the reason */
int cls_run(cls_ctx *c, const cls_job *job, void *stream, char *err, size_t errlen);
/* {grid, launches, device bytes held} of the last run */
void cls_info(const cls_ctx *c, unsigned long long out[4]);
int cls_profile(const cls_ctx *c, unsigned long long *prof, int n, uint32_t iters[4]);
/* which path takes the production run when CL_STREAM is not set: 1 = streaming passes, 0 = tile kernels */
int cls_default_mode(void);
