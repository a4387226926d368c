/* fused.h -- host interface of the function-resident path (fused.cu / fused.cuh),
 * called by culifter.cu's run() for the post-SSA stage. */
#pragma once
#include "kargs.h"

struct clf_ctx;                       /* compiled pattern table + work lists of the fused path (one per cl_ctx) */
int clf_create(clf_ctx **out, int device, int n_sm);
void clf_destroy(clf_ctx *c);
/* compile the pattern table for the fused kernels; returns 1 when they can run it, 0 when the table needs
 * the general kernels (a pattern without a join plan, more slot tests than the compiled form holds) */
int clf_set_patterns(clf_ctx *c, const cl_pattern_blob *blob, void *stream, char *err, size_t errlen);
/* enqueue the stage for functions [0, n_funcs) on `stream`; what the kernels hand back is appended to
 * k.retry_list / k.retry_big_list (device counters k.retry_count / k.retry_big_count)               */
int clf_run(clf_ctx *c, const KArgs *k, uint32_t n_funcs, void *stream, char *err, size_t errlen);
/* {launches, functions per size class S/L/X (after the run; needs a stream sync)} */
void clf_info(const clf_ctx *c, unsigned long long out[4]);
