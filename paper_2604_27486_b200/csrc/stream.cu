/* stream.cu -- the corpus-wide streaming kernel (stream.cuh) and its host side:
 * work buffers sized from the corpus totals, one cooperative launch per run.
 * Compiled with -DCL_SIM by g++ it runs the same code with a one-lane group on
 * host memory (tests/sim only).                                               */
/* core.cuh defines its non-inline device functions with external linkage and is also part of culifter.cu:
 * this translation unit gets its own copy of the namespace */
#define clk clk_stream
#include "stream.cuh"
#include "stream.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#if CL_DEV || (defined(__CUDACC__) && !defined(CL_SIM))
#include <cuda_runtime.h>
#define CLS_CUDA 1
#else
#define CLS_CUDA 0
#endif

using namespace clk;

#ifndef CLS_MINB
#define CLS_MINB 6            /* CTAs of 256 threads per SM the register budget is set for */
#endif

#if CLS_CUDA
/* the run's state block and the reduction words arrive as a kernel parameter, not as an H2D copy / memset: copy-engine
 * work of one context queues behind the bulk transfers of the others in the chunked pipeline                        */
static_assert(sizeof(StreamS) <= 3800, "StreamS travels as a kernel parameter");
__global__ void k_stream_init(StreamS *T, StreamS h, uint32_t *slots) {
    *T = h;
    for (int i = 0; i < 16; i++) slots[i] = 0;
}
__global__ void __launch_bounds__(256, CLS_MINB) k_stream(StreamS *T, StreamP *P, const cl_pattern_blob *pb, StreamIO a,
                                                           uint32_t *part, uint32_t *slots) {
    __shared__ uint32_t red[40];
    GridGrp g;
    g.rank = blockIdx.x * 256u + threadIdx.x; g.size = gridDim.x * 256u;
    g.part = part; g.slots = slots; g.turn = 0;
    g.cta.rank = threadIdx.x; g.cta.size = 256; g.cta.red = red;
    if (g.rank == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(T->prof_t0));
    s_setup(g, *P, pb);
    s_run(g, *T, a);
}
#endif

struct cls_buf { void *p = nullptr; size_t cap = 0; };
struct cls_ctx {
    int device = 0, n_sm = 148, grid = 0;
    std::vector<cls_buf> bufs;
    size_t next = 0, held = 0;
    unsigned long long launches = 0;
    StreamS *d_T = nullptr; StreamP *d_P = nullptr; uint32_t *d_part = nullptr, *d_slots = nullptr;
    StreamS *last_T = nullptr;
};

#define CLS_FAIL(...) do { snprintf(err, errlen, __VA_ARGS__); return -1; } while (0)
#if CLS_CUDA
#define CLS_OK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) CLS_FAIL("%s: %s", #x, cudaGetErrorString(e_)); } while (0)
#endif

/* the next buffer of the run, grown (with slack, so that chunks of similar size do not reallocate) when too small */
template <class T> static int take(cls_ctx *c, T **p, size_t n, char *err, size_t errlen) {
    if (c->next == c->bufs.size()) c->bufs.emplace_back();
    cls_buf &b = c->bufs[c->next++];
    const size_t need = n * sizeof(T) + 256;
    if (b.cap < need) {
#if CLS_CUDA
        if (b.p) CLS_OK(cudaFree(b.p));
        c->held -= b.cap; b.p = nullptr; b.cap = 0;
        const size_t want = need + need / 8;
        CLS_OK(cudaMalloc(&b.p, want));
#else
        free(b.p);
        c->held -= b.cap; b.p = nullptr; b.cap = 0;
        const size_t want = need + need / 8;
        b.p = malloc(want);
        if (!b.p) CLS_FAIL("out of memory");
#endif
        b.cap = want; c->held += want;
    }
    *p = (T *)b.p;
    return 0;
}

/* measured on B200 (profiles/r01_tuning.md, 100M mixed corpus): tile kernels 302 M inst/s, streaming passes 216 M inst/s */
int cls_default_mode(void) { return 0; }

int cls_create(cls_ctx **out, int device, int n_sm) {
    cls_ctx *c = new cls_ctx();
    c->device = device; c->n_sm = n_sm;
    *out = c;
    return 0;
}
void cls_destroy(cls_ctx *c) {
    if (!c) return;
    for (cls_buf &b : c->bufs) {
#if CLS_CUDA
        if (b.p) cudaFree(b.p);
#else
        free(b.p);
#endif
    }
    delete c;
}
void cls_info(const cls_ctx *c, unsigned long long out[4]) { out[0] = c->grid; out[1] = c->launches; out[2] = c->held; out[3] = 0; }
/* nanoseconds per phase and fixpoint iteration counts of the last run (synchronises the device) */
int cls_profile(const cls_ctx *c, unsigned long long *prof, int n, uint32_t iters[4]) {
    if (!c || !c->last_T) return 0;
    StreamS h;
#if CLS_CUDA
    if (cudaDeviceSynchronize() != cudaSuccess) return 0;
    if (cudaMemcpy(&h, c->last_T, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
#else
    memcpy(&h, c->last_T, sizeof h);
#endif
    for (int i = 0; i < n && i < SP__N; i++) prof[i] = h.prof[i];
    for (int i = 0; i < 4; i++) iters[i] = h.iters[i];
    if (getenv("CL_PROF")) {
        fprintf(stderr, "hand-backs by reason:");
        for (int r = 0; r < 24; r++) if (h.redo[r]) fprintf(stderr, " [%d] %u", r, h.redo[r]);
        fprintf(stderr, "\n");
    }
    if (getenv("CL_PROF")) for (uint32_t r = 0; r < h.n_apply && r < 8; r++)
        fprintf(stderr, "apply_patterns call %u: items %u raw matches %u selected %u (stream %u records)\n", r, h.rstat[r][1], h.rstat[r][2], h.rstat[r][3], h.n);
    return SP__N;
}

int cls_run(cls_ctx *c, const cls_job *job, void *stream, char *err, size_t errlen) {
    const KArgs &k = job->k;
    const uint32_t F = k.in.n_funcs, B = k.in.n_blocks;
    const unsigned long long N = job->n_inst;
    StreamCaps cap;
    const unsigned long long capI = N + N / 2 + 4096, capV = job->n_val + N + 8ull * F + 64, capQ = job->n_imm + N / 2 + 8ull * F + 64;
    if (capI >= (1ull << 31) || capV >= (1ull << 32) - 16 || capQ >= (1ull << 32) - 16) CLS_FAIL("corpus too large for 32-bit stream positions: shard it");
    cap.I = (uint32_t)capI; cap.V = (uint32_t)capV; cap.Q = (uint32_t)capQ;
    cap.M = (uint32_t)(N + 4096); cap.S = (uint32_t)(N / 3 + 4096); cap.X = (uint32_t)(N / 8 + 4096); cap.E = (uint32_t)(N / 4 + 4096);
    if (const char *e = getenv("CL_STREAM_SCAP")) cap.S = (uint32_t)atoll(e);        /* testing: force the capacity fallback */

    StreamS h;
    memset(&h, 0, sizeof h);
    c->next = 0;
#define TAKE(field, n) do { if (take(c, &h.field, (size_t)(n), err, errlen)) return -1; } while (0)
    TAKE(hdr, cap.I); TAKE(hdr2, cap.I); TAKE(tag, (size_t)cap.I * 8); TAKE(tag2, (size_t)cap.I * 8);
    TAKE(pay, (size_t)cap.I * 8); TAKE(pay2, (size_t)cap.I * 8);
    TAKE(fidx, cap.I); TAKE(fidx2, cap.I); TAKE(bidx, cap.I); TAKE(bidx2, cap.I);
    TAKE(owner, cap.I); TAKE(outpos, cap.I); TAKE(sel_at, cap.I);
    TAKE(keep, cap.I); TAKE(inscnt, cap.I); TAKE(clsid, cap.I); TAKE(flag, cap.I);
    TAKE(usecnt, cap.V); TAKE(defpos, cap.V); TAKE(redirect, cap.V); TAKE(origin, cap.V); TAKE(def_iid, cap.V); TAKE(alive, cap.V);
    TAKE(imm, cap.Q);
    TAKE(sel, cap.S); TAKE(stage, cap.S);
    TAKE(mt, cap.M); TAKE(mstate, cap.M);
    TAKE(chain, cap.X); TAKE(ev, cap.E);
    TAKE(bo, (size_t)B + 1); TAKE(bo2, (size_t)B + 1); TAKE(b_first, (size_t)B + 1); TAKE(bfun, (size_t)B + 1);
    TAKE(ccnt, (size_t)B + 1); TAKE(cbase, (size_t)B + 1); TAKE(b_over, (size_t)B + 1);
    TAKE(f_vbase, (size_t)F + 1); TAKE(f_qbase, (size_t)F + 1);
    TAKE(f_nvid, F); TAKE(f_niid, F); TAKE(f_nimm, F); TAKE(f_stat, F); TAKE(f_nev, F); TAKE(f_chg, F); TAKE(f_red, F);
    TAKE(f_first, F); TAKE(f_aux, F); TAKE(f_nin, F); TAKE(f_oi, F); TAKE(f_oq, F); TAKE(f_ov, F); TAKE(f_oe, F);
    TAKE(f_stats, F);
    TAKE(f_arch, F); TAKE(f_active, F); TAKE(f_odd, F); TAKE(f_gate, F);
    StreamS *d_T = nullptr; StreamP *d_P = nullptr; uint32_t *d_part = nullptr, *d_slots = nullptr;
    if (take(c, &d_T, 1, err, errlen) || take(c, &d_P, 1, err, errlen) || take(c, &d_part, 4096, err, errlen) || take(c, &d_slots, 16, err, errlen)) return -1;
#undef TAKE
    h.mem = k.o_mem; h.blk = k.o_blk;
    h.f_b0 = k.in.func_blk_off; h.f_mbase = k.in.mem_off;
    h.P = d_P;
    h.cap = cap;
    FS &s = h.fs;
    s.pb = &d_P->pb; s.ms = k.in.modsets; s.opflags = k.opflags; s.solo = !CLS_CUDA;
    s.passes = k.passes; s.max_rounds = k.max_rounds; s.emit_matches = 0;
    s.S.hdr = h.hdr; s.S.tag = h.tag; s.S.pay = h.pay;
    s.usecnt = h.usecnt; s.defpos = h.defpos; s.redirect = h.redirect; s.origin = h.origin;
    s.def_iid = h.def_iid; s.alive = h.alive; s.imm = h.imm; s.mem = h.mem;
    s.cap.I = cap.I; s.cap.V = cap.V; s.cap.Q = cap.Q; s.cap.B = B; s.cap.M = cap.M; s.cap.S = cap.S; s.cap.E = cap.E;
    s.st = &d_T->fail; s.n_ev = &d_T->n_ev;
    s.bo = h.bo; s.bo2 = h.bo2; s.blk = h.blk;

    StreamIO io;
    memset(&io, 0, sizeof io);
    io.in = k.in;
    io.o_hdr = k.o_hdr; io.o_tag = k.o_tag; io.o_pay = k.o_pay; io.o_imm = k.o_imm;
    io.o_alive = k.o_alive; io.o_def_iid = k.o_def_iid; io.o_origin = k.o_origin; io.o_mem = k.o_mem;
    io.o_blk = k.o_blk; io.o_blk_start = k.o_blk_start; io.o_blk_cnt = k.o_blk_cnt;
    io.o_ev = k.o_ev; io.o_func = k.o_func;
    for (int q = 0; q < 4; q++) io.cap[q] = k.cap[q];
    io.cursor = k.cursor; io.stats = k.stats;
    io.retry_list = job->retry_list; io.retry_count = job->retry_count;
    io.retry_big_list = job->retry_big_list; io.retry_big_count = job->retry_big_count; io.small_max = job->small_max;
    io.passes = k.passes; io.max_rounds = k.max_rounds;
    c->launches++;
    c->last_T = d_T;
#if CLS_CUDA
    cudaStream_t st = (cudaStream_t)stream;
    if (!c->grid) {
        int per_sm = 0;
        CLS_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stream, 256, 0));
        if (per_sm < 1) CLS_FAIL("stream kernel does not fit an SM");
        if (const char *e = getenv("CL_STREAM_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
        c->grid = per_sm * c->n_sm;
        if (c->grid > 4096) c->grid = 4096;
    }
    k_stream_init<<<1, 1, 0, st>>>(d_T, h, d_slots);
    CLS_OK(cudaGetLastError());
    const cl_pattern_blob *pb = k.pb;
    void *args[] = { &d_T, &d_P, &pb, &io, &d_part, &d_slots };
    CLS_OK(cudaLaunchCooperativeKernel((void *)k_stream, dim3(c->grid), dim3(256), args, 0, st));
    /* a stage that outgrew the work buffers (fail) hands every function back: the caller's retry kernels take them */
#else
    (void)stream;
    memcpy(d_T, &h, sizeof h);
    c->grid = 1;
    Grp<0> g; g.rank = 0; g.size = 1; g.red = nullptr;
    s_setup(g, *d_P, k.pb);
    s_run(g, *d_T, io);
#endif
    return 0;
}
