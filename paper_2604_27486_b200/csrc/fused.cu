/* fused.cu -- kernels and host side of the function-resident path (fused.cuh).
 *
 * Three launches of one persistent kernel template, one per size class of the
 * resident function (shared-memory slice per group):
 *
 *   class S   1 warp  per function, 16 groups per SM   functions up to 104 records
 *   class L   2 warps per function,  8 groups per SM   up to 208 records
 *   class X   4 warps per function,  4 groups per SM   up to 416 records
 *
 * Every group pulls functions off a counter.  Class S walks all functions and
 * appends what is too large for it to class L's list, L does the same for X;
 * what X cannot take and everything a group hands back goes to the retry lists
 * of the general per-function kernels (culifter.cu).  No host-side planning.
 *
 * Compiled with -DCL_SIM by g++ this file is the one-lane CPU build of the same
 * device code (tests/sim), never loaded by the package.
 */
/* core.cuh defines its non-inline device functions with external linkage and is also part of culifter.cu:
 * this translation unit gets its own copy of the namespace */
#define clk clk_fused
#include "fused.cuh"
#include "fused.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#if defined(__CUDACC__) && !defined(CL_SIM)
#include <cuda_runtime.h>
#define CLF_CUDA 1
#else
#define CLF_CUDA 0
#endif

using namespace clk;

static_assert(sizeof(FProg) % 16 == 0, "FProg is copied in 16-byte pieces");
static_assert(sizeof(KArgs) % 8 == 0, "KArgs is copied in 8-byte pieces");

static const uint8_t F_H_OPFLAGS[] = {
#define CL_OP(name, flags) (uint8_t)(flags),
#include "../../include/culifter_ops.h"
#undef CL_OP
};

/* ------------------------------------------------ pattern table compiler */
/* cl_pattern_blob -> FProg; false when the fused kernels cannot run the table */
static bool fprog_build(const cl_pattern_blob &pb, FProg &P, char *why, size_t whylen) {
    memset(&P, 0, sizeof P);
    P.n_patterns = pb.n_patterns; P.budget = pb.budget;
    memcpy(P.group_pos, pb.group_pos, sizeof P.group_pos);
    memcpy(P.isetp64_ms, pb.isetp64_ms, sizeof P.isetp64_ms);
    memset(P.op_cls, SF_NOCLS, sizeof P.op_cls);
    for (unsigned k = 0; k < (unsigned)CL_OP__COUNT; k++) P.opflags[k] = F_H_OPFLAGS[k];
    uint16_t cls_op[2][MAX_CLS];
    for (unsigned table = 0; table < 2; table++) {
        unsigned n_cls = 0;
        for (unsigned pi = 0; pi < pb.n_patterns; pi++) {
            const cl_pattern &p = pb.p[pi];
            if (p.table != table) continue;
            if (p.n_templates == 3) P.three[table] = 1;
            for (unsigned t = 0; t < p.n_templates; t++) {
                bool seen = false;
                for (unsigned c = 0; c < n_cls; c++) seen |= cls_op[table][c] == p.t[t].op;
                if (seen) continue;
                if (n_cls >= (unsigned)MAX_CLS) { snprintf(why, whylen, "more than %d distinct template opcodes in one table", MAX_CLS); return false; }
                if (p.t[t].op >= CL_OP__COUNT) { snprintf(why, whylen, "template opcode outside the fixed table"); return false; }
                cls_op[table][n_cls++] = p.t[t].op;
            }
        }
        P.n_cls[table] = n_cls;
        for (unsigned c = 0; c < n_cls; c++) P.op_cls[table][cls_op[table][c]] = (uint8_t)c;
    }
    for (unsigned pi = 0; pi < pb.n_patterns; pi++) {
        const cl_pattern &p = pb.p[pi];
        FPat &q = P.p[pi];
        if (!p.join_ok) { snprintf(why, whylen, "pattern %u has no join plan", pi); return false; }
        q.nt = p.n_templates; q.rewrite = p.rewrite; q.table = p.table;
        for (unsigned k = 0; k < 3; k++) { q.order[k] = p.join_order[k]; q.from[k] = p.join_from[k]; q.jslot[k] = p.join_slot[k]; }
        P.anchor_mask[p.table][P.op_cls[p.table][p.t[p.join_order[0]].op]] |= (uint16_t)(1u << pi);
        uint8_t ft[CL_MAX_VARS], fk[CL_MAX_VARS], mt[CL_MAX_GROUPS], mg[CL_MAX_GROUPS];
        memset(ft, 0xFF, sizeof ft); memset(mt, 0xFF, sizeof mt);
        memset(fk, 0, sizeof fk); memset(mg, 0, sizeof mg);
        for (unsigned t = 0; t < p.n_templates; t++) {
            const cl_template &tm = p.t[t];
            FTmpl &ft_ = q.t[t];
            ft_.mods_all = tm.mods_all; ft_.mods_none = tm.mods_none; ft_.op = tm.op;
            ft_.n_defs = tm.n_defs; ft_.n_aux = tm.n_aux; ft_.n_uses = tm.n_uses; ft_.n_mv = tm.n_modvars;
            ft_.cls = P.op_cls[p.table][tm.op];
            for (unsigned k = 0; k < tm.n_modvars && k < 2; k++) {
                ft_.mv_group[k] = tm.modvar_group[k];
                const unsigned mv = tm.modvar_var[k] & (CL_MAX_GROUPS - 1);
                if (mt[mv] == 0xFF) { mt[mv] = (uint8_t)t; mg[mv] = tm.modvar_group[k]; }
                else {
                    if (q.n_mpairs >= 4) { snprintf(why, whylen, "pattern %u: too many modifier-variable bindings", pi); return false; }
                    uint8_t *m = q.mpair[q.n_mpairs++]; m[0] = mt[mv]; m[1] = mg[mv]; m[2] = (uint8_t)t; m[3] = tm.modvar_group[k];
                }
            }
            const unsigned ns = (unsigned)tm.n_defs + tm.n_aux + tm.n_uses;
            if (ns > 8) { snprintf(why, whylen, "pattern %u: template with more than 8 slots", pi); return false; }
            for (unsigned k = 0; k < ns; k++) {
                const cl_slot &sl = tm.slot[k];
                bool test = sl.kind == CL_S_RZ || sl.kind == CL_S_PT || sl.kind == CL_S_IMM;
                if (sl.kind == CL_S_VAR) {
                    test = sl.neg || sl.bitnot || sl.half;
                    const unsigned v = sl.var & (CL_MAX_VARS - 1);
                    if (ft[v] == 0xFF) { ft[v] = (uint8_t)t; fk[v] = (uint8_t)k; }
                    else {
                        if (q.n_pairs >= F_MAX_PAIRS) { snprintf(why, whylen, "pattern %u: too many variable occurrences", pi); return false; }
                        uint8_t *m = q.pair[q.n_pairs++]; m[0] = ft[v]; m[1] = fk[v]; m[2] = (uint8_t)t; m[3] = (uint8_t)k;
                    }
                } else if (sl.kind != CL_S_ANY && !test) { snprintf(why, whylen, "pattern %u: unknown slot kind", pi); return false; }
                if (test) {
                    if (ft_.n_chk >= 8) { snprintf(why, whylen, "pattern %u: too many slot tests", pi); return false; }
                    FChk &c = ft_.chk[ft_.n_chk++];
                    c.imm = sl.imm; c.slot = (uint8_t)k; c.kind = sl.kind; c.neg = sl.neg; c.bitnot = sl.bitnot; c.half = sl.half;
                }
            }
        }
        if (p.rewrite == CL_RW_XMAD) {
            const uint8_t vars[3] = { p.var_a, p.var_b, p.var_c };
            for (unsigned k = 0; k < 3; k++) {
                if (vars[k] >= CL_MAX_VARS || ft[vars[k]] == 0xFF) { snprintf(why, whylen, "pattern %u: xmad plan without $a $b $c", pi); return false; }
                q.var_t[k] = ft[vars[k]]; q.var_k[k] = fk[vars[k]];
            }
        }
        if (p.rewrite == CL_RW_ISETP64) {
            /* "mod:cond" / "mod:bop" of the first template that binds them (template 0 in the reference's table) */
            q.cond_group = q.bop_group = 0;
            bool hc = false, hb = false;
            const cl_template &t0 = p.t[0];
            for (unsigned k = 0; k < t0.n_modvars && k < 2; k++) {
                if (t0.modvar_var[k] == p.modvar_cond) { q.cond_group = t0.modvar_group[k]; hc = true; }
                if (t0.modvar_var[k] == p.modvar_bop) { q.bop_group = t0.modvar_group[k]; hb = true; }
            }
            if (!hc || !hb) { snprintf(why, whylen, "pattern %u: isetp64 plan needs cond and bop on the first template", pi); return false; }
        }
    }
    P.ok = 1;
    return true;
}

/* ------------------------------------------------------------------ kernels */
constexpr size_t F_SMEM_MAX = 232448;      /* 227 KB: the most dynamic shared memory a CTA can opt in to on sm_100 */
CLHD constexpr size_t f_prog_bytes() { return (sizeof(FProg) + sizeof(KArgs) + sizeof(FCta) + 15) & ~(size_t)15; }
template <class C> CLHD constexpr size_t f_slice_bytes() { return (sizeof(FW<C>) + 15) & ~(size_t)15; }

#if CLF_CUDA
template <class C, int NW, int NG, int MINB> __global__ void __launch_bounds__(NW *NG * 32, MINB) k_fused(KArgs a, const FProg *gp, FLoop L) {
    extern __shared__ uint4 dyn_smem[];
    FProg &P = *(FProg *)dyn_smem;
    KArgs &A = *(KArgs *)((uint8_t *)dyn_smem + sizeof(FProg));
    {
        const uint4 *src = (const uint4 *)gp;
        uint4 *dst = (uint4 *)&P;
        for (uint32_t i = threadIdx.x; i < sizeof(FProg) / 16; i += blockDim.x) dst[i] = src[i];
        const unsigned long long *sa = (const unsigned long long *)&a;
        unsigned long long *da = (unsigned long long *)&A;
        for (uint32_t i = threadIdx.x; i < sizeof(KArgs) / 8; i += blockDim.x) da[i] = sa[i];
    }
    __syncthreads();
    const uint32_t grp = threadIdx.x / (NW * 32);
    static_assert(NG <= F_MAXG, "groups per CTA");
    FW<C> &W = *(FW<C> *)((uint8_t *)dyn_smem + f_prog_bytes() + (size_t)grp * f_slice_bytes<C>());
    FG<NW> g; g.rank = threadIdx.x % (NW * 32); g.size = NW * 32; g.bar = 1 + grp; g.red = W.gred;
    FEnv e; e.P = &P; e.a = &A; e.ms = A.in.modsets;
    FCtx<C> x; x.Q = (FCta *)((uint8_t *)dyn_smem + sizeof(FProg) + sizeof(KArgs)); x.w0 = (uint8_t *)dyn_smem + f_prog_bytes(); x.stride = (uint32_t)f_slice_bytes<C>();
    x.ng = NG; x.gi = grp; x.tid = threadIdx.x; x.nthreads = NW * NG * 32;
    f_loop(g, W, e, x, L, blockIdx.x * NG + grp);
}
__global__ void k_fused_zero(uint32_t *p, uint32_t n) { for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0; }
#endif

/* ---------------------------------------------------- size-sorted work list */
/* The groups of a CTA walk through the passes in lock step, so a batch should hold functions of about equal
 * cost: counting sort of the functions by (size class, architecture, record count) on the device.  Functions
 * beyond the largest class go straight to the retry lists of the general kernels.                        */
static constexpr uint32_t FS_NBITS = 10, FS_BINS = 4u << (FS_NBITS + 1);
CLHD uint32_t f_sort_key(const cl_corpus &in, uint32_t f) {
    const uint32_t n = in.blk_off[in.func_blk_off[f + 1]] - in.blk_off[in.func_blk_off[f]];
    const uint32_t cls = n <= FCfgS::IN ? 0u : n <= FCfgL::IN ? 1u : n <= FCfgX::IN ? 2u : 3u;
    const uint32_t nn = cls == 3 ? 0u : n;
    return cls << (FS_NBITS + 1) | (in.func[f].arch == CL_ARCH_SM52 ? 1u : 0u) << FS_NBITS | nn;
}
#if CLF_CUDA
__global__ void k_fsort_hist(cl_corpus in, uint32_t F, uint32_t *hist) {
    for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) atomicAdd(&hist[f_sort_key(in, f)], 1u);
}
__global__ void __launch_bounds__(1024) k_fsort_scan(uint32_t *hist, uint32_t *bounds) {      /* one CTA: exclusive scan of the bins in place */
    __shared__ uint32_t part[1024];
    constexpr uint32_t PER = FS_BINS / 1024;
    uint32_t loc[PER], sum = 0;
    for (uint32_t k = 0; k < PER; k++) { loc[k] = hist[threadIdx.x * PER + k]; sum += loc[k]; }
    part[threadIdx.x] = sum;
    __syncthreads();
    for (uint32_t d = 1; d < 1024; d <<= 1) {
        const uint32_t t = threadIdx.x >= d ? part[threadIdx.x - d] : 0u;
        __syncthreads();
        part[threadIdx.x] += t;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - sum;
    for (uint32_t k = 0; k < PER; k++) {
        const uint32_t bin = threadIdx.x * PER + k;
        hist[bin] = run;
        if ((bin & ((2u << FS_NBITS) - 1u)) == 0) bounds[bin >> (FS_NBITS + 1)] = run;      /* first bin of a size class */
        run += loc[k];
    }
    if (threadIdx.x == 1023) bounds[4] = run;
}
__global__ void k_fsort_scatter(KArgs a, uint32_t F, uint32_t *cursor, uint32_t *list) {
    for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const uint32_t key = f_sort_key(a.in, f);
        list[atomicAdd(&cursor[key], 1u)] = f;
        if (key >> (FS_NBITS + 1) == 3) {        /* too large for every class */
            const uint32_t n = a.in.blk_off[a.in.func_blk_off[f + 1]] - a.in.blk_off[a.in.func_blk_off[f]];
            if (n > a.small_max) a.retry_big_list[atomicAdd(a.retry_big_count, 1u)] = f;
            else a.retry_list[atomicAdd(a.retry_count, 1u)] = f;
        }
    }
}
#endif

/* --------------------------------------------------------------------- host */
enum { FC_COUNT_L = 0, FC_COUNT_X, FC_WORK_S, FC_WORK_L, FC_WORK_X, FC_BOUNDS = 8 /* [5]: start of each size class in the sorted list */, FC_HIST = 16, FC__N = FC_HIST + (4u << 11) };
struct clf_ctx {
    int device = 0, n_sm = 1;
    FProg h_prog;
    bool ok = false;
    FProg *d_prog = nullptr;
    uint32_t *d_words = nullptr;           /* FC_* counters */
    uint32_t *d_list[3] = { nullptr, nullptr, nullptr }; size_t list_cap = 0;      /* [0] [1]: overflow lists of classes L, X; [2]: all functions, sorted */
    cl_event *d_mev = nullptr; size_t mev_cap_bytes = 0;
    unsigned launches = 0;
    bool attr_set = false;
};

#if CLF_CUDA
#define F_CUDA_OK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { snprintf(err, errlen, "%s: %s", #x, cudaGetErrorString(e_)); return -1; } } while (0)
static int f_alloc(void **p, size_t n, char *err, size_t errlen) { F_CUDA_OK(cudaMalloc(p, n ? n : 16)); return 0; }
static void f_free(void *p) { if (p) cudaFree(p); }
#else
static int f_alloc(void **p, size_t n, char *err, size_t errlen) { *p = malloc(n ? n : 16); if (!*p) { snprintf(err, errlen, "out of memory"); return -1; } return 0; }
static void f_free(void *p) { free(p); }
#endif

int clf_create(clf_ctx **out, int device, int n_sm) {
    clf_ctx *c = new clf_ctx();
    c->device = device; c->n_sm = n_sm > 0 ? n_sm : 1;
    char err[128];
    void *p = nullptr;
    if (f_alloc(&p, sizeof(FProg), err, sizeof err)) { delete c; return -1; }
    c->d_prog = (FProg *)p;
    if (f_alloc(&p, sizeof(uint32_t) * FC__N, err, sizeof err)) { f_free(c->d_prog); delete c; return -1; }
    c->d_words = (uint32_t *)p;
    *out = c;
    return 0;
}
void clf_destroy(clf_ctx *c) {
    if (!c) return;
    f_free(c->d_prog); f_free(c->d_words); f_free(c->d_list[0]); f_free(c->d_list[1]); f_free(c->d_list[2]); f_free(c->d_mev);
    delete c;
}
int clf_set_patterns(clf_ctx *c, const cl_pattern_blob *blob, void *stream, char *err, size_t errlen) {
    char why[160] = "";
    c->ok = fprog_build(*blob, c->h_prog, why, sizeof why);
    if (getenv("CL_FUSED_DEBUG") && !c->ok) fprintf(stderr, "fused path off: %s\n", why);
#if CLF_CUDA
    F_CUDA_OK(cudaMemcpyAsync(c->d_prog, &c->h_prog, sizeof(FProg), cudaMemcpyHostToDevice, (cudaStream_t)stream));
    F_CUDA_OK(cudaStreamSynchronize((cudaStream_t)stream));
#else
    memcpy(c->d_prog, &c->h_prog, sizeof(FProg));
    (void)stream; (void)err; (void)errlen;
#endif
    return c->ok ? 1 : 0;
}
void clf_info(const clf_ctx *c, unsigned long long out[4]) {
    out[0] = c->launches; out[1] = out[2] = out[3] = 0;
}

#if CLF_CUDA
template <class C, int NW, int NG, int MINB> static int f_launch(clf_ctx *c, const KArgs &k, const FLoop &L, uint32_t grid, cudaStream_t st, char *err, size_t errlen) {
    constexpr size_t smem = f_prog_bytes() + (size_t)NG * f_slice_bytes<C>();
    static_assert((smem + 1024) * MINB <= F_SMEM_MAX + 1024, "the groups of the resident CTAs do not fit the SM's shared memory");
    F_CUDA_OK(cudaFuncSetAttribute(k_fused<C, NW, NG, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_fused<C, NW, NG, MINB><<<grid * MINB, NW * NG * 32, smem, st>>>(k, c->d_prog, L);
    F_CUDA_OK(cudaGetLastError());
    c->launches++;
    return 0;
}
#endif

/* groups per CTA and CTAs per SM of each class */
#ifndef CLF_GROUPS_S
#define CLF_GROUPS_S 13
#define CLF_CTAS_S 1
#endif
#ifndef CLF_GROUPS_L
#define CLF_GROUPS_L 7
#define CLF_CTAS_L 1
#endif
#ifndef CLF_GROUPS_X
#define CLF_GROUPS_X 3
#define CLF_CTAS_X 1
#endif

int clf_run(clf_ctx *c, const KArgs *kp, uint32_t F, void *stream, char *err, size_t errlen) {
    if (!c->ok) { snprintf(err, errlen, "fused path: pattern table not supported"); return -1; }
    KArgs k = *kp;
    c->launches = 0;
    if (c->list_cap < F) {
        for (int i = 0; i < 3; i++) { f_free(c->d_list[i]); c->d_list[i] = nullptr; }
        const size_t want = (size_t)F + F / 16 + 64;
        void *p = nullptr;
        for (int i = 0; i < 3; i++) { if (f_alloc(&p, want * sizeof(uint32_t), err, errlen)) return -1; c->d_list[i] = (uint32_t *)p; }
        c->list_cap = want;
    }
    const bool emit = k.emit_matches || (k.passes & CL_PASS_MATCH_ONLY);
    const uint32_t groups[3] = { (uint32_t)c->n_sm * CLF_GROUPS_S * CLF_CTAS_S, (uint32_t)c->n_sm * CLF_GROUPS_L * CLF_CTAS_L, (uint32_t)c->n_sm * CLF_GROUPS_X * CLF_CTAS_X };
    const uint32_t mcap[3] = { emit ? 12 * FCfgS::M : 0u, emit ? 12 * FCfgL::M : 0u, emit ? 12 * FCfgX::M : 0u };
    {
        size_t need = 0;
        need = std::max(need, groups[0] * f_scratch_bytes<FCfgS>(mcap[0]));
        need = std::max(need, groups[1] * f_scratch_bytes<FCfgL>(mcap[1]));
        need = std::max(need, groups[2] * f_scratch_bytes<FCfgX>(mcap[2]));
        if (c->mev_cap_bytes < need) {
            f_free(c->d_mev); c->d_mev = nullptr;
            void *p = nullptr;
            if (f_alloc(&p, need, err, errlen)) return -1;
            c->d_mev = (cl_event *)p; c->mev_cap_bytes = need;
        }
    }
    FLoop L[3];
    for (int i = 0; i < 3; i++) {
        L[i].list = c->d_list[2];
        L[i].bounds = c->d_words + FC_BOUNDS + i;
        L[i].list2 = i == 0 ? nullptr : c->d_list[i - 1];
        L[i].n_list2_ptr = i == 0 ? nullptr : c->d_words + FC_COUNT_L + (i - 1);
        L[i].counter = c->d_words + FC_WORK_S + i;
        L[i].next_list = i < 2 ? c->d_list[i] : nullptr;
        L[i].next_count = i < 2 ? c->d_words + FC_COUNT_L + i : nullptr;
        L[i].scr = (uint8_t *)c->d_mev;
        L[i].mev_cap = mcap[i];
    }
#if CLF_CUDA
    cudaStream_t st = (cudaStream_t)stream;
    static_assert(FC_HIST + FS_BINS == FC__N, "histogram bins");
    const uint32_t grid = (uint32_t)c->n_sm, sgrid = std::min<uint32_t>((F + 255) / 256, grid * 8);
    k_fused_zero<<<8, 1024, 0, st>>>(c->d_words, FC__N);
    k_fsort_hist<<<sgrid, 256, 0, st>>>(k.in, F, c->d_words + FC_HIST);
    k_fsort_scan<<<1, 1024, 0, st>>>(c->d_words + FC_HIST, c->d_words + FC_BOUNDS);
    k_fsort_scatter<<<sgrid, 256, 0, st>>>(k, F, c->d_words + FC_HIST, c->d_list[2]);
    F_CUDA_OK(cudaGetLastError());
    c->launches += 4;
    if (f_launch<FCfgS, 1, CLF_GROUPS_S, CLF_CTAS_S>(c, k, L[0], grid, st, err, errlen)) return -1;
    if (f_launch<FCfgL, 2, CLF_GROUPS_L, CLF_CTAS_L>(c, k, L[1], grid, st, err, errlen)) return -1;
    if (f_launch<FCfgX, 4, CLF_GROUPS_X, CLF_CTAS_X>(c, k, L[2], grid, st, err, errlen)) return -1;
#else
    (void)stream;
    memset(c->d_words, 0, sizeof(uint32_t) * FC__N);
    {   /* the same counting sort on the host */
        uint32_t *hist = c->d_words + FC_HIST, *bounds = c->d_words + FC_BOUNDS;
        for (uint32_t f = 0; f < F; f++) hist[f_sort_key(k.in, f)]++;
        uint32_t run = 0;
        for (uint32_t b = 0; b < FS_BINS; b++) { const uint32_t n = hist[b]; hist[b] = run; if ((b & ((2u << FS_NBITS) - 1u)) == 0) bounds[b >> (FS_NBITS + 1)] = run; run += n; }
        bounds[4] = run;
        for (uint32_t f = 0; f < F; f++) {
            const uint32_t key = f_sort_key(k.in, f);
            c->d_list[2][hist[key]++] = f;
            if (key >> (FS_NBITS + 1) == 3) {
                const uint32_t n = k.in.blk_off[k.in.func_blk_off[f + 1]] - k.in.blk_off[k.in.func_blk_off[f]];
                if (n > k.small_max) k.retry_big_list[(*k.retry_big_count)++] = f; else k.retry_list[(*k.retry_count)++] = f;
            }
        }
    }
    FEnv e; e.P = c->d_prog; e.a = &k; e.ms = k.in.modsets;
    FG<0> g; g.rank = 0; g.size = 1; g.bar = 0;
    static FCta Q;
    { static FW<FCfgS> W; g.red = W.gred; FCtx<FCfgS> x; x.Q = &Q; x.w0 = (uint8_t *)&W; x.stride = 0; x.ng = 1; x.gi = 0; x.tid = 0; x.nthreads = 1; f_loop(g, W, e, x, L[0], 0); }
    { static FW<FCfgL> W; g.red = W.gred; FCtx<FCfgL> x; x.Q = &Q; x.w0 = (uint8_t *)&W; x.stride = 0; x.ng = 1; x.gi = 0; x.tid = 0; x.nthreads = 1; f_loop(g, W, e, x, L[1], 0); }
    { static FW<FCfgX> W; g.red = W.gred; FCtx<FCfgX> x; x.Q = &Q; x.w0 = (uint8_t *)&W; x.stride = 0; x.ng = 1; x.gi = 0; x.tid = 0; x.nthreads = 1; f_loop(g, W, e, x, L[2], 0); }
    c->launches = 3;
#endif
    return 0;
}
