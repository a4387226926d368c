/* culifter.cu -- C ABI of include/culifter.h on sm_100a.
 *
 * Host side: context, H2D layout, work partition (warp groups for small
 * functions, CTA groups for large ones), launches, D2H + densification.
 * Device side: persistent kernels that pull functions off a work counter and
 * run core.cuh on them with the stream resident in shared memory when it
 * fits (L2-resident scratch otherwise).
 *
 * Compiled with -DCL_SIM by g++ this same file becomes a one-lane CPU build
 * of the *device code* (cudaMalloc -> malloc, launch -> loop).  That build is
 * debugging / CI infrastructure under tests/sim only: the package never
 * loads it and there is no CPU fallback in the product path.
 */
#include "core.cuh"
#include "tile.cuh"
#include "kargs.h"
#include "fused.h"

#include <algorithm>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#if CL_DEV || (defined(__CUDACC__) && !defined(CL_SIM))
#include <cuda_runtime.h>
#define CL_CUDA 1
#else
#define CL_CUDA 0
#endif

using namespace clk;

static thread_local char g_err[512];
extern "C" const char *cl_last_error(void) { return g_err; }
extern "C" const char *cl_backend(void) { return CL_CUDA ? "cuda-sm_100a" : "sim-device-code"; }
#define FAIL(...) do { snprintf(g_err, sizeof g_err, __VA_ARGS__); return -1; } while (0)

extern "C" long cl_abi_sizeof(int which) {
    static const long sz[] = { sizeof(cl_hdr), sizeof(cl_imm), sizeof(cl_memref), sizeof(cl_blk),
        sizeof(cl_func), sizeof(cl_modset), sizeof(cl_slot), sizeof(cl_template), sizeof(cl_pattern),
        sizeof(cl_pattern_blob), sizeof(cl_event), sizeof(cl_corpus), sizeof(cl_run_opts),
        sizeof(cl_stats), sizeof(cl_sr_entry) };
    return which >= 0 && which < (int)(sizeof sz / sizeof *sz) ? sz[which] : -1;
}

/* ------------------------------------------------------- device memory shim */
#if CL_CUDA
#define CUDA_OK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) FAIL("%s: %s", #x, cudaGetErrorString(e_)); } while (0)
static int dmalloc(void **p, size_t n) { CUDA_OK(cudaMalloc(p, n ? n : 16)); return 0; }
static void dfree(void *p) { if (p) cudaFree(p); }
static int h2d(void *d, const void *h, size_t n, cudaStream_t st) { if (n) CUDA_OK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st)); return 0; }
static int d2h(void *h, const void *d, size_t n, cudaStream_t st) { if (n) CUDA_OK(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st)); return 0; }
/* Zeroing as a kernel, not cudaMemsetAsync: the driver may hand a memset to a copy engine, where the few words a
 * run clears queue behind another context's bulk D2H / H2D (measured in the chunked pipeline: +13 ms on every
 * run that started while a neighbour's download was in flight).                                             */
static thread_local unsigned g_aux_launches = 0;      /* zeroing / densify kernels launched by this thread since the run began */
__global__ void k_zero(uint32_t *p, size_t n_words) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_words; i += (size_t)gridDim.x * blockDim.x) p[i] = 0;
}
static int dzero(void *d, size_t n, cudaStream_t st) {
    if (!n) return 0;
    if (n % 4 == 0 && (uintptr_t)d % 4 == 0) {
        const size_t w = n / 4;
        k_zero<<<(unsigned)std::min<size_t>((w + 255) / 256, 1184), 256, 0, st>>>((uint32_t *)d, w);
        CUDA_OK(cudaGetLastError());
        g_aux_launches++;
    } else
        CUDA_OK(cudaMemsetAsync(d, 0, n, st));
    return 0;
}
#else
typedef int cudaStream_t;
static int dmalloc(void **p, size_t n) { *p = malloc(n ? n : 16); if (!*p) FAIL("out of memory"); return 0; }
static void dfree(void *p) { free(p); }
static int h2d(void *d, const void *h, size_t n, cudaStream_t) { if (n) memcpy(d, h, n); return 0; }
static int d2h(void *h, const void *d, size_t n, cudaStream_t) { if (n) memcpy(h, d, n); return 0; }
static int dzero(void *d, size_t n, cudaStream_t) { if (n) memset(d, 0, n); return 0; }
#endif

static const uint8_t H_OPFLAGS[] = {
#define CL_OP(name, flags) (uint8_t)(flags),
#include "../../include/culifter_ops.h"
#undef CL_OP
};

/* ------------------------------------------------------ work memory layout */
template <class T> CLHD T *carve(uint8_t *&p, size_t n) {
    T *r = (T *)p;
    p += (n * sizeof(T) + 15) & ~(size_t)15;
    return r;
}
/* hot arrays: the stream planes and the two per-value arrays every pass hits */
CLHD size_t hot_size(uint32_t I, uint32_t V) {
    return (size_t)I * 64 + (((size_t)V * 4 + 15) & ~(size_t)15) * 2;
}
CLHD void carve_hot(FS &s, uint8_t *p, uint32_t I, uint32_t V) {
    s.S.hdr = carve<cl_hdr>(p, I);
    s.S.tag = carve<uint16_t>(p, (size_t)I * 8);
    s.S.pay = carve<uint32_t>(p, (size_t)I * 8);
    s.usecnt = carve<uint32_t>(p, V);
    s.defpos = carve<uint32_t>(p, V);
}
/* everything else (and the hot arrays too when `hot` is null); returns bytes */
CLHD size_t carve_cold(FS &s, uint8_t *base, const Caps &c, bool with_hot) {
    uint8_t *p = base;
    if (with_hot) { carve_hot(s, p, c.I, c.V); p += hot_size(c.I, c.V); }
    s.bo = carve<uint32_t>(p, c.B + 1);
    s.bo2 = carve<uint32_t>(p, c.B + 1);
    s.blk_sel = carve<uint32_t>(p, c.B + 1);
    s.blk = carve<cl_blk>(p, c.B);
    s.alive = carve<uint8_t>(p, c.V);
    s.def_iid = carve<int32_t>(p, c.V);
    s.origin = carve<uint32_t>(p, c.V);
    s.redirect = carve<uint32_t>(p, c.V + 1);
    s.xhead = carve<uint32_t>(p, c.V);
    s.root = carve<uint32_t>(p, c.V);
    s.keep = carve<uint8_t>(p, c.I);
    s.inscnt = carve<uint8_t>(p, c.I);
    s.clsid = carve<uint8_t>(p, c.I);
    s.outpos = carve<uint32_t>(p, c.I);
    s.cidx = s.outpos;
    s.cand = carve<uint32_t>(p, c.I);
    s.sel_at = carve<uint32_t>(p, c.I);
    s.owner = carve<unsigned long long>(p, c.I);
    s.mt = carve<MatchRec>(p, c.M);
    s.sel = carve<SelRec>(p, c.S);
    s.stage = carve<Stage>(p, c.S);
    s.imm = carve<cl_imm>(p, c.Q);
    s.ev = carve<cl_event>(p, c.E);
    s.site = carve<uint32_t>(p, c.U);
    s.xr = carve<XRec>(p, c.X);
    return (size_t)(p - base);
}
static size_t scratch_bytes(const Caps &c) {
    FS tmp;
    return carve_cold(tmp, (uint8_t *)0, c, true) + 256;
}

/* group-shared words (shared memory on the device)                          */
enum { GW_STATUS = 0, GW_NEV, GW_WORK, GW_STATS, GW__N = GW_STATS + 64 };

/* ------------------------------------------------------------ load / store */
template <class G> CLF void load_function(const G &g, FS &s, const KArgs &a, uint32_t f) {
    PROF(g, s, PF_LOAD);
    const cl_corpus &in = a.in;
    const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
    const uint32_t i0 = in.blk_off[b0], i1 = in.blk_off[b1];
    const cl_func fn = in.func[f];
    s.f = f; s.arch = fn.arch;
    s.nb = b1 - b0; s.n = i1 - i0;
    s.next_vid = fn.next_vid; s.next_iid = fn.next_iid; s.next_temp = fn.next_temp_reg;
    if (g.rank == 0) { *s.st = 0; *s.n_ev = 0; }
    GFOR(g, b, s.nb + 1) if (b <= s.nb) s.bo[b] = in.blk_off[b0 + b] - i0;
    GFOR(g, b, s.nb) if (b < s.nb) s.blk[b] = in.blk[b0 + b];
    /* coalesced 128-bit loads of the three planes */
    {
        const uint4 *src = (const uint4 *)(in.hdr + i0);
        uint4 *dst = (uint4 *)s.S.hdr;
        GFOR(g, i, s.n) if (i < s.n) dst[i] = src[i];
        const uint4 *st = (const uint4 *)(in.tag + (size_t)i0 * 8);
        uint4 *dt = (uint4 *)s.S.tag;
        GFOR(g, i, s.n) if (i < s.n) dt[i] = st[i];
        const uint4 *sp = (const uint4 *)(in.pay + (size_t)i0 * 8);
        uint4 *dp = (uint4 *)s.S.pay;
        GFOR(g, i, 2 * s.n) if (i < 2 * s.n) dp[i] = sp[i];
    }
    const uint32_t v0 = in.val_off[f], nv_in = in.val_off[f + 1] - v0;
    GFOR(g, v, s.next_vid) if (v < s.next_vid) {
        s.alive[v] = v < nv_in ? in.val_alive[v0 + v] : 0;
        s.def_iid[v] = v < nv_in ? in.val_def_iid[v0 + v] : -1;
        s.origin[v] = CL_ORG_HOST;
    }
    const uint32_t q0 = in.imm_off[f];
    s.n_imm = in.imm_off[f + 1] - q0;
    GFOR(g, q, s.n_imm) if (q < s.n_imm) s.imm[q] = in.imm[q0 + q];
    const uint32_t e0 = in.ext_off[f];
    s.n_ext = in.ext_off[f + 1] - e0;
    s.ext_tag = a.o_ext_tag + e0; s.ext_pay = a.o_ext_pay + e0;
    GFOR(g, e, s.n_ext) if (e < s.n_ext) { s.ext_tag[e] = in.ext_tag[e0 + e]; s.ext_pay[e] = in.ext_pay[e0 + e]; }
    const uint32_t m0 = in.mem_off[f];
    s.n_mem = in.mem_off[f + 1] - m0;
    s.mem = a.o_mem + m0;
    GFOR(g, m, s.n_mem) if (m < s.n_mem) s.mem[m] = in.mem[m0 + m];
    g.sync();
}

CLD uint32_t events_of(const FS &s) { return *s.n_ev <= s.cap.E ? *s.n_ev : s.cap.E; }

/* copy a finished function to the places reserved for it */
template <class G> CLF void store_function_at(const G &g, FS &s, const KArgs &a, uint32_t f, uint32_t r_inst,
                                              uint32_t r_imm, uint32_t r_val, uint32_t r_ev);

template <class G> CLF void store_function(const G &g, FS &s, const KArgs &a, uint32_t f) {
    const uint32_t n_ev = events_of(s);
    uint32_t r_inst = 0, r_imm = 0, r_val = 0, r_ev = 0;
    if (g.rank == 0) {
        r_inst = (uint32_t)a_add64(&a.cursor[CUR_INST], s.n);
        r_imm = (uint32_t)a_add64(&a.cursor[CUR_IMM], s.n_imm);
        r_val = (uint32_t)a_add64(&a.cursor[CUR_VAL], s.next_vid);
        r_ev = (uint32_t)a_add64(&a.cursor[CUR_EV], n_ev);
    }
    r_inst = g.bcast0(r_inst); r_imm = g.bcast0(r_imm); r_val = g.bcast0(r_val); r_ev = g.bcast0(r_ev);
    store_function_at(g, s, a, f, r_inst, r_imm, r_val, r_ev);
}

template <class G> CLF void store_function_at(const G &g, FS &s, const KArgs &a, uint32_t f, uint32_t r_inst,
                                              uint32_t r_imm, uint32_t r_val, uint32_t r_ev) {
    PROF(g, s, PF_STORE);
    const uint32_t st = status(s);
    const uint32_t n_ev = events_of(s);
    const bool fits = (unsigned long long)r_inst + s.n <= a.cap[CUR_INST] && (unsigned long long)r_imm + s.n_imm <= a.cap[CUR_IMM] &&
                      (unsigned long long)r_val + s.next_vid <= a.cap[CUR_VAL] && (unsigned long long)r_ev + n_ev <= a.cap[CUR_EV];
    const uint32_t b0 = a.in.func_blk_off[f];
    if (g.rank == 0) {
        FuncOut o;
        o.f.next_vid = s.next_vid; o.f.next_iid = s.next_iid; o.f.next_temp_reg = s.next_temp;
        o.f.arch = (uint8_t)s.arch; o.f.status = (uint8_t)(fits ? st : (uint32_t)CL_ST_CAPACITY); o.f.reserved = 0;
        o.inst_start = r_inst; o.n_inst = fits ? s.n : 0; o.imm_start = r_imm; o.n_imm = fits ? s.n_imm : 0;
        o.val_start = r_val; o.ev_start = r_ev; o.n_ev = fits ? n_ev : 0; o.pad = 0;
        a.o_func[f] = o;
    }
    if (!fits) {
        GFOR(g, b, s.nb) if (b < s.nb) { a.o_blk[b0 + b] = s.blk[b]; a.o_blk_start[b0 + b] = 0; a.o_blk_cnt[b0 + b] = 0; }
        return;
    }
    GFOR(g, b, s.nb) if (b < s.nb) {
        a.o_blk[b0 + b] = s.blk[b];
        a.o_blk_start[b0 + b] = r_inst + s.bo[b];
        a.o_blk_cnt[b0 + b] = s.bo[b + 1] - s.bo[b];
    }
    {
        uint4 *dh = (uint4 *)(a.o_hdr + r_inst);
        const uint4 *sh = (const uint4 *)s.S.hdr;
        GFOR(g, i, s.n) if (i < s.n) dh[i] = sh[i];
        uint4 *dt = (uint4 *)(a.o_tag + (size_t)r_inst * 8);
        const uint4 *stg = (const uint4 *)s.S.tag;
        GFOR(g, i, s.n) if (i < s.n) dt[i] = stg[i];
        uint4 *dp = (uint4 *)(a.o_pay + (size_t)r_inst * 8);
        const uint4 *sp = (const uint4 *)s.S.pay;
        GFOR(g, i, 2 * s.n) if (i < 2 * s.n) dp[i] = sp[i];
    }
    GFOR(g, q, s.n_imm) if (q < s.n_imm) a.o_imm[r_imm + q] = s.imm[q];
    GFOR(g, v, s.next_vid) if (v < s.next_vid) {
        a.o_alive[r_val + v] = s.alive[v]; a.o_def_iid[r_val + v] = s.def_iid[v]; a.o_origin[r_val + v] = s.origin[v];
    }
    GFOR(g, e, n_ev) if (e < n_ev) a.o_ev[r_ev + e] = s.ev[e];
}

/* one function through the passes on one group; false = queued for the roomy kernel */
template <class G> CLF bool compute_function(const G &g, FS &s, const KArgs &a, uint32_t f, uint8_t *hot,
                                             uint8_t *cold) {
    const cl_corpus &in = a.in;
    const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
    const uint32_t n_in = in.blk_off[b1] - in.blk_off[b0];
    const uint32_t nv_in = in.func[f].next_vid;
    /* placement: hot arrays in shared memory when a 1.5x stream fits */
    Caps tight = a.gcap;
    tight.I = n_in + n_in / 2 + 16;
    tight.V = nv_in + n_in + 16;
    bool use_hot = hot != nullptr && hot_size(tight.I, tight.V) <= a.hot_bytes && tight.I <= a.gcap.I && tight.V <= a.gcap.V;
    for (int attempt = 0; attempt < 2; attempt++) {
        /* slab = [hot arrays at scratch capacity][everything else]; the shared-memory
         * placement only moves the hot arrays and tightens their capacities        */
        carve_cold(s, cold, a.gcap, true);
        s.cap = a.gcap;
        if (use_hot) { carve_hot(s, hot, tight.I, tight.V); s.cap.I = tight.I; s.cap.V = tight.V; }
        load_function(g, s, a, f);
        if (a.raw_passes) run_raw(g, s, a.raw_passes, a.sr, a.n_sr);
        else if (a.passes & CL_PASS_MATCH_ONLY) run_match_only(g, s);
        else run_postssa(g, s);
        g.sync();
        if (status(s) == CL_ST_CAPACITY && use_hot) { use_hot = false; g.sync(); continue; }
        break;
    }
    if (status(s) == CL_ST_CAPACITY && a.retry_list) {
        if (g.rank == 0) a.retry_list[a_add(a.retry_count, 1u)] = f;
        g.sync();
        return false;
    }
    if (status(s) != CL_ST_OK) {              /* hand the function back unchanged */
        const uint32_t code = status(s);
        g.sync();
        carve_cold(s, cold, a.gcap, true);
        s.cap = a.gcap;
        load_function(g, s, a, f);
        if (g.rank == 0) *s.st = code;
        g.sync();
    }
    return true;
}
template <class G> CLF bool process_function(const G &g, FS &s, const KArgs &a, uint32_t f, uint8_t *hot,
                                             uint8_t *cold) {
    if (!compute_function(g, s, a, f, hot, cold)) return false;
    store_function(g, s, a, f);
    g.sync();
    return true;
}

CLD void setup_fs(FS &s, const KArgs &a, uint32_t *gw, unsigned long long *prof, bool solo) {
    s.pb = a.pb; s.ms = a.in.modsets; s.opflags = a.opflags; s.solo = solo;
    s.passes = a.passes; s.max_rounds = a.max_rounds; s.emit_matches = a.emit_matches;
    s.st = gw + GW_STATUS; s.n_ev = gw + GW_NEV;
    s.st_matches = gw + GW_STATS; s.st_selected = gw + GW_STATS + 16;
    s.st_rewrites = gw + GW_STATS + 32; s.st_refused = gw + GW_STATS + 48;
    s.prof = prof;
}

/* persistent group loop                                                      */
template <class G> CLF void group_loop(const G &g, const KArgs &a, uint32_t *gw, uint8_t *hot, uint8_t *cold) {
    FS s;
    unsigned long long prof[PF__N];
    for (int k = 0; k < PF__N; k++) prof[k] = 0;
    const unsigned long long t_begin = now();
    setup_fs(s, a, gw, prof, g.size == 1);
    GFOR(g, k, GW__N) if (k < GW__N) gw[k] = 0;
    g.sync();
    const uint32_t n_list = a.n_list_ptr ? *a.n_list_ptr : a.n_list;
    unsigned long long n_in = 0, n_out = 0, n_ev = 0;
    for (;;) {
        uint32_t w = 0;
        if (g.rank == 0) w = a_add(a.work_counter, 1u);
        w = g.bcast0(w);
        if (w >= n_list) break;
        const uint32_t f = a.list[w];
        uint32_t saved[64];
        if (a.retry_list && g.rank == 0) for (int k = 0; k < 64; k++) saved[k] = gw[GW_STATS + k];
        if (!process_function(g, s, a, f, hot, cold)) {       /* queued: its counters will be redone */
            if (g.rank == 0) for (int k = 0; k < 64; k++) gw[GW_STATS + k] = saved[k];
            g.sync();
            continue;
        }
        const uint32_t b0 = a.in.func_blk_off[f], b1 = a.in.func_blk_off[f + 1];
        n_in += a.in.blk_off[b1] - a.in.blk_off[b0];
        n_out += s.n; n_ev += *s.n_ev;
        g.sync();
    }
    if (g.rank == 0) {
        prof[PF_TOTAL] = now() - t_begin;
        for (int k = 0; k < PF__N; k++) a_add64(&a.prof[k], prof[k]);
        for (int k = 0; k < 64; k++) if (gw[GW_STATS + k]) a_add64(&a.stats[k], gw[GW_STATS + k]);
        a_add64(&a.stats[64], n_in); a_add64(&a.stats[65], n_out); a_add64(&a.stats[66], n_ev);
    }
}

#ifndef CL_CTA_CTAS_PER_SM
#define CL_CTA_CTAS_PER_SM 8
#endif
#if CL_CUDA
/* Phase-synchronous warp-group kernel (the general per-function fallback for small functions).  ncu on the free-running
 * kernel shows 89 % of the warp cycles stalled on instruction fetch: the stage
 * is ~300 KB of straight code and 64 warps per SM, each in a different phase of
 * a different function, thrash the instruction cache.  Here the warps of a CTA
 * take one function each and walk through the passes in lock step (CTA barrier
 * between passes), so an SM runs one pass's code at a time and the warps share
 * it in the instruction cache.  Functions of a batch have similar sizes (the
 * work list is sorted), so little time is lost at the barriers.             */
template <int WARPS, int MINB> __global__ void __launch_bounds__(WARPS * 32, MINB) k_postssa_warp_sync(KArgs a) {
    __shared__ uint32_t gw[WARPS][GW__N];
    const uint32_t w = threadIdx.x >> 5;
    Grp<1> g; g.rank = threadIdx.x & 31u; g.size = 32; g.red = nullptr;
    const uint32_t gid = blockIdx.x * WARPS + w;
    uint8_t *cold = a.scratch + (size_t)gid * a.scratch_per_group;
    FS s;
    unsigned long long prof[PF__N];
    for (int k = 0; k < PF__N; k++) prof[k] = 0;
    const unsigned long long t_begin = now();
    setup_fs(s, a, gw[w], prof, false);
    GFOR(g, k, GW__N) if (k < GW__N) gw[w][k] = 0;
    g.sync();
    const uint32_t n_list = a.n_list_ptr ? *a.n_list_ptr : a.n_list;
    unsigned long long n_in = 0, n_out = 0, n_ev = 0;
    for (;;) {
        uint32_t wi = 0;
        if (g.rank == 0) wi = a_add(a.work_counter, 1u);
        wi = g.bcast0(wi);
        const bool live = wi < n_list;
        if (!__syncthreads_or(live)) break;
        uint32_t f = 0;
        if (live) {
            f = a.list[wi];
            carve_cold(s, cold, a.gcap, true);
            s.cap = a.gcap;
            load_function(g, s, a, f);
        }
        __syncthreads();
        if (a.raw_passes) { if (live) run_raw(g, s, a.raw_passes, a.sr, a.n_sr); }
        else if (a.passes & CL_PASS_MATCH_ONLY) { if (live) run_match_only(g, s); }
        else {
            /* every pass below is cut into pieces of one code region each; the whole CTA
             * finishes a piece before anyone starts the next                             */
            const bool xm = live && (s.passes & CL_PASS_XMAD) && s.arch == CL_ARCH_SM52;
            if (__syncthreads_or(xm)) {
                uint32_t nsel = 0;
                if (xm) ap_prepare(g, s, 1);
                __syncthreads();
                if (xm && !status(s)) nsel = ap_match(g, s, 1, 0);
                __syncthreads();
                if (xm && !status(s) && nsel) ap_rewrite(g, s, 0);
                __syncthreads();
                if (xm && !status(s)) remove_dead_pseudo(g, s);
                __syncthreads();
            }
            if (live && (s.passes & CL_PASS_RECIPROCAL) && !status(s)) normalize_reciprocal(g, s);
            __syncthreads();
            bool more = live && (s.passes & CL_PASS_AGGREGATE);
            for (uint32_t round = 0; round < a.max_rounds; round++) {
                uint32_t n = 0, nsel = 0, red = 0;
                if (more && !status(s)) ap_prepare(g, s, 0);
                __syncthreads();
                if (more && !status(s)) nsel = ap_match(g, s, 0, 2 + round);
                __syncthreads();
                if (more && !status(s) && nsel) n = ap_rewrite(g, s, 2 + round);
                __syncthreads();
                if (more && !status(s)) red = simplify_packs(g, s, false);
                __syncthreads();
                if (more && !status(s) && red) remove_dead_pseudo(g, s);
                n += red;
                if (!n) more = false;
                if (!__syncthreads_or(more)) break;
            }
            if (live && (s.passes & CL_PASS_AGGREGATE) && !status(s)) remove_dead_pseudo(g, s);
            __syncthreads();
            if (live && (s.passes & CL_PASS_TAG) && !status(s)) tag_cuda_objects(g, s);
        }
        __syncthreads();
        if (live) {
            g.sync();
            if (status(s) != CL_ST_OK) {              /* hand the function back unchanged */
                const uint32_t code = status(s);
                g.sync();
                load_function(g, s, a, f);
                if (g.rank == 0) *s.st = code;
                g.sync();
            }
            store_function(g, s, a, f);
            const uint32_t b0 = a.in.func_blk_off[f], b1 = a.in.func_blk_off[f + 1];
            n_in += a.in.blk_off[b1] - a.in.blk_off[b0];
            n_out += s.n; n_ev += *s.n_ev;
        }
        __syncthreads();
    }
    if (g.rank == 0) {
        prof[PF_TOTAL] = now() - t_begin;
        for (int k = 0; k < PF__N; k++) a_add64(&a.prof[k], prof[k]);
        for (int k = 0; k < 64; k++) if (gw[w][GW_STATS + k]) a_add64(&a.stats[k], gw[w][GW_STATS + k]);
        a_add64(&a.stats[64], n_in); a_add64(&a.stats[65], n_out); a_add64(&a.stats[66], n_ev);
    }
}

/* one CTA per function                                                       */
template <int WARPS, int MINB> __global__ void __launch_bounds__(WARPS * 32, MINB) k_postssa_cta(KArgs a) {
    extern __shared__ uint4 dyn_smem[];
    __shared__ uint32_t gw[GW__N];
    __shared__ uint32_t red[WARPS + 2];
    Grp<WARPS> g; g.rank = threadIdx.x; g.size = WARPS * 32; g.red = red;
    uint8_t *hot = a.hot_bytes ? (uint8_t *)dyn_smem : nullptr;
    group_loop(g, a, gw, hot, a.scratch + (size_t)blockIdx.x * a.scratch_per_group);
}
#endif


/* ------------------------------------------------------------- tile kernel */
/* one CTA = one tile of consecutive small functions resident in shared memory
 * (tile.cuh); persistent CTAs pull tiles off a counter                       */
static_assert(sizeof(TFuncOut) == sizeof(FuncOut), "TFuncOut mirrors FuncOut");
template <class C> CLHD size_t tile_scratch_bytes() {
    return ((sizeof(Stage) * C::S + 255) & ~(size_t)255) + ((sizeof(cl_event) * C::E + 255) & ~(size_t)255);
}
CLHD TileIO tile_io(const KArgs &a) {
    TileIO io;
    io.in = a.in;
    io.o_hdr = a.o_hdr; io.o_tag = a.o_tag; io.o_pay = a.o_pay; io.o_imm = a.o_imm;
    io.o_alive = a.o_alive; io.o_def_iid = a.o_def_iid; io.o_origin = a.o_origin; io.o_mem = a.o_mem;
    io.o_blk = a.o_blk; io.o_blk_start = a.o_blk_start; io.o_blk_cnt = a.o_blk_cnt;
    io.o_ev = a.o_ev; io.o_func = a.o_func;
    for (int k = 0; k < 4; k++) io.cap[k] = a.cap[k];
    io.cursor = a.cursor; io.stats = a.stats;
    io.retry_list = a.retry_list; io.retry_count = a.retry_count;
    io.retry_big_list = a.retry_big_list; io.retry_big_count = a.retry_big_count; io.small_max = a.small_max;
    io.flist = a.tile_flist;
    return io;
}
/* persistent loop of one group (a warp or a CTA) over the tiles of its size class */
template <class G, class C> CLF void tile_loop(const G &g, TileS<C> &T, const TileP &P, const KArgs &a, uint32_t group, uint8_t *planes = nullptr) {
    const unsigned long long t_begin = now();
    if (g.rank == 0) {
        FS &s = T.fs;
        memset(&s, 0, sizeof s);
        T.P = &P;
        s.pb = &P.pb; s.ms = a.in.modsets; s.opflags = a.opflags; s.solo = g.size == 1;
        s.passes = a.passes; s.max_rounds = a.max_rounds; s.emit_matches = 0;
        if constexpr (C::PP) {       /* big tiles: two buffers per plane in scratch (128 bytes per record) */
            T.hdr.a = (cl_hdr *)planes; T.hdr.b = (cl_hdr *)(planes + (size_t)16 * C::I);
            T.tag.a = (uint16_t *)(planes + (size_t)32 * C::I); T.tag.b = (uint16_t *)(planes + (size_t)48 * C::I);
            T.pay.a = (uint32_t *)(planes + (size_t)64 * C::I); T.pay.b = (uint32_t *)(planes + (size_t)96 * C::I);
            T.fidx.a = planes + (size_t)128 * C::I; T.fidx.b = planes + (size_t)129 * C::I;
            T.bidx.a = planes + (size_t)130 * C::I; T.bidx.b = planes + (size_t)131 * C::I;
        }
        s.S.hdr = T.hdr.ptr(); s.S.tag = T.tag.ptr(); s.S.pay = T.pay.ptr();
        s.usecnt = T.usecnt; s.defpos = T.defpos; s.redirect = T.redirect; s.origin = T.origin;
        s.def_iid = T.def_iid; s.alive = T.alive; s.imm = T.imm;
        s.cap.I = C::I; s.cap.V = C::V; s.cap.Q = C::Q; s.cap.B = C::B; s.cap.M = C::M; s.cap.S = C::S; s.cap.E = C::E;
        s.st = &T.fail; s.n_ev = &T.n_ev;
        s.prof = T.prof;
        for (int k = 0; k < PF__N; k++) T.prof[k] = 0;
    }
    g.sync();
    TileG<C> tg;
    uint8_t *scr = a.tile_scratch + (size_t)group * a.tile_scratch_per_cta;
    tg.stage = (Stage *)scr;
    tg.ev = (cl_event *)(scr + ((sizeof(Stage) * C::S + 255) & ~(size_t)255));
    tg.mem = a.o_mem;
    tg.tmp = nullptr;
    const TileIO io = tile_io(a);
    for (;;) {
        uint32_t w = 0;
        if (g.rank == 0) w = a_add(a.tile_counter, 1u);
        w = g.bcast0(w);
        if (w >= a.n_tiles) break;
        t_run_tile(g, T, tg, io, a.tiles[w]);
        g.sync();
    }
    if (g.rank == 0) {
        T.prof[PF_TOTAL] = now() - t_begin;
        for (int k = 0; k < PF__N; k++) a_add64(&a.prof[k], T.prof[k]);
    }
}
CLHD size_t tile_p_bytes() { return (sizeof(TileP) + 255) & ~(size_t)255; }
#if CL_CUDA
/* a CTA is one group */
template <class C, int NW, int MINB> __global__ void __launch_bounds__(NW * 32, MINB) k_postssa_tile(KArgs a) {
    extern __shared__ uint4 dyn_smem[];
    TileP &P = *(TileP *)dyn_smem;
    TileS<C> &T = *(TileS<C> *)((uint8_t *)dyn_smem + tile_p_bytes());
    Grp<NW> g; g.rank = threadIdx.x; g.size = NW * 32; g.red = T.red;
    t_setup(g, P, a.pb);
    tile_loop(g, T, P, a, blockIdx.x);
}
/* big tiles resident in L2 (global scratch): a CTA is one group; scratch = stages, events, the tile, a second stream buffer */
template <class C> CLHD size_t gtile_scratch_bytes() {
    return tile_scratch_bytes<C>() + ((sizeof(TileS<C>) + 255) & ~(size_t)255) + (((size_t)132 * C::I + 255) & ~(size_t)255);
}
template <class C, int NW, int MINB> __global__ void __launch_bounds__(NW * 32, MINB) k_postssa_gtile(KArgs a) {
    __shared__ TileP P;
    uint8_t *base = a.tile_scratch + (size_t)blockIdx.x * a.tile_scratch_per_cta;
    TileS<C> &T = *(TileS<C> *)(base + tile_scratch_bytes<C>());
    Grp<NW> g; g.rank = threadIdx.x; g.size = NW * 32; g.red = T.red;
    __shared__ uint32_t red[40];
    g.red = red;
    t_setup(g, P, a.pb);
    tile_loop(g, T, P, a, blockIdx.x, base + tile_scratch_bytes<C>() + ((sizeof(TileS<C>) + 255) & ~(size_t)255));
}
#endif


/* ------------------------------------------------------- densification */
/* The run leaves every function's result at an atomically reserved place
 * (completion order).  cl_download turns that into the dense CSR of the ABI
 * on the device: 4-way exclusive scan of the per-function sizes in function
 * order, then one warp per function copies its pieces to their final place. */
struct DenseArgs {
    const FuncOut *fo; uint32_t n_funcs;
    uint4 *off;                /* [n_funcs + 1] x {inst, imm, val, ev} exclusive  */
    uint4 *block_sums; uint32_t n_scan_blocks;
    const uint32_t *func_blk_off; const uint32_t *blk_start, *blk_cnt;
    const cl_hdr *s_hdr; const uint16_t *s_tag; const uint32_t *s_pay; const cl_imm *s_imm;
    const uint8_t *s_alive; const int32_t *s_def_iid; const uint32_t *s_origin; const cl_event *s_ev;
    cl_hdr *d_hdr; uint16_t *d_tag; uint32_t *d_pay; cl_imm *d_imm;
    uint8_t *d_alive; int32_t *d_def_iid; uint32_t *d_origin; cl_event *d_ev;
    uint32_t *d_blk_off;       /* [n_blocks + 1]                                   */
    uint32_t *d_imm_off, *d_val_off;   /* [n_funcs + 1]                            */
    cl_func *d_func;
    uint32_t n_blocks;
};
#if CL_CUDA
static constexpr int SCAN_T = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_T * SCAN_ITEMS;
__device__ __forceinline__ uint4 add4(uint4 a, uint4 b) { return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ uint4 sizes_of(const DenseArgs &a, uint32_t f) {
    if (f >= a.n_funcs) return make_uint4(0, 0, 0, 0);
    const FuncOut o = a.fo[f];
    return make_uint4(o.n_inst, o.n_imm, o.f.next_vid, o.n_ev);
}
__device__ uint4 block_exscan4(uint4 v, uint4 &total) {
    __shared__ uint4 ws[SCAN_T / 32];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint4 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint4 t = make_uint4(__shfl_up_sync(~0u, inc.x, d), __shfl_up_sync(~0u, inc.y, d), __shfl_up_sync(~0u, inc.z, d), __shfl_up_sync(~0u, inc.w, d));
        if (lane >= (uint32_t)d) inc = add4(inc, t);
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    uint4 pre = make_uint4(0, 0, 0, 0), tot = pre;
    for (int i = 0; i < SCAN_T / 32; i++) { if ((uint32_t)i < w) pre = add4(pre, ws[i]); tot = add4(tot, ws[i]); }
    __syncthreads();
    total = tot;
    return make_uint4(pre.x + inc.x - v.x, pre.y + inc.y - v.y, pre.z + inc.z - v.z, pre.w + inc.w - v.w);
}
__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(DenseArgs a) {       /* pass 1: tile sums */
    uint4 sum = make_uint4(0, 0, 0, 0);
    const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    for (int i = 0; i < SCAN_ITEMS; i++) sum = add4(sum, sizes_of(a, base + i));
    uint4 tot;
    block_exscan4(sum, tot);
    if (threadIdx.x == 0) a.block_sums[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(SCAN_T) k_scan_sums(DenseArgs a) {        /* pass 2: one CTA */
    uint4 run = make_uint4(0, 0, 0, 0);
    for (uint32_t b0 = 0; b0 < a.n_scan_blocks; b0 += SCAN_T) {
        const uint32_t i = b0 + threadIdx.x;
        uint4 v = i < a.n_scan_blocks ? a.block_sums[i] : make_uint4(0, 0, 0, 0), tot;
        uint4 ex = block_exscan4(v, tot);
        if (i < a.n_scan_blocks) a.block_sums[i] = add4(run, ex);
        run = add4(run, tot);
    }
    if (threadIdx.x == 0) a.off[a.n_funcs] = run;
}
__global__ void __launch_bounds__(SCAN_T) k_scan_apply(DenseArgs a) {       /* pass 3 */
    const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    uint4 v[SCAN_ITEMS], sum = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < SCAN_ITEMS; i++) { v[i] = sizes_of(a, base + i); sum = add4(sum, v[i]); }
    uint4 tot;
    uint4 run = add4(block_exscan4(sum, tot), a.block_sums[blockIdx.x]);
    for (int i = 0; i < SCAN_ITEMS; i++) {
        if (base + i < a.n_funcs) a.off[base + i] = run;
        run = add4(run, v[i]);
    }
}
/* one warp per function */
__global__ void __launch_bounds__(256) k_densify(DenseArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t f = blockIdx.x * 8 + (threadIdx.x >> 5); f < a.n_funcs; f += gridDim.x * 8) {
        const FuncOut o = a.fo[f];
        const uint4 off = a.off[f];
        if (lane == 0) { a.d_func[f] = o.f; a.d_imm_off[f] = off.y; a.d_val_off[f] = off.z; }
        const uint32_t b0 = a.func_blk_off[f], b1 = a.func_blk_off[f + 1];
        for (uint32_t b = b0 + lane; b < b1; b += 32)
            a.d_blk_off[b] = off.x + (o.n_inst ? a.blk_start[b] - o.inst_start : 0u);
        const uint4 *sh = (const uint4 *)(a.s_hdr + o.inst_start); uint4 *dh = (uint4 *)(a.d_hdr + off.x);
        const uint4 *st = (const uint4 *)(a.s_tag + (size_t)o.inst_start * 8); uint4 *dt = (uint4 *)(a.d_tag + (size_t)off.x * 8);
        const uint4 *sp = (const uint4 *)(a.s_pay + (size_t)o.inst_start * 8); uint4 *dp = (uint4 *)(a.d_pay + (size_t)off.x * 8);
        for (uint32_t i = lane; i < o.n_inst; i += 32) { dh[i] = sh[i]; dt[i] = st[i]; }
        for (uint32_t i = lane; i < 2 * o.n_inst; i += 32) dp[i] = sp[i];
        for (uint32_t i = lane; i < o.n_imm; i += 32) a.d_imm[off.y + i] = a.s_imm[o.imm_start + i];
        for (uint32_t i = lane; i < o.f.next_vid; i += 32) {
            a.d_alive[off.z + i] = a.s_alive[o.val_start + i];
            a.d_def_iid[off.z + i] = a.s_def_iid[o.val_start + i];
            a.d_origin[off.z + i] = a.s_origin[o.val_start + i];
        }
        for (uint32_t i = lane; i < o.n_ev; i += 32) a.d_ev[off.w + i] = a.s_ev[o.ev_start + i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint4 tot = a.off[a.n_funcs];
        a.d_blk_off[a.n_blocks] = tot.x; a.d_imm_off[a.n_funcs] = tot.y; a.d_val_off[a.n_funcs] = tot.z;
    }
}
#endif

/* ------------------------------------------------------------------ context */
struct Part {                  /* one kernel's share of the functions            */
    std::vector<uint32_t> list;
    uint32_t *d_list = nullptr, *d_counter = nullptr;
    uint8_t *d_scratch = nullptr;
    size_t scratch_per_group = 0;
    Caps cap{};
    uint32_t n_groups = 0, hot_bytes = 0, grid = 0;
};

/* device buffers are grow-only slots: repeated uploads of same-sized corpora
 * (the end-to-end loop) do not pay cudaMalloc/cudaFree again                */
enum {
    B_FUNC = 0, B_FBO, B_EXT_OFF, B_MEM_OFF, B_IMM_OFF, B_VAL_OFF, B_BLK, B_BLK_OFF, B_HDR, B_TAG, B_PAY,
    B_EXT_TAG, B_EXT_PAY, B_MEM, B_IMM, B_ALIVE, B_DEF_IID, B_MODSETS,
    B_O_HDR, B_O_TAG, B_O_PAY, B_O_IMM, B_O_ALIVE, B_O_DEF_IID, B_O_ORIGIN, B_O_EXT_TAG, B_O_EXT_PAY, B_O_MEM,
    B_O_BLK, B_O_BLK_START, B_O_BLK_CNT, B_O_EV, B_O_FUNC,
    B_LIST0, B_LIST1, B_LIST2, B_COUNTER0, B_COUNTER1, B_COUNTER2, B_SCRATCH0, B_SCRATCH1, B_SCRATCH2,
    B_RETRY_LIST, B_RETRY_WORDS, B_TILES0, B_TILES1, B_TILES2, B_TILE_COUNTER0, B_TILE_COUNTER1, B_TILE_COUNTER2, B_TILE_SCRATCH0, B_TILE_SCRATCH1, B_TILE_SCRATCH2, B_TILE_FLIST, B_REST_LIST, B_BIG_REST_LIST, B_RETRY_BIG,
    B_D_OFF, B_D_SUMS, B_D_HDR, B_D_TAG, B_D_PAY, B_D_IMM, B_D_ALIVE, B_D_DEF_IID, B_D_ORIGIN, B_D_EV,
    B_D_BLK_OFF, B_D_IMM_OFF, B_D_VAL_OFF, B_D_FUNC, B_SR_MAP, B__N
};
struct DBuf { void *p = nullptr; size_t cap = 0; };

struct cl_ctx {
    int device = 0;
    cudaStream_t stream = 0;
#if CL_CUDA
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t stream2 = nullptr;     /* the CTA-group kernel runs beside the warp kernel */
    int n_sm = 148;
    int n_sm_or_1() const { return n_sm; }
#else
    int n_sm_or_1() const { return 1; }
#endif
    cl_pattern_blob h_pb{};
    bool have_pb = false, have_in = false, have_out = false;
    cl_pattern_blob *d_pb = nullptr;
    uint8_t *d_opflags = nullptr;
    DBuf buf[B__N];
    uint32_t F = 0, B = 0, n_modsets = 0;
    cl_corpus d_in{};
    uint64_t n_inst = 0, n_ext = 0, n_mem = 0, n_imm = 0, n_val = 0;
    KArgs k{};
    unsigned long long *d_cursor = nullptr, *d_stats = nullptr, *d_prof = nullptr;
    unsigned long long h_prof[PF__N] = { 0 };
    unsigned long long h_cursor[CUR__N] = { 0, 0, 0, 0 };
    Part part[2];              /* general per-function kernels: 0 = warp groups (small functions), 1 = CTA groups (large ones) */
    uint32_t *d_retry_list = nullptr, *d_retry_count = nullptr, *d_retry_counter = nullptr;
    /* tile kernels (tile.cuh): small functions packed into tiles, one CTA per tile */
    int tile_mode = -1;        /* bit 1: shared-memory tiles (small corpora), bit 2: big tiles resident in L2; 0 = general kernels only;
                                  -1 = by corpus size: big tiles when they keep every SM busy, else shared-memory tiles */
    struct TileClass {
        std::vector<TileDesc> tiles;
        TileDesc *d_tiles = nullptr; uint32_t *d_counter = nullptr; uint8_t *d_scratch = nullptr;
        size_t scratch_per_group = 0; uint32_t grid = 0, groups = 0;
    } tc[3];                   /* [0]: one long block per tile (TileCfgG4), [1]: shared-memory tiles, [2]: big tiles in global scratch */
    int gtile_cfg = -1;        /* 0/1/2/3: TileCfgG/G2/G3/G4 (4096/8192/16384/32768 records), -1: by corpus size */
    int tile_mode_env = -1, gtile_cfg_env = -1, gtile_ctas = 2;   /* two 1024-thread CTAs per SM at 32 registers: +27 % over one at 64 (latency bound: resident warps are what counts) */
    std::vector<uint32_t> tile_flist;    /* function ids of all tiles, class 0 first */
    std::vector<uint32_t> rest, big_rest; /* small / large functions that are not in a tile */
    uint32_t *d_tile_flist = nullptr, *d_rest = nullptr, *d_big_rest = nullptr;
    uint32_t *d_retry_big = nullptr, *d_retry_big_count = nullptr, *d_retry_big_counter = nullptr;   /* large functions the tile kernel hands back */
    uint32_t n_tile_funcs = 0, h_retry = 0, n_launches = 0; bool used_tiles = false;
    /* the function-resident path (fused.cuh): default for the post-SSA stage */
    int fused_mode = -1;       /* 1: every post-SSA run, 0: never, -1: the runs that ask for match lists (emit_matches, MATCH_ONLY): there the tile
                                  kernel cannot serve and the fused kernels are the production path; plain runs take the tile kernel (faster, measured) */
    clf_ctx *clf = nullptr; bool fused_ok = false, used_fused = false;
    DenseArgs dense{}; bool have_dense = false;     /* dense result of the last run (device) */
    cl_stats stats{};
    float last_ms = 0;
    uint32_t small_max = 512;  /* records: warp-group kernel up to here, CTA-group kernel above */
};

template <class T> static int dget(cl_ctx *c, int id, T **p, size_t n) {
    DBuf &b = c->buf[id];
    const size_t need = n * sizeof(T);
    if (b.cap < need || !b.p) {
        dfree(b.p);
        b.p = nullptr; b.cap = 0;
        const size_t want = need + need / 16 + 256;
        if (dmalloc(&b.p, want)) return -1;
        b.cap = want;
    }
    *p = (T *)b.p;
    return 0;
}
template <class T> static int dput(cl_ctx *c, int id, T **p, const T *h, size_t n) {
    if (dget(c, id, p, n)) return -1;
    return h2d(*p, h, n * sizeof(T), c->stream);
}

extern "C" int cl_create(int device, cl_ctx **out) {
    cl_ctx *c = new cl_ctx();
    c->device = device;
#if CL_CUDA
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) { delete c; FAIL("no CUDA device: the product path has no CPU fallback"); }
    if (device >= n) { delete c; FAIL("device %d out of range (%d present)", device, n); }
    CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) { delete c; FAIL("device %d is sm_%d%d: this library is built for sm_100a only", device, prop.major, prop.minor); }
    c->n_sm = prop.multiProcessorCount;
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreate(&c->ev0));
    CUDA_OK(cudaEventCreate(&c->ev1));
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
#endif
    if (const char *e = getenv("CL_SMALL_MAX")) c->small_max = (uint32_t)atoi(e);   /* the few knobs the tests and the tuning log use */
    if (const char *e = getenv("CL_FUSED")) c->fused_mode = atoi(e) != 0;
    if (const char *e = getenv("CL_TILE")) c->tile_mode_env = atoi(e) & 6;
    if (const char *e = getenv("CL_GTILE_CFG")) c->gtile_cfg_env = std::min(3, std::max(0, atoi(e)));
    if (const char *e = getenv("CL_GTILE_CTAS")) c->gtile_ctas = std::min(2, std::max(1, atoi(e)));
    void *p = nullptr;
    if (dmalloc(&p, sizeof(H_OPFLAGS))) { delete c; return -1; }
    c->d_opflags = (uint8_t *)p;
    h2d(c->d_opflags, H_OPFLAGS, sizeof(H_OPFLAGS), c->stream);
    if (dmalloc(&p, sizeof(cl_pattern_blob))) { delete c; return -1; }
    c->d_pb = (cl_pattern_blob *)p;
    if (dmalloc(&p, sizeof(unsigned long long) * CUR__N)) { delete c; return -1; }
    c->d_cursor = (unsigned long long *)p;
    if (dmalloc(&p, sizeof(cl_stats))) { delete c; return -1; }
    c->d_stats = (unsigned long long *)p;
    if (dmalloc(&p, sizeof(unsigned long long) * PF__N)) { delete c; return -1; }
    c->d_prof = (unsigned long long *)p;
    *out = c;
    return 0;
}

extern "C" void cl_destroy(cl_ctx *c) {
    if (!c) return;
#if CL_CUDA
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
#endif
    clf_destroy(c->clf);
    for (DBuf &b : c->buf) dfree(b.p);
    dfree(c->d_opflags); dfree(c->d_pb); dfree(c->d_cursor); dfree(c->d_stats);
#if CL_CUDA
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->stream2) cudaStreamDestroy(c->stream2);
    if (c->stream) cudaStreamDestroy(c->stream);
#endif
    delete c;
}

extern "C" int cl_set_patterns(cl_ctx *c, const void *blob, size_t nbytes) {
    if (nbytes != sizeof(cl_pattern_blob)) FAIL("pattern blob: %zu bytes, expected %zu", nbytes, sizeof(cl_pattern_blob));
    memcpy(&c->h_pb, blob, nbytes);
    if (c->h_pb.magic != CL_PATTERN_MAGIC || c->h_pb.n_patterns > CL_MAX_PATTERNS) FAIL("pattern blob: bad magic or count");
    if (c->h_pb.budget >= (1u << 20)) FAIL("pattern blob: budget %u does not fit the 20-bit tuple rank", c->h_pb.budget);
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
#endif
    if (h2d(c->d_pb, &c->h_pb, sizeof(cl_pattern_blob), c->stream)) return -1;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    c->have_pb = true;
    if (!c->clf && clf_create(&c->clf, c->device, c->n_sm_or_1())) FAIL("clf_create failed");
    {
        const int r = clf_set_patterns(c->clf, &c->h_pb, (void *)(uintptr_t)c->stream, g_err, sizeof g_err);
        if (r < 0) return -1;
        c->fused_ok = r == 1;
    }
    return 0;
}
extern "C" int cl_set_threads(cl_ctx *, int) { return 0; }

static Caps caps_for(uint32_t n_max, uint32_t nv_max, uint32_t nb_max, uint32_t imm_max, uint32_t blk_max,
                     uint32_t ext_max) {
    Caps c;
    c.I = 3 * n_max + 64;
    c.V = nv_max + 2 * n_max + 64;
    c.B = nb_max + 1;
    c.M = 4 * std::min(blk_max, c.I) + 4 * n_max + 256;
    c.S = n_max + 16;
    c.Q = imm_max + 2 * n_max + 64;
    c.E = 8 * n_max + 256;
    c.U = 8 * c.I + ext_max + 64;
    c.X = 2 * n_max + 16;
    return c;
}

extern "C" int cl_upload(cl_ctx *c, const cl_corpus *in) {
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    c->have_in = c->have_out = c->have_dense = false;
    const uint32_t F = in->n_funcs, B = in->n_blocks;
    if (in->func_blk_off[F] != B) FAIL("func_blk_off[n_funcs] != n_blocks");
    c->F = F; c->B = B; c->n_modsets = in->n_modsets;
    c->n_inst = in->blk_off[B]; c->n_ext = in->ext_off[F]; c->n_mem = in->mem_off[F];
    c->n_imm = in->imm_off[F]; c->n_val = in->val_off[F];
    if (3 * c->n_inst + 1024 >= (1ull << 32)) FAIL("corpus too large for 32-bit stream offsets: shard it");
    cl_corpus &d = c->d_in;
    d = *in;
    cl_modset *dms = nullptr;
    if (dput(c, B_FUNC, &d.func, in->func, F) || dput(c, B_FBO, &d.func_blk_off, in->func_blk_off, F + 1) ||
        dput(c, B_EXT_OFF, &d.ext_off, in->ext_off, F + 1) || dput(c, B_MEM_OFF, &d.mem_off, in->mem_off, F + 1) ||
        dput(c, B_IMM_OFF, &d.imm_off, in->imm_off, F + 1) || dput(c, B_VAL_OFF, &d.val_off, in->val_off, F + 1) ||
        dput(c, B_BLK, &d.blk, in->blk, B) || dput(c, B_BLK_OFF, &d.blk_off, in->blk_off, B + 1) ||
        dput(c, B_HDR, &d.hdr, in->hdr, c->n_inst) || dput(c, B_TAG, &d.tag, in->tag, c->n_inst * 8) ||
        dput(c, B_PAY, &d.pay, in->pay, c->n_inst * 8) || dput(c, B_EXT_TAG, &d.ext_tag, in->ext_tag, c->n_ext) ||
        dput(c, B_EXT_PAY, &d.ext_pay, in->ext_pay, c->n_ext) || dput(c, B_MEM, &d.mem, in->mem, c->n_mem) ||
        dput(c, B_IMM, &d.imm, in->imm, c->n_imm) || dput(c, B_ALIVE, &d.val_alive, in->val_alive, c->n_val) ||
        dput(c, B_DEF_IID, &d.val_def_iid, in->val_def_iid, c->n_val) ||
        dput(c, B_MODSETS, &dms, in->modsets, in->n_modsets))
        return -1;
    d.modsets = dms;
    d.val_origin = nullptr;

    /* work partition of the general per-function kernels (while the copies are in flight): one warp per
     * small function, one CTA per large one.  A counting sort by record count replaces round 1's three
     * comparison sorts (same purpose: a CTA's batch of functions has one size, long poles first).       */
    uint32_t n_max[2] = { 0, 0 }, nv_max[2] = { 0, 0 }, nb_max[2] = { 0, 0 }, imm_max[2] = { 0, 0 }, blk_max[2] = { 0, 0 }, ext_max[2] = { 0, 0 };
    for (Part &p : c->part) p.list.clear();
    std::vector<uint32_t> small_cnt(2 * ((size_t)c->small_max + 2), 0);
    std::vector<std::pair<uint32_t, uint32_t>> big;
    for (uint32_t f = 0; f < F; f++) {
        const uint32_t b0 = in->func_blk_off[f], b1 = in->func_blk_off[f + 1];
        const uint32_t n = in->blk_off[b1] - in->blk_off[b0];
        if (in->val_off[f + 1] - in->val_off[f] != in->func[f].next_vid)
            FAIL("function %u: value region holds %u entries, next_vid is %u", f, in->val_off[f + 1] - in->val_off[f], in->func[f].next_vid);
        const int k = n <= c->small_max ? 0 : 1;
        if (k == 1) big.emplace_back(~n, f);
        else small_cnt[(in->func[f].arch == CL_ARCH_SM52 ? 0u : c->small_max + 1) + (c->small_max - n)]++;      /* by arch (sm52 runs an extra pass), then size, largest first */
        n_max[k] = std::max(n_max[k], n);
        nv_max[k] = std::max(nv_max[k], in->func[f].next_vid);
        nb_max[k] = std::max(nb_max[k], b1 - b0);
        imm_max[k] = std::max(imm_max[k], in->imm_off[f + 1] - in->imm_off[f]);
        ext_max[k] = std::max(ext_max[k], in->ext_off[f + 1] - in->ext_off[f]);
        if (b1 - b0 == 1) blk_max[k] = std::max(blk_max[k], n);
        else for (uint32_t b = b0; b < b1; b++) blk_max[k] = std::max(blk_max[k], in->blk_off[b + 1] - in->blk_off[b]);
    }
    std::sort(big.begin(), big.end());            /* long poles first (a handful of functions) */
    for (auto &pr : big) c->part[1].list.push_back(pr.second);
    {
        uint32_t run = 0;
        for (uint32_t &x : small_cnt) { const uint32_t t = x; x = run; run += t; }
        c->part[0].list.resize(run);
        for (uint32_t f = 0; f < F; f++) {
            const uint32_t n = in->blk_off[in->func_blk_off[f + 1]] - in->blk_off[in->func_blk_off[f]];
            if (n <= c->small_max) c->part[0].list[small_cnt[(in->func[f].arch == CL_ARCH_SM52 ? 0u : c->small_max + 1) + (c->small_max - n)]++] = f;
        }
    }
    for (int k = 0; k < 2; k++) {
        Part &p = c->part[k];
        if (p.list.empty()) continue;
        p.cap = caps_for(n_max[k], nv_max[k], nb_max[k], imm_max[k], blk_max[k], ext_max[k]);
        p.scratch_per_group = (scratch_bytes(p.cap) + 255) & ~(size_t)255;
        p.hot_bytes = 0;
#if CL_CUDA
        if (k == 0) { p.grid = (uint32_t)std::min<size_t>((size_t)c->n_sm, (p.list.size() + 31) / 32); p.n_groups = p.grid * 32; }      /* 32 warps per CTA, one CTA per SM */
        else { p.grid = (uint32_t)std::min<size_t>((size_t)c->n_sm * CL_CTA_CTAS_PER_SM, p.list.size()); p.n_groups = p.grid; }
#else
        p.grid = 1; p.n_groups = 1;
#endif
        static const int LIST_ID[2] = { B_LIST0, B_LIST1 }, CNT_ID[2] = { B_COUNTER0, B_COUNTER1 }, SCR_ID[2] = { B_SCRATCH0, B_SCRATCH1 };
        if (dput(c, LIST_ID[k], &p.d_list, p.list.data(), p.list.size())) return -1;
        if (dget(c, CNT_ID[k], &p.d_counter, 1)) return -1;
        if (dget(c, SCR_ID[k], &p.d_scratch, p.scratch_per_group * p.n_groups)) return -1;
    }
    /* tiles: small functions without overflow slots, by size class, packed in size order */
    for (auto &t : c->tc) t.tiles.clear();
    c->tile_flist.clear(); c->rest.clear(); c->big_rest.clear(); c->n_tile_funcs = 0;
    if (!(c->fused_mode == 1 && (c->fused_ok || !c->have_pb))) {       /* the fused path needs no host-side plan */
        struct Need { uint32_t I, V, Q, B, f; };
        /* tile size by corpus size: the bigger the tile the better the passes amortise (profiles/r01_tuning.md),
         * as long as there are a few tiles per SM                                                              */
        {
            uint64_t n_small = 0;
            for (uint32_t f = 0; f < F; f++) {
                const uint32_t n = in->blk_off[in->func_blk_off[f + 1]] - in->blk_off[in->func_blk_off[f]];
                if (tile_icap(n) <= TileCfgG4::I) n_small += n;          /* everything a tile can take */
            }
            int n_sm = 148;
#if CL_CUDA
            n_sm = c->n_sm;
#endif
            const uint64_t per_sm = n_small / (uint64_t)n_sm;
            c->gtile_cfg = per_sm >= 3 * 19600 ? 3 : per_sm >= 3 * 9800 ? 2 : per_sm >= 3 * 4900 ? 1 : 0;
            c->tile_mode = per_sm >= 3 * 2450 ? 4 : 2;
            if (c->gtile_cfg_env >= 0) c->gtile_cfg = c->gtile_cfg_env;
            if (c->tile_mode_env >= 0) c->tile_mode = c->tile_mode_env;
        }
        const int gc = c->gtile_cfg;
        const uint32_t gI = gc == 3 ? TileCfgG4::I : gc == 2 ? TileCfgG3::I : gc == 1 ? TileCfgG2::I : TileCfgG::I,
                       gV = gc == 3 ? TileCfgG4::V : gc == 2 ? TileCfgG3::V : gc == 1 ? TileCfgG2::V : TileCfgG::V,
                       gQ = gc == 3 ? TileCfgG4::Q : gc == 2 ? TileCfgG3::Q : gc == 1 ? TileCfgG2::Q : TileCfgG::Q,
                       gB = gc == 3 ? TileCfgG4::B : gc == 2 ? TileCfgG3::B : gc == 1 ? TileCfgG2::B : TileCfgG::B,
                       gF = gc == 3 ? TileCfgG4::F : gc == 2 ? TileCfgG3::F : gc == 1 ? TileCfgG2::F : TileCfgG::F;
        /* functions of each tile class in order of decreasing size (counting sort by record count, stable in
         * function order: the same packing as round 1's stable_sort, without its n log n)                    */
        std::vector<uint8_t> cls_of(F, 0xFF);
        std::vector<uint32_t> cnt[3];
        /* big tiles also take the functions above small_max that fit one (a 4096-instruction block is a tile of its
         * own): the passes of tile.cuh are data parallel inside a block, the CTA kernel walks its chains and
         * matches with one lane.  What they hand back goes to the CTA kernel (retry_big).                      */
        const uint32_t tile_max = std::max(c->small_max, (c->tile_mode & 4) ? (uint32_t)TileCfgG4::I : 0u);
        for (int k = 0; k < 3; k++) cnt[k].assign((size_t)tile_max + 2, 0);
        auto need_of = [&](uint32_t f) {
            const uint32_t b0 = in->func_blk_off[f], b1 = in->func_blk_off[f + 1];
            const uint32_t n = in->blk_off[b1] - in->blk_off[b0];
            return Need{ tile_icap(n), tile_vcap(in->func[f].next_vid, n), tile_qcap(in->imm_off[f + 1] - in->imm_off[f], n), b1 - b0, f };
        };
        for (uint32_t f = 0; f < F; f++) {
            const uint32_t b0 = in->func_blk_off[f], b1 = in->func_blk_off[f + 1];
            const uint32_t n = in->blk_off[b1] - in->blk_off[b0], nb = b1 - b0;
            const bool small = n <= c->small_max;
            const Need nd = need_of(f);
            const bool plain = in->ext_off[f + 1] == in->ext_off[f] && nb > 0;
            int k = -1;
            if (small && plain && (c->tile_mode & 2) && nd.I <= TileCfgL::I && nd.V <= TileCfgL::V && nd.Q <= TileCfgL::Q && nd.B <= TileCfgL::B) k = 1;
            else if (n <= tile_max && plain && (c->tile_mode & 4) && nd.I <= gI && nd.V <= gV && nd.Q <= gQ && nd.B <= gB) k = 2;
            else if (n <= tile_max && plain && (c->tile_mode & 4) && nd.I <= TileCfgG4::I && nd.V <= TileCfgG4::V && nd.Q <= TileCfgG4::Q && nd.B <= TileCfgG4::B) k = 0;
            if (k >= 0) { cls_of[f] = (uint8_t)k; cnt[k][tile_max - n]++; }
            else if (small) c->rest.push_back(f);
            else c->big_rest.push_back(f);
        }
        const uint32_t capI[3] = { TileCfgG4::I, TileCfgL::I, gI }, capV[3] = { TileCfgG4::V, TileCfgL::V, gV }, capQ[3] = { TileCfgG4::Q, TileCfgL::Q, gQ },
                       capB[3] = { TileCfgG4::B, TileCfgL::B, gB }, capF[3] = { TileCfgG4::F, TileCfgL::F, gF };
        for (int k = 0; k < 3; k++) {
            uint32_t run = 0;
            for (uint32_t &x : cnt[k]) { const uint32_t t = x; x = run; run += t; }
            std::vector<uint32_t> order(run);
            for (uint32_t f = 0; f < F; f++) if (cls_of[f] == k) {
                const uint32_t n = in->blk_off[in->func_blk_off[f + 1]] - in->blk_off[in->func_blk_off[f]];
                order[cnt[k][tile_max - n]++] = f;
            }
            TileDesc cur = { (uint32_t)c->tile_flist.size(), 0 };
            uint32_t sI = 0, sV = 0, sQ = 0, sB = 0;
            auto flush = [&]() { if (cur.nf) c->tc[k].tiles.push_back(cur); cur.first = (uint32_t)c->tile_flist.size(); cur.nf = 0; sI = sV = sQ = sB = 0; };
            for (const uint32_t f : order) {
                const Need nd = need_of(f);
                if (cur.nf && (sI + nd.I > capI[k] || sV + nd.V > capV[k] || sQ + nd.Q > capQ[k] || sB + nd.B > capB[k] || cur.nf >= capF[k])) flush();
                c->tile_flist.push_back(nd.f);
                cur.nf++; sI += nd.I; sV += nd.V; sQ += nd.Q; sB += nd.B;
            }
            flush();
        }
        c->n_tile_funcs = (uint32_t)c->tile_flist.size();
    }
    {
        uint32_t *words = nullptr;
        if (dget(c, B_RETRY_LIST, &c->d_retry_list, (size_t)F)) return -1;
        if (dget(c, B_RETRY_WORDS, &words, 4)) return -1;
        c->d_retry_count = words; c->d_retry_counter = words + 1;
    }
    if (c->n_tile_funcs) {
        static const int T_ID[3] = { B_TILES0, B_TILES1, B_TILES2 }, C_ID[3] = { B_TILE_COUNTER0, B_TILE_COUNTER1, B_TILE_COUNTER2 },
                         S_ID[3] = { B_TILE_SCRATCH0, B_TILE_SCRATCH1, B_TILE_SCRATCH2 };
        for (int k = 0; k < 3; k++) {
            cl_ctx::TileClass &t = c->tc[k];
            if (t.tiles.empty()) continue;
#if CL_CUDA
            if (k == 0) {
                t.scratch_per_group = gtile_scratch_bytes<TileCfgG4>();
                t.grid = (uint32_t)std::min<size_t>((size_t)c->n_sm * c->gtile_ctas, t.tiles.size());
                t.groups = t.grid;
            } else if (k == 1) {
                t.scratch_per_group = tile_scratch_bytes<TileCfgL>();
                t.grid = (uint32_t)std::min<size_t>((size_t)c->n_sm, t.tiles.size());
                t.groups = t.grid;
            } else {
                t.scratch_per_group = c->gtile_cfg == 3 ? gtile_scratch_bytes<TileCfgG4>() : c->gtile_cfg == 2 ? gtile_scratch_bytes<TileCfgG3>() : c->gtile_cfg == 1 ? gtile_scratch_bytes<TileCfgG2>() : gtile_scratch_bytes<TileCfgG>();
                t.grid = (uint32_t)std::min<size_t>((size_t)c->n_sm * c->gtile_ctas, t.tiles.size());
                t.groups = t.grid;
            }
#else
            t.scratch_per_group = k == 1 ? tile_scratch_bytes<TileCfgL>() : tile_scratch_bytes<TileCfgG4>();      /* the largest configuration */
            t.grid = t.groups = 1;
#endif
            if (dput(c, T_ID[k], &t.d_tiles, t.tiles.data(), t.tiles.size())) return -1;
            if (dget(c, C_ID[k], &t.d_counter, 1)) return -1;
            if (dget(c, S_ID[k], &t.d_scratch, t.scratch_per_group * t.groups)) return -1;
        }
        if (dput(c, B_TILE_FLIST, &c->d_tile_flist, c->tile_flist.data(), c->tile_flist.size())) return -1;
    }
    if (dput(c, B_REST_LIST, &c->d_rest, c->rest.data(), c->rest.size())) return -1;
    if (dput(c, B_BIG_REST_LIST, &c->d_big_rest, c->big_rest.data(), c->big_rest.size())) return -1;
    {
        uint32_t *w = nullptr;
        if (dget(c, B_RETRY_BIG, &w, (size_t)c->part[1].list.size() + 4)) return -1;
        c->d_retry_big_count = w; c->d_retry_big_counter = w + 1; c->d_retry_big = w + 4;
    }

    /* result buffers (worst-case growth, G3/G4) */
    KArgs &k = c->k;
    memset(&k, 0, sizeof k);
    k.in = d; k.pb = c->d_pb; k.opflags = c->d_opflags;
    k.cap[CUR_INST] = 3 * c->n_inst + 1024;
    k.cap[CUR_IMM] = c->n_imm + 2 * c->n_inst + 1024;
    k.cap[CUR_VAL] = c->n_val + 2 * c->n_inst + 1024;
    k.cap[CUR_EV] = 2 * c->n_inst + 4096;
    if (dget(c, B_O_HDR, &k.o_hdr, k.cap[CUR_INST]) || dget(c, B_O_TAG, &k.o_tag, k.cap[CUR_INST] * 8) ||
        dget(c, B_O_PAY, &k.o_pay, k.cap[CUR_INST] * 8) || dget(c, B_O_IMM, &k.o_imm, k.cap[CUR_IMM]) ||
        dget(c, B_O_ALIVE, &k.o_alive, k.cap[CUR_VAL]) || dget(c, B_O_DEF_IID, &k.o_def_iid, k.cap[CUR_VAL]) ||
        dget(c, B_O_ORIGIN, &k.o_origin, k.cap[CUR_VAL]) || dget(c, B_O_EXT_TAG, &k.o_ext_tag, c->n_ext) ||
        dget(c, B_O_EXT_PAY, &k.o_ext_pay, c->n_ext) || dget(c, B_O_MEM, &k.o_mem, c->n_mem) ||
        dget(c, B_O_BLK, &k.o_blk, B) || dget(c, B_O_BLK_START, &k.o_blk_start, B) || dget(c, B_O_BLK_CNT, &k.o_blk_cnt, B) ||
        dget(c, B_O_EV, &k.o_ev, k.cap[CUR_EV]) || dget(c, B_O_FUNC, &k.o_func, F))
        return -1;
    k.cursor = c->d_cursor; k.stats = c->d_stats; k.prof = c->d_prof;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));     /* the caller may reuse its buffers */
#endif
    c->have_in = true;
    return 0;
}

/* launch one kernel: `which` selects the kernel and the scratch, the work list is
 * that part's own, or (mode 1) what an earlier kernel queued on the device, or
 * (mode 2) the small functions outside the tiles                                */
static int launch_part(cl_ctx *c, int which, KArgs k, int mode = 0, bool side = false) {
#if CL_CUDA
    cudaStream_t st = side ? c->stream2 : c->stream;
#else
    cudaStream_t st = c->stream; (void)side;
#endif
    Part &p = c->part[which];
    const bool retry = mode == 1 || mode == 3;
    if (mode == 0 && p.list.empty()) return 0;
    if (mode == 2 && c->rest.empty()) return 0;
    if (mode == 4 && c->big_rest.empty()) return 0;
    if (mode == 3 && p.list.empty()) return 0;             /* no large function at all */
    if (mode == 1 && p.grid == 0) return 0;                /* no small function at all */
    k.list = mode == 1 ? c->d_retry_list : mode == 3 ? c->d_retry_big : mode == 2 ? c->d_rest : mode == 4 ? c->d_big_rest : p.d_list;
    k.n_list = mode == 1 ? c->F : mode == 3 ? (uint32_t)p.list.size()
             : mode == 2 ? (uint32_t)c->rest.size() : mode == 4 ? (uint32_t)c->big_rest.size() : (uint32_t)p.list.size();
    k.n_list_ptr = mode == 1 ? c->d_retry_count : mode == 3 ? c->d_retry_big_count : nullptr;
    k.work_counter = mode == 1 ? c->d_retry_counter : mode == 3 ? c->d_retry_big_counter : p.d_counter;
    k.retry_list = nullptr; k.retry_count = nullptr;
    (void)retry;
    k.scratch = p.d_scratch; k.scratch_per_group = p.scratch_per_group; k.gcap = p.cap; k.hot_bytes = p.hot_bytes;
    if (dzero(k.work_counter, sizeof(uint32_t), st)) return -1;
    c->n_launches++;
#if CL_CUDA
    if (which == 0) k_postssa_warp_sync<32, 1><<<p.grid, 1024, 0, st>>>(k);     /* 1 CTA/SM, 64 registers */
    else k_postssa_cta<8, CL_CTA_CTAS_PER_SM><<<p.grid, 256, 0, st>>>(k);
    CUDA_OK(cudaGetLastError());
#else
    static uint32_t gw[GW__N];
    Grp<0> g; g.rank = 0; g.size = 1; g.red = nullptr;
    group_loop(g, k, gw, (uint8_t *)nullptr, k.scratch);
#endif
    return 0;
}

#if CL_CUDA
template <class C, int NW, int MINB> static int launch_tile_kernel(cl_ctx *c, const KArgs &k, uint32_t grid, cudaStream_t st) {
    const size_t smem = tile_p_bytes() + sizeof(TileS<C>);
    CUDA_OK(cudaFuncSetAttribute(k_postssa_tile<C, NW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_postssa_tile<C, NW, MINB><<<grid, NW * 32, smem, st>>>(k);
    CUDA_OK(cudaGetLastError());
    (void)c;
    return 0;
}
#endif
/* class 1 (shared-memory tiles) on the side stream, class 2 (big tiles) on the main stream */
static int launch_tiles(cl_ctx *c, KArgs k, int cls) {
    cl_ctx::TileClass &t = c->tc[cls];
    if (t.tiles.empty()) return 0;
    k.tiles = t.d_tiles; k.n_tiles = (uint32_t)t.tiles.size(); k.tile_counter = t.d_counter;
    k.tile_scratch = t.d_scratch; k.tile_scratch_per_cta = t.scratch_per_group; k.tile_flist = c->d_tile_flist;
    k.retry_list = c->d_retry_list; k.retry_count = c->d_retry_count;
    k.retry_big_list = c->d_retry_big; k.retry_big_count = c->d_retry_big_count; k.small_max = c->small_max;
    c->n_launches++;
#if CL_CUDA
    cudaStream_t st = cls == 2 ? c->stream : c->stream2;
    if (dzero(k.tile_counter, sizeof(uint32_t), st)) return -1;
    if (cls == 0) {
        if (c->gtile_ctas == 2) k_postssa_gtile<TileCfgG4, 32, 2><<<t.grid, 1024, 0, st>>>(k);
        else k_postssa_gtile<TileCfgG4, 32, 1><<<t.grid, 1024, 0, st>>>(k);
        CUDA_OK(cudaGetLastError());
        return 0;
    }
    if (cls == 2) {
        if (c->gtile_ctas == 2) {
            if (c->gtile_cfg == 3) k_postssa_gtile<TileCfgG4, 32, 2><<<t.grid, 1024, 0, st>>>(k);
            else if (c->gtile_cfg == 2) k_postssa_gtile<TileCfgG3, 32, 2><<<t.grid, 1024, 0, st>>>(k);
            else if (c->gtile_cfg == 1) k_postssa_gtile<TileCfgG2, 32, 2><<<t.grid, 1024, 0, st>>>(k);
            else k_postssa_gtile<TileCfgG, 32, 2><<<t.grid, 1024, 0, st>>>(k);
        } else {
            if (c->gtile_cfg == 3) k_postssa_gtile<TileCfgG4, 32, 1><<<t.grid, 1024, 0, st>>>(k);
            else if (c->gtile_cfg == 2) k_postssa_gtile<TileCfgG3, 32, 1><<<t.grid, 1024, 0, st>>>(k);
            else if (c->gtile_cfg == 1) k_postssa_gtile<TileCfgG2, 32, 1><<<t.grid, 1024, 0, st>>>(k);
            else k_postssa_gtile<TileCfgG, 32, 1><<<t.grid, 1024, 0, st>>>(k);
        }
        CUDA_OK(cudaGetLastError());
        return 0;
    }
    return launch_tile_kernel<TileCfgL, 16, 1>(c, k, t.grid, st);
#else
    if (dzero(k.tile_counter, sizeof(uint32_t), c->stream)) return -1;
    static TileP P;
    Grp<0> g; g.rank = 0; g.size = 1; g.red = nullptr;
    t_setup(g, P, k.pb);
    if (cls == 1) { static TileS<TileCfgL> T; g.red = T.red; tile_loop(g, T, P, k, 0); }
    else if (cls == 0) { static TileS<TileCfgG4> T; alignas(16) static uint8_t pl[132 * TileCfgG4::I]; g.red = T.red; tile_loop(g, T, P, k, 0, pl); }
    else if (c->gtile_cfg == 3) { static TileS<TileCfgG4> T; alignas(16) static uint8_t pl[132 * TileCfgG4::I]; g.red = T.red; tile_loop(g, T, P, k, 0, pl); }
    else if (c->gtile_cfg == 2) { static TileS<TileCfgG3> T; alignas(16) static uint8_t pl[132 * TileCfgG3::I]; g.red = T.red; tile_loop(g, T, P, k, 0, pl); }
    else if (c->gtile_cfg == 1) { static TileS<TileCfgG2> T; alignas(16) static uint8_t pl[132 * TileCfgG2::I]; g.red = T.red; tile_loop(g, T, P, k, 0, pl); }
    else { static TileS<TileCfgG> T; alignas(16) static uint8_t pl[132 * TileCfgG::I]; g.red = T.red; tile_loop(g, T, P, k, 0, pl); }
    return 0;
#endif
}

static int densify(cl_ctx *c);
static int run(cl_ctx *c, KArgs k) {
    if (!c->have_in) FAIL("no corpus uploaded");
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
#endif
    if (dzero(c->d_cursor, sizeof(unsigned long long) * CUR__N, c->stream)) return -1;
    if (dzero(c->d_stats, sizeof(cl_stats), c->stream)) return -1;
    if (dzero(c->d_prof, sizeof(unsigned long long) * PF__N, c->stream)) return -1;
    if (c->d_retry_count && dzero(c->d_retry_count, sizeof(uint32_t), c->stream)) return -1;
    /* the tile kernel takes the production run of the post-SSA stage; match lists
     * (emit_matches / MATCH_ONLY), the raw stage and tables with a pattern that has
     * no join plan go through the general kernels                                  */
    c->n_launches = 0;
#if CL_CUDA
    g_aux_launches = 0;
#endif
    bool use_tiles = c->n_tile_funcs && !k.raw_passes && !k.emit_matches && !(k.passes & CL_PASS_MATCH_ONLY);
    for (uint32_t pi = 0; pi < c->h_pb.n_patterns; pi++) use_tiles = use_tiles && c->h_pb.p[pi].join_ok;
#if CL_CUDA
    CUDA_OK(cudaEventRecord(c->ev0, c->stream));
    /* large functions (CTA groups) on a side stream, concurrently with the rest */
    CUDA_OK(cudaEventRecord(c->ev_fork, c->stream));
    CUDA_OK(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
#endif
    if (c->d_retry_big_count && dzero(c->d_retry_big_count, sizeof(uint32_t), c->stream)) return -1;
    const bool wants_lists = k.emit_matches || (k.passes & CL_PASS_MATCH_ONLY);
    const bool use_fused = c->fused_ok && c->F && !k.raw_passes && (c->fused_mode == 1 || (c->fused_mode == -1 && wants_lists));
    c->used_fused = use_fused;
    if (use_fused) {
        /* one function resident in shared memory per group (fused.cuh); hand-backs and everything too
         * large for a shared-memory slice (long blocks) go to the general kernels                  */
        use_tiles = false;
        KArgs kf = k;
        kf.retry_list = c->d_retry_list; kf.retry_count = c->d_retry_count;
        kf.retry_big_list = c->d_retry_big; kf.retry_big_count = c->d_retry_big_count; kf.small_max = c->small_max;
        if (clf_run(c->clf, &kf, c->F, (void *)(uintptr_t)c->stream, g_err, sizeof g_err)) return -1;
        { unsigned long long info[4]; clf_info(c->clf, info); c->n_launches += (uint32_t)info[0]; }
        if (launch_part(c, 0, k, 1)) return -1;
        if (launch_part(c, 1, k, 3)) return -1;
    } else if (use_tiles) {
        if (launch_part(c, 1, k, 4, true)) return -1;     /* large functions outside the tiles: side stream */
        if (launch_tiles(c, k, 0)) return -1;    /* one long block per tile: side stream, long poles first */
        if (launch_tiles(c, k, 1)) return -1;    /* CTA tiles: side stream, after the large functions */
        if (launch_tiles(c, k, 2)) return -1;    /* big L2-resident tiles */
        if (launch_part(c, 0, k, 2)) return -1;  /* small functions outside the tiles */
#if CL_CUDA
        CUDA_OK(cudaEventRecord(c->ev_join, c->stream2));
        CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
#endif
        if (launch_part(c, 0, k, 1)) return -1;  /* what the tile kernels handed back */
        if (launch_part(c, 1, k, 3)) return -1;
    } else {
        if (launch_part(c, 1, k, 0, true)) return -1;
        if (launch_part(c, 0, k)) return -1;
    }
#if CL_CUDA
    CUDA_OK(cudaEventRecord(c->ev_join, c->stream2));
    CUDA_OK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
#endif
    if (d2h(c->h_cursor, c->d_cursor, sizeof c->h_cursor, c->stream)) return -1;
    if (d2h(&c->stats, c->d_stats, sizeof(cl_stats), c->stream)) return -1;
    if (d2h(c->h_prof, c->d_prof, sizeof c->h_prof, c->stream)) return -1;
    c->h_retry = 0; c->used_tiles = use_tiles;
    if (c->d_retry_count && d2h(&c->h_retry, c->d_retry_count, sizeof(uint32_t), c->stream)) return -1;
    uint32_t h_retry_big = 0;
    if (c->d_retry_big_count && d2h(&h_retry_big, c->d_retry_big_count, sizeof(uint32_t), c->stream)) return -1;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    c->h_retry += h_retry_big;
    c->have_out = true;
    c->have_dense = false;
    if (densify(c)) return -1;             /* the dense result of the ABI is part of the timed stage */
#if CL_CUDA
    CUDA_OK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    c->n_launches += g_aux_launches;      /* every kernel of the run: main, zeroing, densify */
#endif
    return 0;
}

extern "C" int cl_run_postssa(cl_ctx *c, const cl_run_opts *opts) {
    if (!c->have_pb) FAIL("no pattern table set");
    KArgs k = c->k;
    k.passes = opts->passes; k.max_rounds = opts->max_rounds ? opts->max_rounds : 4; k.emit_matches = opts->emit_matches;
    k.raw_passes = 0;
    return run(c, k);
}
extern "C" int cl_run_raw(cl_ctx *c, uint32_t passes, const cl_sr_entry *map, uint32_t n_map) {
    if (!(passes & (CL_RAW_X4 | CL_RAW_SR))) FAIL("cl_run_raw: no pass selected");
    if (n_map > 64) FAIL("cl_run_raw: more than 64 special-register aliases");
    KArgs k = c->k;
    cl_sr_entry *dmap = nullptr;
    if (dput(c, B_SR_MAP, &dmap, map, (size_t)n_map)) return -1;
    k.passes = 0; k.max_rounds = 0; k.emit_matches = 0;
    k.raw_passes = passes; k.sr = dmap; k.n_sr = n_map;
    return run(c, k);
}

extern "C" int cl_out_sizes(cl_ctx *c, uint64_t sizes[6]) {
    if (!c->have_out) FAIL("no result: call cl_run_* first");
    sizes[0] = c->h_cursor[CUR_INST]; sizes[1] = c->n_ext; sizes[2] = c->n_mem;
    sizes[3] = c->h_cursor[CUR_IMM]; sizes[4] = c->h_cursor[CUR_VAL]; sizes[5] = c->h_cursor[CUR_EV];
    for (int i = 0; i < CUR__N; i++)
        if (c->h_cursor[i] > c->k.cap[i]) FAIL("result stream %d overflowed its capacity (%llu > %llu)", i, c->h_cursor[i], c->k.cap[i]);
    return 0;
}

#if !CL_CUDA
/* host rendition of the densify kernels for the sim build */
static void densify_host(const DenseArgs &a) {
    uint32_t oi = 0, oq = 0, ov = 0, oe = 0;
    for (uint32_t f = 0; f < a.n_funcs; f++) {
        const FuncOut o = a.fo[f];
        a.d_func[f] = o.f; a.d_imm_off[f] = oq; a.d_val_off[f] = ov;
        for (uint32_t b = a.func_blk_off[f]; b < a.func_blk_off[f + 1]; b++)
            a.d_blk_off[b] = oi + (o.n_inst ? a.blk_start[b] - o.inst_start : 0u);
        memcpy(a.d_hdr + oi, a.s_hdr + o.inst_start, sizeof(cl_hdr) * o.n_inst);
        memcpy(a.d_tag + (size_t)oi * 8, a.s_tag + (size_t)o.inst_start * 8, 16ull * o.n_inst);
        memcpy(a.d_pay + (size_t)oi * 8, a.s_pay + (size_t)o.inst_start * 8, 32ull * o.n_inst);
        memcpy(a.d_imm + oq, a.s_imm + o.imm_start, sizeof(cl_imm) * o.n_imm);
        memcpy(a.d_alive + ov, a.s_alive + o.val_start, o.f.next_vid);
        memcpy(a.d_def_iid + ov, a.s_def_iid + o.val_start, 4ull * o.f.next_vid);
        memcpy(a.d_origin + ov, a.s_origin + o.val_start, 4ull * o.f.next_vid);
        memcpy(a.d_ev + oe, a.s_ev + o.ev_start, sizeof(cl_event) * o.n_ev);
        oi += o.n_inst; oq += o.n_imm; ov += o.f.next_vid; oe += o.n_ev;
    }
    a.d_blk_off[a.n_blocks] = oi; a.d_imm_off[a.n_funcs] = oq; a.d_val_off[a.n_funcs] = ov;
}
#endif

/* results of the last run to the dense CSR of the ABI, on the device.  Enqueued by the run itself
 * (right behind its kernels), so that a later cl_download is a plain copy that overlaps the kernels
 * of other contexts instead of queueing behind their persistent grids                           */
static int densify(cl_ctx *c) {
    uint64_t sz[6];
    if (cl_out_sizes(c, sz)) return -1;
    const uint32_t F = c->F, B = c->B;
    const KArgs &k = c->k;
    DenseArgs &a = c->dense;
    memset(&a, 0, sizeof a);
    a.fo = k.o_func; a.n_funcs = F; a.n_blocks = B;
    a.func_blk_off = c->d_in.func_blk_off; a.blk_start = k.o_blk_start; a.blk_cnt = k.o_blk_cnt;
    a.s_hdr = k.o_hdr; a.s_tag = k.o_tag; a.s_pay = k.o_pay; a.s_imm = k.o_imm;
    a.s_alive = k.o_alive; a.s_def_iid = k.o_def_iid; a.s_origin = k.o_origin; a.s_ev = k.o_ev;
#if CL_CUDA
    a.n_scan_blocks = (F + SCAN_TILE - 1) / SCAN_TILE;
#else
    a.n_scan_blocks = 1;
#endif
    if (dget(c, B_D_OFF, &a.off, (size_t)F + 1) || dget(c, B_D_SUMS, &a.block_sums, (size_t)a.n_scan_blocks + 1) ||
        dget(c, B_D_HDR, &a.d_hdr, sz[0]) || dget(c, B_D_TAG, &a.d_tag, sz[0] * 8) || dget(c, B_D_PAY, &a.d_pay, sz[0] * 8) ||
        dget(c, B_D_IMM, &a.d_imm, sz[3]) || dget(c, B_D_ALIVE, &a.d_alive, sz[4]) || dget(c, B_D_DEF_IID, &a.d_def_iid, sz[4]) ||
        dget(c, B_D_ORIGIN, &a.d_origin, sz[4]) || dget(c, B_D_EV, &a.d_ev, sz[5]) || dget(c, B_D_BLK_OFF, &a.d_blk_off, (size_t)B + 1) ||
        dget(c, B_D_IMM_OFF, &a.d_imm_off, (size_t)F + 1) || dget(c, B_D_VAL_OFF, &a.d_val_off, (size_t)F + 1) ||
        dget(c, B_D_FUNC, &a.d_func, F))
        return -1;
#if CL_CUDA
    if (F) {
        k_scan_tiles<<<a.n_scan_blocks, SCAN_T, 0, c->stream>>>(a);
        k_scan_sums<<<1, SCAN_T, 0, c->stream>>>(a);
        k_scan_apply<<<a.n_scan_blocks, SCAN_T, 0, c->stream>>>(a);
        k_densify<<<std::min<uint32_t>((F + 7) / 8, (uint32_t)c->n_sm * 16), 256, 0, c->stream>>>(a);
        CUDA_OK(cudaGetLastError());
        g_aux_launches += 4;
    }
    CUDA_OK(cudaEventRecord(c->ev1, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
#else
    densify_host(a);
#endif
    c->have_dense = true;
    return 0;
}

/* D2H of the dense result straight into the caller's arrays                     */
extern "C" int cl_download(cl_ctx *c, cl_corpus *o, cl_event *events) {
    uint64_t sz[6];
    if (cl_out_sizes(c, sz)) return -1;
    const uint32_t F = c->F, B = c->B;
    const KArgs &k = c->k;
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
#endif
    if (!c->have_dense && densify(c)) return -1;
    const DenseArgs &a = c->dense;
    o->n_funcs = F; o->n_blocks = B; o->n_modsets = c->n_modsets;
    if (d2h(o->func, a.d_func, F * sizeof(cl_func), c->stream) || d2h(o->func_blk_off, c->d_in.func_blk_off, 4ull * (F + 1), c->stream) ||
        d2h(o->ext_off, c->d_in.ext_off, 4ull * (F + 1), c->stream) || d2h(o->mem_off, c->d_in.mem_off, 4ull * (F + 1), c->stream) ||
        d2h(o->imm_off, a.d_imm_off, 4ull * (F + 1), c->stream) || d2h(o->val_off, a.d_val_off, 4ull * (F + 1), c->stream) ||
        d2h(o->blk, k.o_blk, B * sizeof(cl_blk), c->stream) || d2h(o->blk_off, a.d_blk_off, 4ull * (B + 1), c->stream) ||
        d2h(o->hdr, a.d_hdr, sz[0] * sizeof(cl_hdr), c->stream) || d2h(o->tag, a.d_tag, sz[0] * 16, c->stream) ||
        d2h(o->pay, a.d_pay, sz[0] * 32, c->stream) || d2h(o->ext_tag, k.o_ext_tag, c->n_ext * 2, c->stream) ||
        d2h(o->ext_pay, k.o_ext_pay, c->n_ext * 4, c->stream) || d2h(o->mem, k.o_mem, c->n_mem * sizeof(cl_memref), c->stream) ||
        d2h(o->imm, a.d_imm, sz[3] * sizeof(cl_imm), c->stream) || d2h(o->val_alive, a.d_alive, sz[4], c->stream) ||
        d2h(o->val_def_iid, a.d_def_iid, sz[4] * 4, c->stream) || d2h(o->val_origin, a.d_origin, sz[4] * 4, c->stream))
        return -1;
    if (events && d2h(events, a.d_ev, sz[5] * sizeof(cl_event), c->stream)) return -1;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    if (events) {
        /* events of one function are contiguous now; order each run the way the
         * reference appends (seq, kind, idx, ...)                              */
        auto less = [](const cl_event &x, const cl_event &y) {
            const uint32_t *p = (const uint32_t *)&x, *q = (const uint32_t *)&y;
            for (int i = 0; i < 8; i++) if (p[i] != q[i]) return p[i] < q[i];
            return false;
        };
        uint64_t i = 0;
        while (i < sz[5]) {
            uint64_t j = i + 1;
            while (j < sz[5] && events[j].func == events[i].func) j++;
            if (j - i > 1) std::sort(events + i, events + j, less);
            i = j;
        }
    }
    return 0;
}

/* debugging aid (not part of include/culifter.h): per-phase cycle sums of the last run */
extern "C" int cl_debug_profile(cl_ctx *c, unsigned long long *out, int n) {
    for (int i = 0; i < n && i < PF__N; i++) out[i] = c->h_prof[i];
    return PF__N;
}
/* debugging aid: how the last run was partitioned: {tiles, functions in tiles, functions the tile kernel
 * handed back to the general kernel, small functions outside tiles, tile kernel used}            */
extern "C" int cl_debug_partition(cl_ctx *c, unsigned long long *out) {
    out[0] = c->tc[0].tiles.size() + c->tc[1].tiles.size() + c->tc[2].tiles.size(); out[1] = c->n_tile_funcs; out[2] = c->h_retry; out[3] = c->rest.size(); out[4] = c->used_tiles; out[5] = c->n_launches;
    out[6] = c->used_fused ? 16 : c->tile_mode; out[7] = c->gtile_cfg;
    return 0;
}
extern "C" int cl_get_stats(cl_ctx *c, cl_stats *out) { *out = c->stats; return 0; }
extern "C" int cl_last_run_ms(cl_ctx *c, float *ms) { *ms = c->last_ms; return 0; }
extern "C" void *cl_device_counts_ptr(cl_ctx *c) { return c->d_stats; }
extern "C" void *cl_stream(cl_ctx *c) { return (void *)(uintptr_t)c->stream; }

/* For typeseed.cu (same library, not part of the C ABI): the device view of the uploaded corpus, the context's
 * stream and where the device time of a call is kept.                                                           */
extern "C" int cli_corpus_view(cl_ctx *c, uint32_t source, cl_corpus *view, uint64_t counts[2], void **stream, float **last_ms) {
    if (!c || !c->have_in) FAIL("no corpus uploaded");
    *view = c->d_in;
    view->n_funcs = c->F; view->n_blocks = c->B; view->n_modsets = c->n_modsets;
    counts[0] = c->n_inst; counts[1] = c->n_val;
    if (source == 1) {                         /* CL_SEED_RESULT: the dense result of the last run, as cl_download copies it */
        uint64_t sz[6];
        if (cl_out_sizes(c, sz)) return -1;
#if CL_CUDA
        CUDA_OK(cudaSetDevice(c->device));
#endif
        if (!c->have_dense && densify(c)) return -1;
        const DenseArgs &a = c->dense;
        const KArgs &k = c->k;
        view->blk = k.o_blk; view->blk_off = a.d_blk_off;
        view->hdr = a.d_hdr; view->tag = a.d_tag; view->pay = a.d_pay;
        view->ext_tag = k.o_ext_tag; view->ext_pay = k.o_ext_pay; view->mem = k.o_mem;
        view->imm = a.d_imm; view->imm_off = a.d_imm_off; view->val_off = a.d_val_off;
        view->val_alive = a.d_alive; view->val_def_iid = a.d_def_iid; view->val_origin = a.d_origin; view->func = a.d_func;
        counts[0] = sz[0]; counts[1] = sz[4];
    } else if (source != 0) FAIL("cl_seed_types: unknown source %u", source);
    *stream = (void *)(uintptr_t)c->stream;
    *last_ms = &c->last_ms;
    return 0;
}
extern "C" void cli_set_error(const char *msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
