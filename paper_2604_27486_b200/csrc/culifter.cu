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
static int dzero(void *d, size_t n, cudaStream_t st) { if (n) CUDA_OK(cudaMemsetAsync(d, 0, n, st)); return 0; }
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

/* ----------------------------------------------------------- kernel params */
struct FuncOut {               /* where a function's result lives (device)       */
    cl_func f;
    uint32_t inst_start, n_inst, imm_start, n_imm, val_start, ev_start, n_ev, pad;
};
enum { CUR_INST = 0, CUR_IMM, CUR_VAL, CUR_EV, CUR__N };

struct KArgs {
    cl_corpus in;              /* device pointers                               */
    const cl_pattern_blob *pb;
    const uint8_t *opflags;
    /* results: dense, in completion order; FuncOut says where                 */
    cl_hdr *o_hdr; uint16_t *o_tag; uint32_t *o_pay;
    cl_imm *o_imm;
    uint8_t *o_alive; int32_t *o_def_iid; uint32_t *o_origin;
    uint16_t *o_ext_tag; uint32_t *o_ext_pay; cl_memref *o_mem;      /* input offsets */
    cl_blk *o_blk; uint32_t *o_blk_start, *o_blk_cnt;                /* by global block */
    cl_event *o_ev;
    FuncOut *o_func;
    unsigned long long cap[CUR__N];
    unsigned long long *cursor;          /* [CUR__N]                            */
    unsigned long long *stats;           /* cl_stats as u64[]                   */
    /* work */
    const uint32_t *list; uint32_t n_list; uint32_t *work_counter;
    uint8_t *scratch; unsigned long long scratch_per_group;
    Caps gcap;                 /* capacities of the scratch placement            */
    uint32_t hot_bytes;        /* shared memory per group for the hot arrays     */
    uint32_t passes, max_rounds, emit_matches, raw_passes;
    const cl_sr_entry *sr; uint32_t n_sr;
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
    s.cand = carve<uint32_t>(p, c.I);
    s.sel_at = carve<uint32_t>(p, c.I);
    s.owner = carve<unsigned long long>(p, c.I);
    s.mt = carve<MatchRec>(p, c.M);
    s.sel = carve<SelRec>(p, c.S);
    s.plan = carve<Plan>(p, c.S);
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
    const cl_corpus &in = a.in;
    const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
    const uint32_t i0 = in.blk_off[b0], i1 = in.blk_off[b1];
    const cl_func fn = in.func[f];
    s.f = f; s.arch = fn.arch;
    s.nb = b1 - b0; s.n = i1 - i0;
    s.next_vid = fn.next_vid; s.next_iid = fn.next_iid;
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

template <class G> CLF void store_function(const G &g, FS &s, const KArgs &a, uint32_t f, uint32_t next_temp) {
    const uint32_t st = status(s);
    const uint32_t n_ev = *s.n_ev <= s.cap.E ? *s.n_ev : s.cap.E;
    uint32_t r_inst = 0, r_imm = 0, r_val = 0, r_ev = 0;
    if (g.rank == 0) {
        r_inst = (uint32_t)a_add64(&a.cursor[CUR_INST], s.n);
        r_imm = (uint32_t)a_add64(&a.cursor[CUR_IMM], s.n_imm);
        r_val = (uint32_t)a_add64(&a.cursor[CUR_VAL], s.next_vid);
        r_ev = (uint32_t)a_add64(&a.cursor[CUR_EV], n_ev);
    }
    r_inst = g.bcast0(r_inst); r_imm = g.bcast0(r_imm); r_val = g.bcast0(r_val); r_ev = g.bcast0(r_ev);
    const bool fits = (unsigned long long)r_inst + s.n <= a.cap[CUR_INST] && (unsigned long long)r_imm + s.n_imm <= a.cap[CUR_IMM] &&
                      (unsigned long long)r_val + s.next_vid <= a.cap[CUR_VAL] && (unsigned long long)r_ev + n_ev <= a.cap[CUR_EV];
    const uint32_t b0 = a.in.func_blk_off[f];
    if (g.rank == 0) {
        FuncOut o;
        o.f.next_vid = s.next_vid; o.f.next_iid = s.next_iid; o.f.next_temp_reg = next_temp;
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

/* one function, start to finish, on one group                               */
template <class G> CLF void process_function(const G &g, FS &s, const KArgs &a, uint32_t f, uint8_t *hot,
                                             uint8_t *cold) {
    const cl_corpus &in = a.in;
    const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
    const uint32_t n_in = in.blk_off[b1] - in.blk_off[b0];
    const uint32_t nv_in = in.func[f].next_vid;
    uint32_t next_temp = in.func[f].next_temp_reg;
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
        if (a.raw_passes) {
            /* raw stage kernels live in raw.cuh */
        } else if (a.passes & CL_PASS_MATCH_ONLY) run_match_only(g, s);
        else run_postssa(g, s);
        g.sync();
        if (status(s) == CL_ST_CAPACITY && use_hot) { use_hot = false; g.sync(); continue; }
        break;
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
    store_function(g, s, a, f, next_temp);
    g.sync();
}

/* persistent group loop                                                      */
template <class G> CLF void group_loop(const G &g, const KArgs &a, uint32_t *gw, uint8_t *hot, uint8_t *cold) {
    FS s;
    s.pb = a.pb; s.ms = a.in.modsets; s.opflags = a.opflags;
    s.passes = a.passes; s.max_rounds = a.max_rounds; s.emit_matches = a.emit_matches;
    s.st = gw + GW_STATUS; s.n_ev = gw + GW_NEV;
    s.st_matches = gw + GW_STATS; s.st_selected = gw + GW_STATS + 16;
    s.st_rewrites = gw + GW_STATS + 32; s.st_refused = gw + GW_STATS + 48;
    GFOR(g, k, GW__N) if (k < GW__N) gw[k] = 0;
    g.sync();
    unsigned long long n_in = 0, n_out = 0, n_ev = 0;
    for (;;) {
        uint32_t w = 0;
        if (g.rank == 0) w = a_add(a.work_counter, 1u);
        w = g.bcast0(w);
        if (w >= a.n_list) break;
        const uint32_t f = a.list[w];
        process_function(g, s, a, f, hot, cold);
        const uint32_t b0 = a.in.func_blk_off[f], b1 = a.in.func_blk_off[f + 1];
        n_in += a.in.blk_off[b1] - a.in.blk_off[b0];
        n_out += s.n; n_ev += *s.n_ev;
        g.sync();
    }
    if (g.rank == 0) {
        for (int k = 0; k < 64; k++) if (gw[GW_STATS + k]) a_add64(&a.stats[k], gw[GW_STATS + k]);
        a_add64(&a.stats[64], n_in); a_add64(&a.stats[65], n_out); a_add64(&a.stats[66], n_ev);
    }
}

#if CL_CUDA
/* one warp per function: 4 independent groups per CTA                        */
template <int WARPS> __global__ void __launch_bounds__(WARPS * 32) k_postssa_warp(KArgs a) {
    extern __shared__ uint4 dyn_smem[];
    __shared__ uint32_t gw[WARPS][GW__N];
    const uint32_t w = threadIdx.x >> 5;
    Grp<1> g; g.rank = threadIdx.x & 31u; g.size = 32; g.red = nullptr;
    const uint32_t gid = blockIdx.x * WARPS + w;
    uint8_t *hot = a.hot_bytes ? (uint8_t *)dyn_smem + (size_t)w * a.hot_bytes : nullptr;
    group_loop(g, a, gw[w], hot, a.scratch + (size_t)gid * a.scratch_per_group);
}
/* one CTA per function                                                       */
template <int WARPS> __global__ void __launch_bounds__(WARPS * 32) k_postssa_cta(KArgs a) {
    extern __shared__ uint4 dyn_smem[];
    __shared__ uint32_t gw[GW__N];
    __shared__ uint32_t red[WARPS + 2];
    Grp<WARPS> g; g.rank = threadIdx.x; g.size = WARPS * 32; g.red = red;
    uint8_t *hot = a.hot_bytes ? (uint8_t *)dyn_smem : nullptr;
    group_loop(g, a, gw, hot, a.scratch + (size_t)blockIdx.x * a.scratch_per_group);
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

struct cl_ctx {
    int device = 0;
    cudaStream_t stream = 0;
#if CL_CUDA
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int n_sm = 148;
#endif
    cl_pattern_blob h_pb{};
    bool have_pb = false, have_in = false, have_out = false;
    cl_pattern_blob *d_pb = nullptr;
    uint8_t *d_opflags = nullptr;
    /* host copy of the small arrays + device corpus */
    std::vector<cl_func> h_func;
    std::vector<uint32_t> h_fbo, h_ext_off, h_mem_off, h_imm_off, h_val_off, h_blk_off;
    std::vector<cl_blk> h_blk;
    cl_corpus d_in{};
    std::vector<void *> d_in_allocs;
    uint64_t n_inst = 0, n_ext = 0, n_mem = 0, n_imm = 0, n_val = 0;
    /* results */
    KArgs k{};
    std::vector<void *> d_out_allocs;
    unsigned long long *d_cursor = nullptr, *d_stats = nullptr;
    unsigned long long h_cursor[CUR__N] = { 0, 0, 0, 0 };
    Part part[2];              /* 0 = warp groups, 1 = CTA groups                */
    cl_stats stats{};
    float last_ms = 0;
    uint32_t small_max = 128;  /* records: warp-group kernel up to here          */
};

static void free_list(std::vector<void *> &v) { for (void *p : v) dfree(p); v.clear(); }
template <class T> static int dalloc(cl_ctx *c, std::vector<void *> &pool, T **p, size_t n) {
    (void)c;
    void *q = nullptr;
    if (dmalloc(&q, n * sizeof(T))) return -1;
    pool.push_back(q);
    *p = (T *)q;
    return 0;
}
template <class T> static int dupload(cl_ctx *c, std::vector<void *> &pool, T **p, const T *h, size_t n) {
    if (dalloc(c, pool, p, n)) return -1;
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
#endif
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
    *out = c;
    return 0;
}

static void free_parts(cl_ctx *c) {
    for (Part &p : c->part) {
        dfree(p.d_list); dfree(p.d_counter); dfree(p.d_scratch);
        p = Part();
    }
}
extern "C" void cl_destroy(cl_ctx *c) {
    if (!c) return;
#if CL_CUDA
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
#endif
    free_list(c->d_in_allocs); free_list(c->d_out_allocs); free_parts(c);
    dfree(c->d_opflags); dfree(c->d_pb); dfree(c->d_cursor); dfree(c->d_stats);
#if CL_CUDA
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
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
    free_list(c->d_in_allocs); free_list(c->d_out_allocs); free_parts(c);
    c->have_in = c->have_out = false;
    const uint32_t F = in->n_funcs, B = in->n_blocks;
    if (in->func_blk_off[F] != B) FAIL("func_blk_off[n_funcs] != n_blocks");
    c->n_inst = in->blk_off[B]; c->n_ext = in->ext_off[F]; c->n_mem = in->mem_off[F];
    c->n_imm = in->imm_off[F]; c->n_val = in->val_off[F];
    c->h_func.assign(in->func, in->func + F);
    c->h_fbo.assign(in->func_blk_off, in->func_blk_off + F + 1);
    c->h_ext_off.assign(in->ext_off, in->ext_off + F + 1);
    c->h_mem_off.assign(in->mem_off, in->mem_off + F + 1);
    c->h_imm_off.assign(in->imm_off, in->imm_off + F + 1);
    c->h_val_off.assign(in->val_off, in->val_off + F + 1);
    c->h_blk_off.assign(in->blk_off, in->blk_off + B + 1);
    c->h_blk.assign(in->blk, in->blk + B);
    for (uint32_t f = 0; f < F; f++)
        if (in->val_off[f + 1] - in->val_off[f] != in->func[f].next_vid)
            FAIL("function %u: value region holds %u entries, next_vid is %u", f, in->val_off[f + 1] - in->val_off[f], in->func[f].next_vid);
    cl_corpus &d = c->d_in;
    d = *in;
    auto &pool = c->d_in_allocs;
    if (dupload(c, pool, &d.func, in->func, F) || dupload(c, pool, &d.func_blk_off, in->func_blk_off, F + 1) ||
        dupload(c, pool, &d.ext_off, in->ext_off, F + 1) || dupload(c, pool, &d.mem_off, in->mem_off, F + 1) ||
        dupload(c, pool, &d.imm_off, in->imm_off, F + 1) || dupload(c, pool, &d.val_off, in->val_off, F + 1) ||
        dupload(c, pool, &d.blk, in->blk, B) || dupload(c, pool, &d.blk_off, in->blk_off, B + 1) ||
        dupload(c, pool, &d.hdr, in->hdr, c->n_inst) || dupload(c, pool, &d.tag, in->tag, c->n_inst * 8) ||
        dupload(c, pool, &d.pay, in->pay, c->n_inst * 8) || dupload(c, pool, &d.ext_tag, in->ext_tag, c->n_ext) ||
        dupload(c, pool, &d.ext_pay, in->ext_pay, c->n_ext) || dupload(c, pool, &d.mem, in->mem, c->n_mem) ||
        dupload(c, pool, &d.imm, in->imm, c->n_imm) || dupload(c, pool, &d.val_alive, in->val_alive, c->n_val) ||
        dupload(c, pool, &d.val_def_iid, in->val_def_iid, c->n_val))
        return -1;
    cl_modset *dms = nullptr;
    if (dupload(c, pool, &dms, in->modsets, in->n_modsets)) return -1;
    d.modsets = dms;
    d.val_origin = nullptr;

    /* work partition: warp groups take the small functions */
    uint32_t n_max[2] = { 0, 0 }, nv_max[2] = { 0, 0 }, nb_max[2] = { 0, 0 }, imm_max[2] = { 0, 0 }, blk_max[2] = { 0, 0 }, ext_max[2] = { 0, 0 };
    for (uint32_t f = 0; f < F; f++) {
        const uint32_t b0 = in->func_blk_off[f], b1 = in->func_blk_off[f + 1];
        const uint32_t n = in->blk_off[b1] - in->blk_off[b0];
        const int k = n <= c->small_max ? 0 : 1;
        c->part[k].list.push_back(f);
        n_max[k] = std::max(n_max[k], n);
        nv_max[k] = std::max(nv_max[k], in->func[f].next_vid);
        nb_max[k] = std::max(nb_max[k], b1 - b0);
        imm_max[k] = std::max(imm_max[k], in->imm_off[f + 1] - in->imm_off[f]);
        ext_max[k] = std::max(ext_max[k], in->ext_off[f + 1] - in->ext_off[f]);
        for (uint32_t b = b0; b < b1; b++) blk_max[k] = std::max(blk_max[k], in->blk_off[b + 1] - in->blk_off[b]);
    }
    /* big functions first: the tail of the work list is cheap */
    for (int k = 0; k < 2; k++) {
        Part &p = c->part[k];
        std::stable_sort(p.list.begin(), p.list.end(), [&](uint32_t x, uint32_t y) {
            const uint32_t nx = in->blk_off[in->func_blk_off[x + 1]] - in->blk_off[in->func_blk_off[x]];
            const uint32_t ny = in->blk_off[in->func_blk_off[y + 1]] - in->blk_off[in->func_blk_off[y]];
            return nx > ny;
        });
        if (p.list.empty()) continue;
        p.cap = caps_for(n_max[k], nv_max[k], nb_max[k], imm_max[k], blk_max[k], ext_max[k]);
        p.scratch_per_group = (scratch_bytes(p.cap) + 255) & ~(size_t)255;
#if CL_CUDA
        if (k == 0) { p.hot_bytes = 12 * 1024; p.grid = c->n_sm * 4; p.n_groups = p.grid * 4; }
        else { p.hot_bytes = 100 * 1024; p.grid = c->n_sm * 2; p.n_groups = p.grid; }
        p.grid = (uint32_t)std::min<size_t>(p.grid, k == 0 ? (p.list.size() + 3) / 4 : p.list.size());
        p.n_groups = k == 0 ? p.grid * 4 : p.grid;
#else
        p.hot_bytes = 0; p.grid = 1; p.n_groups = 1;
#endif
        void *q = nullptr;
        if (dmalloc(&q, p.list.size() * sizeof(uint32_t))) return -1;
        p.d_list = (uint32_t *)q;
        if (h2d(p.d_list, p.list.data(), p.list.size() * sizeof(uint32_t), c->stream)) return -1;
        if (dmalloc(&q, sizeof(uint32_t))) return -1;
        p.d_counter = (uint32_t *)q;
        if (dmalloc(&q, p.scratch_per_group * p.n_groups)) return -1;
        p.d_scratch = (uint8_t *)q;
    }

    /* result buffers (worst-case growth, G3/G4) */
    KArgs &k = c->k;
    memset(&k, 0, sizeof k);
    k.in = d; k.pb = c->d_pb; k.opflags = c->d_opflags;
    k.cap[CUR_INST] = 3 * c->n_inst + 1024;
    k.cap[CUR_IMM] = c->n_imm + 2 * c->n_inst + 1024;
    k.cap[CUR_VAL] = c->n_val + 2 * c->n_inst + 1024;
    k.cap[CUR_EV] = 2 * c->n_inst + 4096;
    auto &op = c->d_out_allocs;
    if (dalloc(c, op, &k.o_hdr, k.cap[CUR_INST]) || dalloc(c, op, &k.o_tag, k.cap[CUR_INST] * 8) ||
        dalloc(c, op, &k.o_pay, k.cap[CUR_INST] * 8) || dalloc(c, op, &k.o_imm, k.cap[CUR_IMM]) ||
        dalloc(c, op, &k.o_alive, k.cap[CUR_VAL]) || dalloc(c, op, &k.o_def_iid, k.cap[CUR_VAL]) ||
        dalloc(c, op, &k.o_origin, k.cap[CUR_VAL]) || dalloc(c, op, &k.o_ext_tag, c->n_ext) ||
        dalloc(c, op, &k.o_ext_pay, c->n_ext) || dalloc(c, op, &k.o_mem, c->n_mem) ||
        dalloc(c, op, &k.o_blk, B) || dalloc(c, op, &k.o_blk_start, B) || dalloc(c, op, &k.o_blk_cnt, B) ||
        dalloc(c, op, &k.o_ev, k.cap[CUR_EV]) || dalloc(c, op, &k.o_func, F))
        return -1;
    k.cursor = c->d_cursor; k.stats = c->d_stats;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    c->have_in = true;
    return 0;
}

static int launch_part(cl_ctx *c, int which, KArgs k) {
    Part &p = c->part[which];
    if (p.list.empty()) return 0;
    k.list = p.d_list; k.n_list = (uint32_t)p.list.size(); k.work_counter = p.d_counter;
    k.scratch = p.d_scratch; k.scratch_per_group = p.scratch_per_group; k.gcap = p.cap; k.hot_bytes = p.hot_bytes;
    if (dzero(p.d_counter, sizeof(uint32_t), c->stream)) return -1;
#if CL_CUDA
    if (which == 0) {
        const size_t smem = (size_t)p.hot_bytes * 4;
        CUDA_OK(cudaFuncSetAttribute(k_postssa_warp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_postssa_warp<4><<<p.grid, 128, smem, c->stream>>>(k);
    } else {
        const size_t smem = p.hot_bytes;
        CUDA_OK(cudaFuncSetAttribute(k_postssa_cta<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_postssa_cta<8><<<p.grid, 256, smem, c->stream>>>(k);
    }
    CUDA_OK(cudaGetLastError());
#else
    static uint32_t gw[GW__N];
    Grp<0> g; g.rank = 0; g.size = 1; g.red = nullptr;
    group_loop(g, k, gw, (uint8_t *)nullptr, k.scratch);
#endif
    return 0;
}

static int run(cl_ctx *c, KArgs k) {
    if (!c->have_in) FAIL("no corpus uploaded");
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
#endif
    if (dzero(c->d_cursor, sizeof(unsigned long long) * CUR__N, c->stream)) return -1;
    if (dzero(c->d_stats, sizeof(cl_stats), c->stream)) return -1;
#if CL_CUDA
    CUDA_OK(cudaEventRecord(c->ev0, c->stream));
#endif
    if (launch_part(c, 1, k)) return -1;       /* the long poles first */
    if (launch_part(c, 0, k)) return -1;
#if CL_CUDA
    CUDA_OK(cudaEventRecord(c->ev1, c->stream));
#endif
    if (d2h(c->h_cursor, c->d_cursor, sizeof c->h_cursor, c->stream)) return -1;
    if (d2h(&c->stats, c->d_stats, sizeof(cl_stats), c->stream)) return -1;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
    CUDA_OK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
#endif
    c->have_out = true;
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
    (void)c; (void)passes; (void)map; (void)n_map;
    FAIL("cl_run_raw: the raw stage is not built yet");
}

extern "C" int cl_out_sizes(cl_ctx *c, uint64_t sizes[6]) {
    if (!c->have_out) FAIL("no result: call cl_run_* first");
    sizes[0] = c->h_cursor[CUR_INST]; sizes[1] = c->n_ext; sizes[2] = c->n_mem;
    sizes[3] = c->h_cursor[CUR_IMM]; sizes[4] = c->h_cursor[CUR_VAL]; sizes[5] = c->h_cursor[CUR_EV];
    for (int i = 0; i < CUR__N; i++)
        if (c->h_cursor[i] > c->k.cap[i]) FAIL("result stream %d overflowed its capacity (%llu > %llu)", i, c->h_cursor[i], c->k.cap[i]);
    return 0;
}

/* D2H, then densify: the device wrote functions in completion order; the ABI
 * returns them in function order (dense CSR).                               */
extern "C" int cl_download(cl_ctx *c, cl_corpus *o, cl_event *events) {
    uint64_t sz[6];
    if (cl_out_sizes(c, sz)) return -1;
    const uint32_t F = (uint32_t)c->h_func.size(), B = (uint32_t)c->h_blk.size();
    const KArgs &k = c->k;
    std::vector<FuncOut> fo(F);
    std::vector<cl_hdr> hdr(sz[0]); std::vector<uint16_t> tag(sz[0] * 8); std::vector<uint32_t> pay(sz[0] * 8);
    std::vector<cl_imm> imm(sz[3]);
    std::vector<uint8_t> alive(sz[4]); std::vector<int32_t> def_iid(sz[4]); std::vector<uint32_t> origin(sz[4]);
    std::vector<cl_event> ev(sz[5]);
    std::vector<uint32_t> bstart(B), bcnt(B);
#if CL_CUDA
    CUDA_OK(cudaSetDevice(c->device));
#endif
    if (d2h(fo.data(), k.o_func, F * sizeof(FuncOut), c->stream) || d2h(hdr.data(), k.o_hdr, sz[0] * sizeof(cl_hdr), c->stream) ||
        d2h(tag.data(), k.o_tag, sz[0] * 16, c->stream) || d2h(pay.data(), k.o_pay, sz[0] * 32, c->stream) ||
        d2h(imm.data(), k.o_imm, sz[3] * sizeof(cl_imm), c->stream) || d2h(alive.data(), k.o_alive, sz[4], c->stream) ||
        d2h(def_iid.data(), k.o_def_iid, sz[4] * 4, c->stream) || d2h(origin.data(), k.o_origin, sz[4] * 4, c->stream) ||
        d2h(ev.data(), k.o_ev, sz[5] * sizeof(cl_event), c->stream) || d2h(bstart.data(), k.o_blk_start, B * 4ull, c->stream) ||
        d2h(bcnt.data(), k.o_blk_cnt, B * 4ull, c->stream) || d2h(o->blk, k.o_blk, B * sizeof(cl_blk), c->stream) ||
        d2h(o->ext_tag, k.o_ext_tag, c->n_ext * 2, c->stream) || d2h(o->ext_pay, k.o_ext_pay, c->n_ext * 4, c->stream) ||
        d2h(o->mem, k.o_mem, c->n_mem * sizeof(cl_memref), c->stream))
        return -1;
#if CL_CUDA
    CUDA_OK(cudaStreamSynchronize(c->stream));
#endif
    o->n_funcs = F; o->n_blocks = B; o->n_modsets = c->d_in.n_modsets;
    uint64_t ni = 0, nq = 0, nv = 0, ne = 0;
    for (uint32_t f = 0; f < F; f++) {
        const FuncOut &r = fo[f];
        o->func[f] = r.f;
        o->func_blk_off[f] = c->h_fbo[f]; o->ext_off[f] = c->h_ext_off[f]; o->mem_off[f] = c->h_mem_off[f];
        o->imm_off[f] = (uint32_t)nq; o->val_off[f] = (uint32_t)nv;
        for (uint32_t b = c->h_fbo[f]; b < c->h_fbo[f + 1]; b++) {
            o->blk_off[b] = (uint32_t)ni;
            if (bcnt[b]) {
                memcpy(o->hdr + ni, hdr.data() + bstart[b], sizeof(cl_hdr) * bcnt[b]);
                memcpy(o->tag + ni * 8, tag.data() + (size_t)bstart[b] * 8, 16ull * bcnt[b]);
                memcpy(o->pay + ni * 8, pay.data() + (size_t)bstart[b] * 8, 32ull * bcnt[b]);
            }
            ni += bcnt[b];
        }
        if (r.n_imm) memcpy(o->imm + nq, imm.data() + r.imm_start, sizeof(cl_imm) * r.n_imm);
        nq += r.n_imm;
        const uint32_t nvf = r.f.next_vid;
        if (nvf) {
            memcpy(o->val_alive + nv, alive.data() + r.val_start, nvf);
            memcpy(o->val_def_iid + nv, def_iid.data() + r.val_start, 4ull * nvf);
            memcpy(o->val_origin + nv, origin.data() + r.val_start, 4ull * nvf);
        }
        nv += r.f.next_vid;
        if (events && r.n_ev) memcpy(events + ne, ev.data() + r.ev_start, sizeof(cl_event) * r.n_ev);
        ne += r.n_ev;
    }
    o->func_blk_off[F] = B; o->ext_off[F] = c->h_ext_off[F]; o->mem_off[F] = c->h_mem_off[F];
    o->imm_off[F] = (uint32_t)nq; o->val_off[F] = (uint32_t)nv; o->blk_off[B] = (uint32_t)ni;
    if (events)
        std::sort(events, events + ne, [](const cl_event &x, const cl_event &y) {
            const uint32_t *a = (const uint32_t *)&x, *b = (const uint32_t *)&y;
            for (int i = 0; i < 8; i++) if (a[i] != b[i]) return a[i] < b[i];
            return false;
        });
    return 0;
}

extern "C" int cl_get_stats(cl_ctx *c, cl_stats *out) { *out = c->stats; return 0; }
extern "C" int cl_last_run_ms(cl_ctx *c, float *ms) { *ms = c->last_ms; return 0; }
extern "C" void *cl_device_counts_ptr(cl_ctx *c) { return c->d_stats; }
extern "C" void *cl_stream(cl_ctx *c) { return (void *)(uintptr_t)c->stream; }
