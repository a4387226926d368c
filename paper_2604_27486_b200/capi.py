"""ctypes binding of the C ABI in ``include/culifter.h``.

``Engine()`` loads the product library (``csrc/libculifter.so``: sm_100a CUDA
kernels).  There is no CPU fallback: if the library is missing or no CUDA
device answers, construction raises.  Tests and ``bench.py``'s CPU-baseline
leg may point ``Engine`` at the oracle library explicitly (``Engine(path)``);
nothing in the package does.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import layout as L
from .patterns import BLOB, PATTERN, SLOT, TEMPLATE, compile_patterns
from .soa import Corpus

# Streams are multiplexed onto CUDA_DEVICE_MAX_CONNECTIONS hardware queues (default 8); two streams that share a
# queue serialise falsely.  The pipeline runs 2 streams per context: measured on B200, a chunk's kernels waited a full
# H2D copy of another context (+50 % run time on every other chunk) with the default.  Read when the CUDA context
# is created, so it has to be in the environment before the first CUDA call of the process.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

PKG = Path(__file__).resolve().parent
PRODUCT_LIB = PKG / "csrc" / "libculifter.so"

SR_ENTRY = np.dtype([("arch", "<u4"), ("offset", "<u4"), ("sreg", "<u4")])
STATS = np.dtype([("matches", "<u8", (16,)), ("selected", "<u8", (16,)),
                  ("rewrites", "<u8", (16,)), ("refused", "<u8", (16,)),
                  ("n_inst_in", "<u8"), ("n_inst_out", "<u8"), ("n_events", "<u8"),
                  ("reserved", "<u8")])


class CorpusStruct(C.Structure):
    _fields_ = [("n_funcs", C.c_uint32), ("n_blocks", C.c_uint32),
                ("n_modsets", C.c_uint32), ("reserved", C.c_uint32)] + \
        [(name, C.c_void_p) for name in (
            "func", "func_blk_off", "ext_off", "mem_off", "imm_off", "val_off", "blk",
            "blk_off", "hdr", "tag", "pay", "ext_tag", "ext_pay", "mem", "imm",
            "val_alive", "val_def_iid", "val_origin", "modsets")]


class RunOpts(C.Structure):
    _fields_ = [("passes", C.c_uint32), ("max_rounds", C.c_uint32),
                ("emit_matches", C.c_uint32), ("reserved", C.c_uint32)]


_ABI_SIZES = (L.HDR.itemsize, L.IMM.itemsize, L.MEMREF.itemsize, L.BLK.itemsize,
              L.FUNC.itemsize, L.MODSET.itemsize, SLOT.itemsize, TEMPLATE.itemsize,
              PATTERN.itemsize, BLOB.itemsize, L.EVENT.itemsize, C.sizeof(CorpusStruct),
              C.sizeof(RunOpts), STATS.itemsize, SR_ENTRY.itemsize)

EXPORTS = ("cl_last_error", "cl_backend", "cl_abi_sizeof", "cl_create", "cl_destroy",
           "cl_set_patterns", "cl_set_threads", "cl_upload", "cl_run_postssa", "cl_run_raw",
           "cl_out_sizes", "cl_download", "cl_get_stats", "cl_last_run_ms",
           "cl_device_counts_ptr", "cl_stream")


class EngineError(RuntimeError):
    pass


def load_library(path=None):
    import os
    if path is None and os.environ.get("CL_LIB"):      # development knob: another build of the CUDA library
        path = os.environ["CL_LIB"]
    path = Path(path) if path is not None else PRODUCT_LIB
    if not path.exists():
        raise EngineError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(str(path))
    for name in EXPORTS:
        if not hasattr(lib, name):
            raise EngineError(f"{path}: symbol {name} is not exported")
    lib.cl_last_error.restype = C.c_char_p
    lib.cl_backend.restype = C.c_char_p
    lib.cl_abi_sizeof.restype = C.c_long
    lib.cl_device_counts_ptr.restype = C.c_void_p
    lib.cl_stream.restype = C.c_void_p
    lib.cl_device_counts_ptr.argtypes = lib.cl_stream.argtypes = [C.c_void_p]
    lib.cl_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.cl_destroy.argtypes = [C.c_void_p]
    lib.cl_destroy.restype = None
    lib.cl_set_patterns.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    lib.cl_set_threads.argtypes = [C.c_void_p, C.c_int]
    lib.cl_upload.argtypes = [C.c_void_p, C.POINTER(CorpusStruct)]
    lib.cl_run_postssa.argtypes = [C.c_void_p, C.POINTER(RunOpts)]
    lib.cl_run_raw.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
    lib.cl_out_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    lib.cl_download.argtypes = [C.c_void_p, C.POINTER(CorpusStruct), C.c_void_p]
    lib.cl_get_stats.argtypes = [C.c_void_p, C.c_void_p]
    lib.cl_last_run_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
    for i, want in enumerate(_ABI_SIZES):
        got = lib.cl_abi_sizeof(i)
        if got != want:
            raise EngineError(f"{path}: ABI struct {i} is {got} bytes, binding expects {want}")
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _struct_of(c: Corpus, modsets: np.ndarray) -> CorpusStruct:
    st = CorpusStruct()
    st.n_funcs, st.n_blocks, st.n_modsets = c.n_funcs, c.n_blocks, len(modsets)
    for name in Corpus.ARRAYS:
        a = getattr(c, name)
        if not a.flags["C_CONTIGUOUS"]:
            raise EngineError(f"corpus array {name} is not contiguous")
        setattr(st, name, _ptr(a))
    st.modsets = _ptr(modsets)
    return st


class Engine:
    """One ``cl_ctx``: a device (or, for the oracle library, host threads)."""

    def __init__(self, lib_path=None, device: int = 0, patterns=None):
        self.lib = load_library(lib_path)
        self.backend = self.lib.cl_backend().decode()
        self._ctx = C.c_void_p()
        self._check(self.lib.cl_create(device, C.byref(self._ctx)))
        self._blob = None
        self._n_blocks = 0
        self._keep = None
        self.set_patterns(*(patterns or (None, None)))

    def _check(self, rc):
        if rc != 0:
            raise EngineError(f"{self.backend}: {self.lib.cl_last_error().decode()}")

    def close(self):
        if self._ctx:
            self.lib.cl_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def set_patterns(self, aggregation=None, xmad=None, budget=50_000):
        self._blob = compile_patterns(aggregation, xmad, budget)
        self._tables = (list(aggregation) if aggregation is not None else None, list(xmad) if xmad is not None else None)
        self._check(self.lib.cl_set_patterns(self._ctx, _ptr(self._blob), self._blob.nbytes))

    def pattern_blob(self):
        """The compiled table the device holds (``restore_patterns`` puts it back)."""
        return self._blob, self._tables

    def restore_patterns(self, saved):
        self._blob, self._tables = saved
        self._check(self.lib.cl_set_patterns(self._ctx, _ptr(self._blob), self._blob.nbytes))

    def pattern_names(self):
        """Names of the device table's patterns in table order (aggregation, then xmad): what a
        CL_EV_REFUSED / CL_EV_MATCH event's pattern index refers to."""
        from .patterns import AGGREGATION_PATTERNS, XMAD_PATTERNS
        agg, xm = self._tables
        return [p.name for p in (AGGREGATION_PATTERNS if agg is None else agg)] + [p.name for p in (XMAD_PATTERNS if xm is None else xm)]

    def set_threads(self, n: int):
        self._check(self.lib.cl_set_threads(self._ctx, n))

    def upload(self, corpus: Corpus):
        modsets = np.ascontiguousarray(L.TABLES.modset_info())
        st = _struct_of(corpus, modsets)
        self._keep = (corpus, modsets)
        self._check(self.lib.cl_upload(self._ctx, C.byref(st)))
        self._src = corpus

    def run_postssa(self, passes=L.PASS_ALL, max_rounds=4, emit_matches=False):
        opts = RunOpts(passes, max_rounds, int(emit_matches), 0)
        self._check(self.lib.cl_run_postssa(self._ctx, C.byref(opts)))

    def run_raw(self, passes, sr_map=()):
        m = np.array([tuple(e) for e in sr_map], SR_ENTRY) if len(sr_map) else np.zeros(0, SR_ENTRY)
        self._check(self.lib.cl_run_raw(self._ctx, passes, _ptr(m), len(m)))

    def download(self, into: Corpus | None = None) -> Corpus:
        """Result of the last run as a dense corpus.  ``into``: caller-owned arrays
        (e.g. pinned host memory) at least as large as the result; the returned
        corpus is made of views of them trimmed to the actual sizes."""
        sizes = (C.c_uint64 * 6)()
        self._check(self.lib.cl_out_sizes(self._ctx, sizes))
        n_inst, n_ext, n_mem, n_imm, n_val, n_ev = (int(x) for x in sizes)
        src = self._src
        F, B = src.n_funcs, src.n_blocks
        want = dict(func=F, func_blk_off=F + 1, ext_off=F + 1, mem_off=F + 1, imm_off=F + 1, val_off=F + 1,
                    blk=B, blk_off=B + 1, hdr=n_inst, tag=n_inst, pay=n_inst, ext_tag=n_ext, ext_pay=n_ext,
                    mem=n_mem, imm=n_imm, val_alive=n_val, val_def_iid=n_val, val_origin=n_val)
        if into is not None:
            for name, n in want.items():
                if len(getattr(into, name)) < n:
                    raise EngineError(f"download: array {name} holds {len(getattr(into, name))} rows, result has {n}")
            if len(into.events) < n_ev:
                raise EngineError(f"download: events array holds {len(into.events)} rows, result has {n_ev}")
            out = Corpus(**{name: getattr(into, name)[:n] for name, n in want.items()},
                         events=into.events[:n_ev], functions=src.functions, raw=src.raw)
        else:
            out = Corpus(
                func=np.zeros(F, L.FUNC), func_blk_off=np.zeros(F + 1, np.uint32),
                ext_off=np.zeros(F + 1, np.uint32), mem_off=np.zeros(F + 1, np.uint32),
                imm_off=np.zeros(F + 1, np.uint32), val_off=np.zeros(F + 1, np.uint32),
                blk=np.zeros(B, L.BLK), blk_off=np.zeros(B + 1, np.uint32),
                hdr=np.zeros(n_inst, L.HDR), tag=np.zeros((n_inst, 8), np.uint16),
                pay=np.zeros((n_inst, 8), np.uint32), ext_tag=np.zeros(n_ext, np.uint16),
                ext_pay=np.zeros(n_ext, np.uint32), mem=np.zeros(n_mem, L.MEMREF),
                imm=np.zeros(n_imm, L.IMM), val_alive=np.zeros(n_val, np.uint8),
                val_def_iid=np.zeros(n_val, np.int32), val_origin=np.zeros(n_val, np.uint32),
                events=np.zeros(n_ev, L.EVENT), functions=src.functions, raw=src.raw)
        st = _struct_of(out, self._keep[1])
        self._check(self.lib.cl_download(self._ctx, C.byref(st), _ptr(out.events)))
        return out

    def stats(self):
        s = np.zeros(1, STATS)
        self._check(self.lib.cl_get_stats(self._ctx, _ptr(s)))
        return s[0]

    def last_run_ms(self) -> float:
        ms = C.c_float()
        self._check(self.lib.cl_last_run_ms(self._ctx, C.byref(ms)))
        return float(ms.value)

    PROFILE_SLOTS = ("total", "load", "store", "usecount", "seed", "match", "select", "plan+emit", "emit",
                     "move", "simplify", "dce", "recip", "tag", "setup", "-")

    def debug_profile(self):
        """Per-phase cycle sums (lane 0 of every group) of the last run; CUDA library only."""
        if not hasattr(self.lib, "cl_debug_profile"):
            return {}
        buf = (C.c_ulonglong * 16)()
        self.lib.cl_debug_profile(self._ctx, buf, 16)
        return dict(zip(self.PROFILE_SLOTS, (int(x) for x in buf)))


    def debug_partition(self):
        """{tiles, tile_funcs, handed_back, outside, used_tiles} of the last run (CUDA / sim builds only)."""
        if not hasattr(self.lib, "cl_debug_partition"):
            return None
        out = (C.c_uint64 * 8)()
        self.lib.cl_debug_partition.argtypes = [C.c_void_p, C.c_void_p]
        self.lib.cl_debug_partition(self._ctx, out)
        return dict(zip(("tiles", "tile_funcs", "handed_back", "outside", "used_tiles", "launches", "tile_mode", "tile_cfg"),
                        (int(x) for x in out)))

    def device_counts_ptr(self):
        return self.lib.cl_device_counts_ptr(self._ctx)

    def stream(self):
        return self.lib.cl_stream(self._ctx)


class Pipeline:
    """Chunks of a corpus through ``depth`` contexts of one device, so that the
    host-to-device copy of one chunk, the kernels of another and the
    device-to-host copy of a third overlap (each context has its own streams).
    Functions are independent (``ssir.py:215-235``), so a chunk is any
    contiguous function range (``Corpus.split`` / ``Corpus.slice_funcs``) and
    the results are those of one big run, chunk by chunk."""

    def __init__(self, device: int = 0, depth: int = 3, lib_path=None, patterns=None, runners: int = 1):
        self.engines = [Engine(lib_path, device, patterns) for _ in range(max(1, depth))]
        self.runners = runners

    def close(self):
        for e in self.engines:
            e.close()

    def run_postssa(self, chunks, passes=L.PASS_ALL, max_rounds=4, into=None):
        """``chunks``: list of corpora (pinned host arrays make the copies
        asynchronous); ``into``: optional list of result holders (see
        ``Engine.download``).  Returns (results, summed stats, device ms summed over chunks).

        Three stage threads (upload, run, download) hand chunks to each other
        through queues; chunk k lives in context k mod depth from its upload to
        its download.  Symmetric workers (one thread per context doing all three
        steps) fall into lock step -- all upload, then all run, then all
        download -- and overlap nothing (measured)."""
        import queue
        import threading
        import time
        n = len(chunks)
        results, stats, ms, trace = [None] * n, [None] * n, [0.0] * n, [[0, 0.0, 0.0, 0.0, 0.0, 0.0] for _ in range(n)]
        errors = []
        t_begin = time.perf_counter()
        q_run, q_down = queue.Queue(), queue.Queue()
        # chunk k always takes context k mod depth: a context sees the same chunks every time the same list is
        # streamed again, so its grow-only device buffers stop growing (a reallocation synchronises the device)
        depth = len(self.engines)
        free = [threading.Semaphore(1) for _ in range(depth)]
        import os
        strict = os.environ.get("CL_PIPE_STRICT", "1") != "0"
        # two run threads: the tail of one chunk's persistent kernels overlaps the head of the next chunk's
        n_runners = max(1, min(int(os.environ.get("CL_PIPE_RUNNERS", self.runners)), depth))
        done, done_lock = [0], threading.Lock()
        free_q = queue.Queue()
        for i in range(depth):
            free_q.put(i)

        def now():
            return time.perf_counter() - t_begin

        def uploader():
            try:
                for k in range(n):
                    if strict:
                        i = k % depth
                        free[i].acquire()
                    else:
                        i = free_q.get()
                    if errors or i is None:
                        break
                    trace[k][0], trace[k][1] = i, now()
                    self.engines[i].upload(chunks[k])
                    trace[k][2] = now()
                    q_run.put((k, i))
            except Exception as e:  # noqa: BLE001 - re-raised on the caller's thread
                errors.append(e)
            for _ in range(n_runners):
                q_run.put(None)

        def runner():
            try:
                while True:
                    item = q_run.get()
                    if item is None or errors:
                        break
                    k, i = item
                    trace[k][3] = now()
                    self.engines[i].run_postssa(passes, max_rounds)
                    trace[k][4] = now()
                    q_down.put(item)
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                free_q.put(None)
                for sem in free:
                    sem.release()
            with done_lock:
                done[0] += 1
                if done[0] == n_runners:
                    q_down.put(None)

        def downloader():
            try:
                while True:
                    item = q_down.get()
                    if item is None or errors:
                        break
                    k, i = item
                    eng = self.engines[i]
                    results[k] = eng.download(into[k] if into is not None else None)
                    stats[k] = eng.stats().copy()
                    ms[k] = eng.last_run_ms()
                    trace[k][5] = now()
                    trace[k].append(ms[k])
                    free[i].release() if strict else free_q.put(i)
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                free_q.put(None)
                for sem in free:
                    sem.release()

        threads = [threading.Thread(target=f) for f in (uploader, downloader, *([runner] * n_runners))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        self.last_trace = trace      # per chunk: [context, upload start, upload end, run start, run end, download end] in seconds
        total = np.zeros(1, STATS)[0]
        for s in stats:
            for name in STATS.names:
                total[name] += s[name]
        return results, total, float(sum(ms))
