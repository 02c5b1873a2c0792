"""Thin ctypes binding of libautoscout.so (include/autoscout.h) -- argument marshalling only.

Every step of the scoring path runs in the library (host C++ for parsing/fit, sm_100a kernels
for scoring).  There is no Python or CPU fallback: if the shared library is missing this
module raises at import time, and scoring on a host-only handle raises AS_ERR_STATE.

Names mirror the C ABI (autoscout_space_create, autoscout_observe, autoscout_score_batch,
autoscout_topk, ...).  Device buffers are passed as raw pointers taken from torch tensors;
streams as the integer handle of a torch.cuda.Stream.
"""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AUTOSCOUT_LIB") or os.path.join(HERE, "libautoscout.so")   # env: dev A/B builds only

AS_MODE_RANGE, AS_MODE_SAMPLE = 0, 1
AS_ACQ_EI, AS_ACQ_LCB, AS_ACQ_SIM = 0, 1, 2
ACQ = {"ei": AS_ACQ_EI, "lcb": AS_ACQ_LCB, "sim": AS_ACQ_SIM}
AS_MODE_LIST = 2
MODE = {"range": AS_MODE_RANGE, "sample": AS_MODE_SAMPLE, "list": AS_MODE_LIST}
STATUS = {0: "AS_OK", 1: "AS_ERR_INVALID_ARG", 2: "AS_ERR_SPACE_SCHEMA", 3: "AS_ERR_SPACE_CYCLE",
          4: "AS_ERR_SPACE_ORDER", 5: "AS_ERR_SPACE_EMPTY", 6: "AS_ERR_INDEX_RANGE", 7: "AS_ERR_INVALID_CONFIG",
          8: "AS_ERR_NO_OBSERVATIONS", 9: "AS_ERR_NUMERIC", 10: "AS_ERR_CAPACITY", 11: "AS_ERR_STATE",
          12: "AS_ERR_UNCERTIFIED", 13: "AS_ERR_CUDA", 14: "AS_ERR_OOM"}
ENTRY_DTYPE = np.dtype([("score", "<f8"), ("raw", "<u8")])

EXPORTS = ["autoscout_space_create", "autoscout_space_destroy", "autoscout_space_info", "autoscout_observe",
           "autoscout_observe_clear", "autoscout_observe_info", "autoscout_score_batch", "autoscout_topk",
           "autoscout_topk_pool", "autoscout_topk_merge", "autoscout_decode", "autoscout_cvi_to_raw",
           "autoscout_sample_to_cvi", "autoscout_simulate", "autoscout_mask_range", "autoscout_set_path",
           "autoscout_set_timing", "autoscout_raw_to_cvi", "autoscout_subtree_range", "autoscout_neighbors",
           "autoscout_prior", "autoscout_ensemble_info", "autoscout_gp_lml", "autoscout_set_gp_hyper",
           "autoscout_ml2", "autoscout_set_slice", "autoscout_topk_pool_device", "autoscout_topk_merge_device",
           "autoscout_activity", "autoscout_set_async_observe",
           "autoscout_last_kernel_ms", "autoscout_last_phase_ms", "autoscout_last_error"]


class SpaceInfo(ctypes.Structure):
    _fields_ = [("n_raw", ctypes.c_uint64), ("n_cvi", ctypes.c_uint64), ("n_features", ctypes.c_int32),
                ("n_structures", ctypes.c_int32), ("n_prefix", ctypes.c_int32), ("n_components", ctypes.c_int32),
                ("n_observed", ctypes.c_int32), ("max_observed", ctypes.c_int32), ("n_launches", ctypes.c_uint64),
                ("fit_upload_bytes", ctypes.c_uint64)]


class ScoreArgs(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("acq", ctypes.c_int32), ("begin", ctypes.c_uint64),
                ("count", ctypes.c_uint64), ("seed", ctypes.c_uint64), ("kappa", ctypes.c_double),
                ("xi", ctypes.c_double), ("k", ctypes.c_int32), ("accumulate", ctypes.c_int32),
                ("d_scores", ctypes.c_void_p), ("d_raw", ctypes.c_void_p), ("d_valid_count", ctypes.c_void_p),
                ("d_positions", ctypes.c_void_p), ("d_screen", ctypes.c_void_p)]


class AutoscoutError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2603_11603_b200.build` "
                          "(there is no CPU fallback for the scoring path)")
    lib = ctypes.CDLL(LIB_PATH)
    P, U64, I32, I64, D = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pU64, pI32, pD = ctypes.POINTER(U64), ctypes.POINTER(I32), ctypes.POINTER(D)
    sig = {
        "autoscout_space_create": ([ctypes.c_char_p, I32, ctypes.POINTER(P)], I32),
        "autoscout_space_destroy": ([P], None),
        "autoscout_space_info": ([P, ctypes.POINTER(SpaceInfo)], I32),
        "autoscout_observe": ([P, pU64, pD, I64, P], I32),
        "autoscout_observe_clear": ([P], I32),
        "autoscout_observe_info": ([P, pI32, pD, pD], I32),
        "autoscout_score_batch": ([P, ctypes.POINTER(ScoreArgs), P], I32),
        "autoscout_topk": ([P, I32, pU64, pD, pI32, P], I32),
        "autoscout_topk_pool": ([P, I32, P, I32, pI32, P, P], I32),
        "autoscout_topk_merge": ([P, P, pI32, P, I32, I32, I32, pU64, pD, pI32, pI32], I32),
        "autoscout_topk_pool_device": ([P, I32, P, I32, P], I32),
        "autoscout_topk_merge_device": ([P, P, I32, I32, I32, P, P], I32),
        "autoscout_decode": ([P, U64, pI32, pI32], I32),
        "autoscout_activity": ([P, U64, ctypes.POINTER(ctypes.c_uint32)], I32),
        "autoscout_cvi_to_raw": ([P, U64, pU64], I32),
        "autoscout_sample_to_cvi": ([P, U64, U64, pU64], I32),
        "autoscout_raw_to_cvi": ([P, U64, pU64, pI32], I32),
        "autoscout_prior": ([P, U64, pD, pI32], I32),
        "autoscout_gp_lml": ([P, pD, I32, pD, P], I32),
        "autoscout_set_gp_hyper": ([P, pD, D, D], I32),
        "autoscout_ml2": ([P, I32, U64, I32, pD, pD, pI32, P], I32),
        "autoscout_ensemble_info": ([P, pD, pD, pI32], I32),
        "autoscout_subtree_range": ([P, pI32, I32, pU64, pU64], I32),
        "autoscout_neighbors": ([P, U64, pU64, I32, pI32], I32),
        "autoscout_simulate": ([P, U64, pD, pD, pI32], I32),
        "autoscout_mask_range": ([P, U64, U64, P, P, P], I32),
        "autoscout_set_path": ([P, I32], I32),
        "autoscout_set_timing": ([P, I32], I32),
        "autoscout_set_async_observe": ([P, I32], I32),
        "autoscout_set_slice": ([P, U64], I32),
        "autoscout_last_kernel_ms": ([P, pD, pD], I32),
        "autoscout_last_phase_ms": ([P, pD, pD], I32),
        "autoscout_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_LIB = _load()


def lib():
    return _LIB


def _check(st):
    if st != 0:
        raise AutoscoutError(st, _LIB.autoscout_last_error().decode())


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return ctypes.c_void_p(0)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Space:
    """Owning wrapper of an as_space* handle."""

    def __init__(self, space_json, device=0):
        if isinstance(space_json, dict):
            space_json = json.dumps(space_json)
        elif not str(space_json).lstrip().startswith("{"):
            with open(space_json) as fh:
                space_json = fh.read()
        self.doc = json.loads(space_json)
        h = ctypes.c_void_p()
        _check(_LIB.autoscout_space_create(space_json.encode(), int(device), ctypes.byref(h)))
        self.h = h
        self.device = device
        self.info = self.space_info()

    def n_launches(self):
        return self.space_info()["n_launches"]

    def close(self):
        if getattr(self, "h", None):
            _LIB.autoscout_space_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --------------------------------------------------------------- introspection
    def space_info(self):
        inf = SpaceInfo()
        _check(_LIB.autoscout_space_info(self.h, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in SpaceInfo._fields_}

    @property
    def n_cvi(self):
        return self.info["n_cvi"]

    @property
    def d(self):
        return self.info["n_features"]

    def decode(self, raw):
        dig = (ctypes.c_int32 * self.d)()
        valid = ctypes.c_int32()
        _check(_LIB.autoscout_decode(self.h, int(raw), dig, ctypes.byref(valid)))
        return list(dig), bool(valid.value)

    def activity(self, raw):
        """-> list[bool]: feature j active for this raw index."""
        m = ctypes.c_uint32()
        _check(_LIB.autoscout_activity(self.h, int(raw), ctypes.byref(m)))
        return [bool((m.value >> j) & 1) for j in range(self.d)]

    def cvi_to_raw(self, cvi):
        r = ctypes.c_uint64()
        _check(_LIB.autoscout_cvi_to_raw(self.h, int(cvi), ctypes.byref(r)))
        return r.value

    def gp_lml(self, hyp, stream=None):
        """Log marginal likelihoods of hyper-parameter settings hyp [n, d + 2] (NEXT-4)."""
        hyp = np.ascontiguousarray(hyp, dtype=np.float64)
        n = hyp.shape[0]
        out = np.zeros(max(n, 1))
        _check(_LIB.autoscout_gp_lml(self.h, hyp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n,
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream_ptr(stream)))
        return out[:n]

    def set_gp_hyper(self, lengthscale, sf2, sn2):
        ls = np.ascontiguousarray(lengthscale, dtype=np.float64)
        _check(_LIB.autoscout_set_gp_hyper(self.h, ls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                           float(sf2), float(sn2)))
        self.info = self.space_info()

    def ml2(self, n_set=1024, seed=0, apply=True, stream=None):
        """-> (best hyper-parameters [d + 2], best lml, best index) of a batched ML-II search."""
        best = np.zeros(self.d + 2)
        lml, idx = ctypes.c_double(), ctypes.c_int32()
        _check(_LIB.autoscout_ml2(self.h, int(n_set), int(seed), 1 if apply else 0,
                                  best.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(lml),
                                  ctypes.byref(idx), _stream_ptr(stream)))
        self.info = self.space_info()
        return best, lml.value, idx.value

    def prior(self, raw):
        """-> (m0, source): GP prior mean of a configuration (source 1 = regression ensemble)."""
        m, src = ctypes.c_double(), ctypes.c_int32()
        _check(_LIB.autoscout_prior(self.h, int(raw), ctypes.byref(m), ctypes.byref(src)))
        return m.value, int(src.value)

    def ensemble_info(self):
        """-> (r2[4], w[4], available) of the regression-simulator ensemble (NEXT-1)."""
        r2, w, av = (ctypes.c_double * 4)(), (ctypes.c_double * 4)(), ctypes.c_int32()
        _check(_LIB.autoscout_ensemble_info(self.h, r2, w, ctypes.byref(av)))
        return list(r2), list(w), bool(av.value)

    def raw_to_cvi(self, raw):
        """-> (position, member): position of raw in the CVI if member, else #members below it."""
        r, m = ctypes.c_uint64(), ctypes.c_int32()
        _check(_LIB.autoscout_raw_to_cvi(self.h, int(raw), ctypes.byref(r), ctypes.byref(m)))
        return r.value, bool(m.value)

    def subtree_range(self, digits):
        """CVI range (begin, count) of the completions of a partial assignment of the first
        len(digits) features (MCTS subtree, NEXT-2(i))."""
        d = (ctypes.c_int32 * max(len(digits), 1))(*[int(x) for x in digits])
        b, c = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_LIB.autoscout_subtree_range(self.h, d, len(digits), ctypes.byref(b), ctypes.byref(c)))
        return b.value, c.value

    def neighbors(self, raw, cap=4096):
        """CVI positions of the coordinate neighbours of raw (NEXT-2(ii)), as a uint64 numpy array."""
        out = np.zeros(max(cap, 1), dtype=np.uint64)
        n = ctypes.c_int32()
        _check(_LIB.autoscout_neighbors(self.h, int(raw), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                        int(cap), ctypes.byref(n)))
        return out[:n.value].copy()

    def sample_to_cvi(self, seed, ordinal):
        r = ctypes.c_uint64()
        _check(_LIB.autoscout_sample_to_cvi(self.h, int(seed), int(ordinal), ctypes.byref(r)))
        return r.value

    def simulate(self, raw):
        c, m, ok = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        _check(_LIB.autoscout_simulate(self.h, int(raw), ctypes.byref(c), ctypes.byref(m), ctypes.byref(ok)))
        return c.value, m.value, bool(ok.value)

    # --------------------------------------------------------------- observed set
    def observe(self, raws, costs, stream=None):
        raws = np.ascontiguousarray(raws, dtype=np.uint64)
        costs = np.ascontiguousarray(costs, dtype=np.float64)
        assert raws.shape == costs.shape
        _check(_LIB.autoscout_observe(self.h, raws.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                      costs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(raws),
                                      _stream_ptr(stream)))
        # (no space_info() refresh here: it would wait for an asynchronous fit; self.info only
        # caches the space's constants)

    def observe_clear(self):
        _check(_LIB.autoscout_observe_clear(self.h))

    def observe_info(self):
        m, b, f = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
        _check(_LIB.autoscout_observe_info(self.h, ctypes.byref(m), ctypes.byref(b), ctypes.byref(f)))
        return m.value, b.value, f.value

    # --------------------------------------------------------------- scoring
    def score_batch(self, mode="range", begin=0, count=None, seed=0, acq="ei", k=32, kappa=None, xi=None,
                    accumulate=False, d_scores=None, d_raw=None, d_valid_count=None, d_positions=None,
                    d_screen=None, stream=None):
        """mode "list": candidate j is CVI position d_positions[begin + j] (device uint64 tensor the
        caller keeps alive until topk); count defaults to len(d_positions) - begin."""
        gp = self.doc.get("gp", {})
        a = ScoreArgs(MODE[mode] if isinstance(mode, str) else int(mode),
                      ACQ[acq] if isinstance(acq, str) else int(acq), int(begin),
                      int((self.n_cvi if d_positions is None else d_positions.numel()) - begin
                          if count is None else count), int(seed),
                      float(gp.get("kappa", 2.0) if kappa is None else kappa),
                      float(gp.get("xi", 0.0) if xi is None else xi), int(k), 1 if accumulate else 0,
                      _ptr(d_scores), _ptr(d_raw), _ptr(d_valid_count), _ptr(d_positions), _ptr(d_screen))
        _check(_LIB.autoscout_score_batch(self.h, ctypes.byref(a), _stream_ptr(stream)))

    def topk(self, k, stream=None, allow_uncertified=False):
        raw = (ctypes.c_uint64 * k)()
        sc = (ctypes.c_double * k)()
        n = ctypes.c_int32()
        st = _LIB.autoscout_topk(self.h, int(k), raw, sc, ctypes.byref(n), _stream_ptr(stream))
        if st != 0 and not (allow_uncertified and st == 12):
            _check(st)
        return [(int(raw[i]), float(sc[i])) for i in range(n.value)]

    def topk_pool(self, k, cap, stream=None):
        """-> (pool [cap] ENTRY_DTYPE, n, cut ENTRY_DTYPE scalar array of 1)."""
        buf = np.zeros(cap, dtype=ENTRY_DTYPE)
        cut = np.zeros(1, dtype=ENTRY_DTYPE)
        n = ctypes.c_int32()
        _check(_LIB.autoscout_topk_pool(self.h, int(k), buf.ctypes.data_as(ctypes.c_void_p), int(cap),
                                        ctypes.byref(n), cut.ctypes.data_as(ctypes.c_void_p), _stream_ptr(stream)))
        return buf, n.value, cut

    def topk_pool_device(self, k, cap, out=None, stream=None):
        """Refined local pool packed on the device -> int64 tensor [(cap + 2) * 2] (16-byte entries:
        header {n, certified}, cut, cap entries; include/autoscout.h).  No host copy of the pool."""
        import torch
        if out is None:
            out = torch.empty((cap + 2) * 2, dtype=torch.int64, device=torch.device("cuda", self.device))
        _check(_LIB.autoscout_topk_pool_device(self.h, int(k), _ptr(out), int(cap), _stream_ptr(stream)))
        return out

    def topk_merge_device(self, d_pools, n_pools, cap, k, stream=None):
        """Merge gathered packed pools on the device; one D2H of the (k + 2)-entry result.
        -> (list[(raw, score)], certified)."""
        import torch
        out = torch.empty((k + 2) * 2, dtype=torch.int64, device=d_pools.device)
        _check(_LIB.autoscout_topk_merge_device(self.h, _ptr(d_pools), int(n_pools), int(cap), int(k), _ptr(out),
                                                _stream_ptr(stream)))
        ent = np.ascontiguousarray(out.cpu().numpy()).view(ENTRY_DTYPE)
        n, cert = int(ent[0]["score"]), bool(ent[0]["raw"])
        return [(int(ent[2 + i]["raw"]), float(ent[2 + i]["score"])) for i in range(n)], cert

    def mask_range(self, raw_begin, count, d_bits, d_valid_count=None, stream=None):
        _check(_LIB.autoscout_mask_range(self.h, int(raw_begin), int(count), _ptr(d_bits), _ptr(d_valid_count),
                                         _stream_ptr(stream)))

    def set_path(self, path):
        """0 auto, 1 SIMT, 2 tensor cores (SIMT r^2), 3 tensor cores (one-hot r^2 on the tensor cores);
        or 'auto' / 'simt' / 'tc' / 'tc2'."""
        path = {"auto": 0, "simt": 1, "tc": 2, "tc2": 3}.get(path, path)
        _check(_LIB.autoscout_set_path(self.h, int(path)))

    def set_slice(self, max_candidates):
        """Candidates per generate + score slice of the one-hot path (list memory 40 B each)."""
        _check(_LIB.autoscout_set_slice(self.h, int(max_candidates)))

    def set_async_observe(self, enable=True):
        """observe() returns before the GP fit; score_batch overlaps it with candidate generation."""
        _check(_LIB.autoscout_set_async_observe(self.h, 1 if enable else 0))

    def set_timing(self, enable=True):
        _check(_LIB.autoscout_set_timing(self.h, 1 if enable else 0))

    def last_kernel_ms(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(_LIB.autoscout_last_kernel_ms(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def last_phase_ms(self):
        """(generate kernels ms, tensor-core score kernels ms) of the last timed launch (one-hot path)."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(_LIB.autoscout_last_phase_ms(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


def topk_merge(pools, counts, cuts, k):
    """Merge gathered pools ([n_pools, cap] ENTRY_DTYPE, counts [n_pools], cuts [n_pools] ENTRY_DTYPE)
    -> (list[(raw, score)], certified)."""
    pools = np.ascontiguousarray(pools, dtype=ENTRY_DTYPE)
    n_pools, cap = pools.shape
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    cuts = np.ascontiguousarray(cuts, dtype=ENTRY_DTYPE).reshape(n_pools)
    raw = (ctypes.c_uint64 * k)()
    sc = (ctypes.c_double * k)()
    n = ctypes.c_int32()
    cert = ctypes.c_int32()
    st = _LIB.autoscout_topk_merge(None, pools.ctypes.data_as(ctypes.c_void_p),
                                   counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   cuts.ctypes.data_as(ctypes.c_void_p), int(n_pools), int(cap),
                                   int(k), raw, sc, ctypes.byref(n), ctypes.byref(cert))
    if st not in (0, 12):
        _check(st)
    return [(int(raw[i]), float(sc[i])) for i in range(n.value)], bool(cert.value)


def no_cut():
    c = np.zeros(1, dtype=ENTRY_DTYPE)
    c["score"] = -np.inf
    c["raw"] = np.iinfo(np.uint64).max
    return c


# C-ABI-named entry points (same names as include/autoscout.h)
def autoscout_space_create(space_json, device=0):
    return Space(space_json, device)


def autoscout_observe(space, raws, costs, stream=None):
    return space.observe(raws, costs, stream)


def autoscout_score_batch(space, **kw):
    return space.score_batch(**kw)


def autoscout_topk(space, k, stream=None):
    return space.topk(k, stream)


autoscout_topk_merge = topk_merge


def autoscout_raw_to_cvi(space, raw):
    return space.raw_to_cvi(raw)


def autoscout_subtree_range(space, digits):
    return space.subtree_range(digits)


def autoscout_neighbors(space, raw, cap=4096):
    return space.neighbors(raw, cap)


def autoscout_prior(space, raw):
    return space.prior(raw)


def autoscout_ensemble_info(space):
    return space.ensemble_info()


def autoscout_gp_lml(space, hyp, stream=None):
    return space.gp_lml(hyp, stream)


def autoscout_set_gp_hyper(space, lengthscale, sf2, sn2):
    return space.set_gp_hyper(lengthscale, sf2, sn2)


def autoscout_ml2(space, n_set=1024, seed=0, apply=True, stream=None):
    return space.ml2(n_set, seed, apply, stream)


def autoscout_set_slice(space, max_candidates):
    return space.set_slice(max_candidates)


def autoscout_set_async_observe(space, enable=True):
    return space.set_async_observe(enable)
