"""B200-native NFFT hot path (arXiv:2208.00049, NFFT.jl) — Python binding.

A thin ctypes layer over the C ABI in include/nfft.h (libnfft_b200.so, built
in-tree by `__graft_entry__.build()` / `python -m paper_2208_00049_b200.build`).
It only marshals arguments: every step of the transform runs in the library's
CUDA kernels (and cuFFT for the oversampled FFT). PyTorch is used for device
memory and streams. There is no CPU fallback: if the shared library is
missing, importing `lib()` raises.

    plan = NfftPlan(nodes, N=(512, 512), m=4, sigma=2.0)
    plan.precompute()
    f = plan.forward(fhat)      # direct NFFT, Alg. 1
    y = plan.adjoint(f)         # adjoint NFFT, Alg. 2
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnfft_b200.so")

# Every symbol include/nfft.h declares (checked by tests/test_abi.py).
NFFT_SYMBOLS = (
    "nfft_default_options", "nfft_plan_create", "nfft_plan_create_ex", "nfft_set_nodes",
    "nfft_precompute", "nfft_forward", "nfft_adjoint", "nfft_plan_destroy", "nfft_status_string",
    "nfft_plan_info", "nfft_get_binning", "nfft_get_window_tables", "nfft_get_stage_times",
    "nfft_get_stage_times_ex",
    "nfft_get_launch_count", "nfft_run_stage", "nfft_execute", "nfft_get_cell_binning", "nfft_get_features",
    "nfft_autotune_tile",
)
PRECOMPUTE = {"auto": 0, "polynomial": 1, "tensor": 2, "full": 3}
STAGES = {"precompute": 0, "fwd_deconv": 1, "fwd_fft": 2, "fwd_interp": 3, "adj_spread": 4, "adj_fft": 5,
          "adj_crop": 6}

STATUS = {
    0: "NFFT_SUCCESS", 1: "NFFT_ERROR_INVALID_VALUE", 2: "NFFT_ERROR_BAD_GEOMETRY",
    3: "NFFT_ERROR_NONFINITE_NODE", 4: "NFFT_ERROR_BAD_TILE", 5: "NFFT_ERROR_NOT_PRECOMPUTED",
    6: "NFFT_ERROR_OUT_OF_MEMORY", 7: "NFFT_ERROR_CUDA", 8: "NFFT_ERROR_CUFFT", 9: "NFFT_ERROR_UNSUPPORTED",
}
METHODS = {"auto": 0, "tiled": 1, "direct": 2, "tiled_cas": 3, "tiled_loc": 4, "tiled_own": 5, "tiled_sorted": 6, "tiled_v1": 7}
PRECISIONS = {"c64": 0, "c128": 1}


class NfftError(RuntimeError):
    def __init__(self, status, what):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{what}: {self.name} ({_lib.nfft_status_string(status).decode()})")


class Options(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int64), ("tile", ctypes.c_int64 * 3), ("stream", ctypes.c_void_p),
        ("device", ctypes.c_int), ("method", ctypes.c_int), ("max_subproblem", ctypes.c_int64),
        ("node_begin", ctypes.c_int64), ("node_end", ctypes.c_int64), ("timing", ctypes.c_int),
        ("check_nodes", ctypes.c_int), ("precompute", ctypes.c_int), ("window_points", ctypes.c_int),
    ]


_lib = None


def lib():
    """Load libnfft_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2208_00049_b200.build` "
                          "(or __graft_entry__.build()). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
    P = ctypes.POINTER
    sigs = {
        "nfft_default_options": [P(Options)],
        "nfft_plan_create": [P(vp), c_int, P(i64), i64, vp, ctypes.c_double, c_int, c_int, c_int],
        "nfft_plan_create_ex": [P(vp), c_int, P(i64), i64, vp, ctypes.c_double, c_int, c_int, c_int, P(Options)],
        "nfft_set_nodes": [vp, vp],
        "nfft_precompute": [vp],
        "nfft_forward": [vp, vp, vp],
        "nfft_adjoint": [vp, vp, vp],
        "nfft_plan_destroy": [vp],
        "nfft_plan_info": [vp, P(i64), P(i64), P(i64), P(i64)],
        "nfft_get_binning": [vp, P(i32), P(i32)],
        "nfft_get_cell_binning": [vp, P(i32), P(i32)],
        "nfft_get_window_tables": [vp, P(ctypes.c_double), P(ctypes.c_double), P(c_int)],
        "nfft_get_stage_times": [vp, P(ctypes.c_float), P(ctypes.c_float), P(ctypes.c_float)],
        "nfft_get_stage_times_ex": [vp, c_int, P(ctypes.c_float)],
        "nfft_get_launch_count": [vp, P(i64)],
        "nfft_get_features": [vp, P(c_int)],
        "nfft_autotune_tile": [c_int, P(i64), i64, vp, ctypes.c_double, c_int, c_int, vp, P(i64), c_int, c_int,
                               P(i64), P(ctypes.c_float)],
        "nfft_run_stage": [vp, c_int, vp, vp],
        "nfft_execute": [vp, c_int, vp, vp, vp, vp],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = c_int
    L.nfft_status_string.argtypes = [c_int]
    L.nfft_status_string.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(status, what):
    if status != 0:
        raise NfftError(status, what)


def _ptr(x):
    """Device pointer of a torch tensor or host pointer of a numpy array."""
    if isinstance(x, np.ndarray):
        return ctypes.c_void_p(x.ctypes.data)
    return ctypes.c_void_p(x.data_ptr())


def _torch():
    import torch
    return torch


class NfftPlan:
    """NFFT plan over fixed nodes.

    nodes: (M, D) float64 (c128) or float32 (c64), torch (any device) or numpy.
    N: grid size per dimension (even). Outputs follow the inputs: torch CUDA in
    -> torch CUDA out; numpy in -> numpy out (host staging inside the library).
    node_range: (begin, end) shard of the plan's SORTED node order (cell order
    in cell mode) processed by forward/adjoint (multi-GPU sharding, DESIGN.md
    §Multi-GPU). precompute: "auto" | "polynomial" | "tensor" | "full" (window
    taps per call / stored taps / the stored sparse matrix B). window_points: "2m" |
    "2m+2" (NFFT3's continued-window variant).
    """

    def __init__(self, nodes, N, m=4, sigma=2.0, precision="c128", batch=1, tile=None, stream=None,
                 device=None, method="auto", max_subproblem=0, node_range=None, timing=False,
                 check_nodes=True, precompute="auto", window_points="2m"):
        L = lib()
        self.N = tuple(int(n) for n in N)
        self.D = len(self.N)
        self.m = int(m)
        self.sigma = float(sigma)
        self.precision = precision
        self.batch = int(batch)
        self.rdtype = np.float64 if precision == "c128" else np.float32
        self.cdtype = np.complex128 if precision == "c128" else np.complex64
        torch = _torch()
        self.tdtype_c = torch.complex128 if precision == "c128" else torch.complex64
        self.tdtype_r = torch.float64 if precision == "c128" else torch.float32
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        if stream is None and torch.cuda.is_available():
            stream = torch.cuda.current_stream(self.device).cuda_stream
        self.stream = stream
        # the plan stream as a torch stream (for ordering against the caller's current stream)
        self._pstream = None
        if torch.cuda.is_available():
            self._pstream = (torch.cuda.default_stream(self.device) if not stream
                             else torch.cuda.ExternalStream(stream, device=self.device))
        nodes = self._nodes_arg(nodes)
        self.M = int(nodes.shape[0])
        opt = Options()
        L.nfft_default_options(ctypes.byref(opt))
        opt.batch = self.batch
        for d, q in enumerate(tile or ()):
            opt.tile[d] = int(q)
        opt.stream = stream
        opt.device = self.device
        opt.method = METHODS[method]
        opt.max_subproblem = int(max_subproblem)
        if node_range is not None:
            opt.node_begin, opt.node_end = int(node_range[0]), int(node_range[1])
        opt.timing = int(bool(timing))
        opt.check_nodes = int(bool(check_nodes))
        opt.precompute = PRECOMPUTE[precompute]
        opt.window_points = {"2m": 0, "2m+2": 1}[window_points]
        self.opts = opt
        Narr = (ctypes.c_int64 * self.D)(*self.N)
        h = ctypes.c_void_p()
        _check(L.nfft_plan_create_ex(ctypes.byref(h), self.D, Narr, self.M, _ptr(nodes), self.sigma, self.m, 0,
                                     PRECISIONS[precision], ctypes.byref(opt)), "nfft_plan_create")
        self._h = h
        self._keep = nodes  # keep the source alive until the async copy is done
        self.precomputed = False

    # -- argument marshalling ------------------------------------------------
    def _nodes_arg(self, nodes):
        torch = _torch()
        if isinstance(nodes, np.ndarray):
            return np.ascontiguousarray(nodes.reshape(nodes.shape[0], -1), dtype=self.rdtype)
        t = nodes.reshape(nodes.shape[0], -1)
        if t.dtype != self.tdtype_r or not t.is_contiguous():
            t = t.to(self.tdtype_r).contiguous()
        return t

    def _grid_shape(self):
        return (self.batch,) + self.N

    def _data_arg(self, x, shape):
        torch = _torch()
        if isinstance(x, np.ndarray):
            x = np.ascontiguousarray(x, dtype=self.cdtype)
            if x.size != int(np.prod(shape)):
                raise ValueError(f"expected {shape} elements, got {x.shape}")
            return x
        if x.dtype != self.tdtype_c or not x.is_contiguous():
            x = x.to(self.tdtype_c).contiguous()
        if x.numel() != int(np.prod(shape)):
            raise ValueError(f"expected {shape} elements, got {tuple(x.shape)}")
        return x

    def _empty_like_kind(self, ref, shape):
        if isinstance(ref, np.ndarray):
            return np.empty(shape, dtype=self.cdtype)
        torch = _torch()
        return torch.empty(shape, dtype=self.tdtype_c, device=ref.device)

    def _enter(self, *tensors):
        """The library enqueues on the plan stream; when the caller's current
        stream is another one, the plan stream first waits for it (inputs written
        there are complete). Returns the caller's stream (or None)."""
        if self._pstream is None or not any(getattr(t, "is_cuda", False) for t in tensors):
            return None
        torch = _torch()
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream == self._pstream.cuda_stream:
            return None
        self._pstream.wait_stream(cur)
        return cur

    def _exit(self, cur, *tensors):
        """...and afterwards the caller's stream waits for the plan stream, and the
        tensors the call used are marked as in use on it (the caching allocator
        then does not hand temporaries to another allocation too early)."""
        if cur is None:
            return
        cur.wait_stream(self._pstream)
        for t in tensors:
            if getattr(t, "is_cuda", False):
                t.record_stream(self._pstream)

    # -- ABI calls -----------------------------------------------------------
    def set_nodes(self, nodes):
        nodes = self._nodes_arg(nodes)
        _check(lib().nfft_set_nodes(self._h, _ptr(nodes)), "nfft_set_nodes")
        self._keep = nodes
        self.precomputed = False

    def precompute(self):
        _check(lib().nfft_precompute(self._h), "nfft_precompute")
        self.precomputed = True
        return self

    def forward(self, fhat, out=None):
        """Direct NFFT: fhat (B, *N) or (*N) -> f (B, M)."""
        fhat = self._data_arg(fhat, self._grid_shape())
        if out is None:
            out = self._empty_like_kind(fhat, (self.batch, self.M))
        cur = self._enter(fhat, out)
        _check(lib().nfft_forward(self._h, _ptr(fhat), _ptr(out)), "nfft_forward")
        self._exit(cur, fhat, out)
        return out

    def adjoint(self, f, out=None):
        """Adjoint NFFT: f (B, M) or (M,) -> y (B, *N)."""
        f = self._data_arg(f, (self.batch, self.M))
        if out is None:
            out = self._empty_like_kind(f, self._grid_shape())
        cur = self._enter(f, out)
        _check(lib().nfft_adjoint(self._h, _ptr(f), _ptr(out)), "nfft_adjoint")
        self._exit(cur, f, out)
        return out

    def run_stage(self, stage, inp=None, out=None):
        """One stage of Alg. 1/2 on device tensors (nfft_run_stage)."""
        cur = self._enter(inp, out)
        _check(lib().nfft_run_stage(self._h, STAGES[stage], None if inp is None else _ptr(inp),
                                    None if out is None else _ptr(out)), f"nfft_run_stage({stage})")
        self._exit(cur, inp, out)
        if stage == "precompute":
            self.precomputed = True
        return out

    def execute(self, precompute=True, fhat=None, f_out=None, f_in=None, y_out=None):
        """nfft_execute: precompute and/or direct (fhat -> f_out) and/or adjoint
        (f_in -> y_out) NFFT with the independent parts run concurrently.
        Device tensors only; outputs are allocated when not given."""
        torch = _torch()
        flags = 1 if precompute else 0
        if fhat is not None:
            flags |= 2
            fhat = self._data_arg(fhat, self._grid_shape())
            if f_out is None:
                f_out = torch.empty((self.batch, self.M), dtype=self.tdtype_c, device=fhat.device)
        if f_in is not None:
            flags |= 4
            f_in = self._data_arg(f_in, (self.batch, self.M))
            if y_out is None:
                y_out = torch.empty(self._grid_shape(), dtype=self.tdtype_c, device=f_in.device)
        cur = self._enter(fhat, f_out, f_in, y_out)
        _check(lib().nfft_execute(self._h, flags, None if fhat is None else _ptr(fhat),
                                  None if f_out is None else _ptr(f_out), None if f_in is None else _ptr(f_in),
                                  None if y_out is None else _ptr(y_out)), "nfft_execute")
        self._exit(cur, fhat, f_out, f_in, y_out)
        if precompute:
            self.precomputed = True
        return f_out, y_out

    def info(self):
        nt = (ctypes.c_int64 * 3)()
        q = (ctypes.c_int64 * 3)()
        p = (ctypes.c_int64 * 3)()
        n = ctypes.c_int64()
        _check(lib().nfft_plan_info(self._h, nt, q, p, ctypes.byref(n)), "nfft_plan_info")
        return dict(Ntilde=tuple(nt[: self.D]), tile=tuple(q[: self.D]), tiles_per_dim=tuple(p[: self.D]),
                    n_tiles=n.value)

    def binning(self):
        n_tiles = self.info()["n_tiles"]
        perm = np.empty(self.M, np.int32)
        offs = np.empty(n_tiles + 1, np.int32)
        _check(lib().nfft_get_binning(self._h, perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "nfft_get_binning")
        return perm, offs

    def cell_binning(self):
        """(order, cstart) of the cell-mode sort (tile = 1 cell), or None when the
        plan sorts by tiles (include/nfft.h: nfft_get_cell_binning)."""
        ncells = int(np.prod(self.info()["Ntilde"]))
        order = np.empty(self.M, np.int32)
        cstart = np.empty(ncells + 1, np.int32)
        st = lib().nfft_get_cell_binning(self._h, order.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                         cstart.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        if st == 9:  # NFFT_ERROR_UNSUPPORTED: tile mode
            return None
        _check(st, "nfft_get_cell_binning")
        return order, cstart

    def sorted_order(self):
        """Node index of every position of the order node shards refer to."""
        cb = self.cell_binning()
        return cb[0] if cb is not None else self.binning()[0]

    def window_tables(self):
        deg = ctypes.c_int()
        _check(lib().nfft_get_window_tables(self._h, None, None, ctypes.byref(deg)), "nfft_get_window_tables")
        beta = np.empty(sum(self.N), np.float64)
        poly = np.empty((self.D, 2 * self.m, deg.value + 1), np.float64)
        _check(lib().nfft_get_window_tables(self._h, beta.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            poly.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            ctypes.byref(deg)), "nfft_get_window_tables")
        return beta, poly, deg.value

    def stage_times(self, which):
        ms = (ctypes.c_float * 5)()
        _check(lib().nfft_get_stage_times_ex(self._h, 0 if which == "forward" else 1, ms), "nfft_get_stage_times_ex")
        return dict(deconv=ms[0], fft=ms[1], resample=ms[2], zero=ms[3], precompute=ms[4])

    def features(self):
        """Paths in use: {"cell_mode", "tensor", "batch", "wblock", "full"} (include/nfft.h: nfft_get_features)."""
        v = ctypes.c_int()
        _check(lib().nfft_get_features(self._h, ctypes.byref(v)), "nfft_get_features")
        return {k for k, bit in (("cell_mode", 1), ("tensor", 4), ("batch", 8), ("wblock", 16), ("full", 32))
                if v.value & bit}

    def launches(self):
        n = ctypes.c_int64()
        _check(lib().nfft_get_launch_count(self._h, ctypes.byref(n)), "nfft_get_launch_count")
        return n.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(lib().nfft_plan_destroy(self._h), "nfft_plan_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nfft(nodes, fhat, N, m=4, sigma=2.0, precision="c128"):
    """One-shot direct NFFT."""
    p = NfftPlan(nodes, N, m=m, sigma=sigma, precision=precision).precompute()
    out = p.forward(fhat)
    p.close()
    return out


def nfft_adjoint(nodes, N, f, m=4, sigma=2.0, precision="c128"):
    """One-shot adjoint NFFT."""
    p = NfftPlan(nodes, N, m=m, sigma=sigma, precision=precision).precompute()
    out = p.adjoint(f)
    p.close()
    return out


def autotune_tile(nodes, N, m=4, sigma=2.0, precision="c128", batch=1, candidates=None, reps=5, method="auto"):
    """Online block-size benchmark (include/nfft.h: nfft_autotune_tile; the
    FFTW_MEASURE-like mode of PAPER.md:793). candidates: list of D-tuples or
    None (built-in list). Returns (best_tile, ms per direct + adjoint pair)."""
    N = tuple(int(n) for n in N)
    D = len(N)
    rd = np.float64 if precision == "c128" else np.float32
    if isinstance(nodes, np.ndarray):
        nodes = np.ascontiguousarray(nodes.reshape(nodes.shape[0], -1), dtype=rd)
    else:
        torch = _torch()
        nodes = nodes.reshape(nodes.shape[0], -1).to(torch.float64 if precision == "c128" else torch.float32)
        nodes = nodes.contiguous()
    opt = Options()
    lib().nfft_default_options(ctypes.byref(opt))
    opt.batch = int(batch)
    opt.method = METHODS[method]
    cand = None
    nc = 0
    if candidates:
        flat = [int(q) for t in candidates for q in t]
        cand = (ctypes.c_int64 * len(flat))(*flat)
        nc = len(candidates)
    best = (ctypes.c_int64 * D)()
    ms = ctypes.c_float()
    _check(lib().nfft_autotune_tile(D, (ctypes.c_int64 * D)(*N), int(nodes.shape[0]), _ptr(nodes), float(sigma), int(m),
                                    PRECISIONS[precision], ctypes.byref(opt), cand, nc, int(reps), best,
                                    ctypes.byref(ms)), "nfft_autotune_tile")
    return tuple(int(q) for q in best), float(ms.value)
