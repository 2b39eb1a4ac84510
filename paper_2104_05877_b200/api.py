"""Thin Python binding over libskel.so: argument marshalling only.

Every step of the path runs in the library's CUDA kernels; torch provides device
memory and the current stream.  Names follow include/skel.h (and the paper:
J_s, I_s, Z, eta).  Layout conventions:

  A   (m, n) float64 CUDA tensor, COLUMN-major (A.stride() == (1, lda));
      ``fortran(t)`` converts a row-major tensor.
  X   (l, n) float64, row-major (the sketch, X^T column-major).
  Lf  (n, k) float64, column-major.   Z (k, n) float64, column-major.
  Js, Is  (k,) int64 CUDA tensors (0-based, pivot order).
"""
import ctypes

import torch

from . import _lib

GAUSSIAN, SPARSE_SIGN, SRTT = 0, 1, 2
COL_ID, ROW_ID, CUR, ID_COEFFS, ROW_COEFFS, CUR_CSS = 0, 1, 2, 3, 4, 5
_EMB = {"gaussian": GAUSSIAN, "sparse_sign": SPARSE_SIGN, "srtt": SRTT, GAUSSIAN: GAUSSIAN, SPARSE_SIGN: SPARSE_SIGN,
        SRTT: SRTT}
_KIND = {"col_id": COL_ID, "row_id": ROW_ID, "cur": CUR, "id_coeffs": ID_COEFFS, "row_coeffs": ROW_COEFFS,
         "cur_css": CUR_CSS, COL_ID: COL_ID, ROW_ID: ROW_ID, CUR: CUR, ID_COEFFS: ID_COEFFS, ROW_COEFFS: ROW_COEFFS,
         CUR_CSS: CUR_CSS}


class SkelError(RuntimeError):
    def __init__(self, status, msg, info=0):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.info = info


_ctxs = {}


def lib():
    return _lib.load()


def context(device=None):
    """The (cached) sk_ctx for the device, re-targeted to torch's current stream."""
    L = lib()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    key = dev.index
    if key not in _ctxs:
        h = ctypes.c_void_p()
        st = L.sk_create(ctypes.byref(h), dev.index, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        if st != 0:
            raise SkelError(st, "sk_create failed (is this a B200 / sm_100 device?)")
        _ctxs[key] = h
    h = _ctxs[key]
    L.sk_set_stream(h, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return h


class DistSession:
    """A column-sharded library context (sk_create_dist) installed as this
    device's context while the session is open: the library owns the NCCL communicator and every
    call below (sketch, select_cols, gather_cols, id_coeffs, residual, rand_lupp) takes this rank's
    column block and performs the exchanges itself.  The torch.distributed group is used once, to
    share the NCCL unique id.  exchange: "replicate" (one all-gather of the k sketch rows LUPP
    reads) or "step" (one all-gather of candidate records per pivot step, CUDA graph)."""

    def __init__(self, n_global, group=None, device=None, exchange="replicate"):
        import torch.distributed as tdist

        from .dist import shard
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)
        self.n_global = n_global
        self.col0, self.ncols = shard(n_global, self.world, self.rank)
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            st = lib().sk_nccl_unique_id(uid)
            if st != 0:
                raise SkelError(st, "sk_nccl_unique_id failed (libnccl.so.2 not loadable?)")
        obj = [bytes(uid)]
        tdist.broadcast_object_list(obj, src=tdist.get_global_rank(group, 0) if group is not None else 0, group=group)
        ctypes.memmove(uid, obj[0], 128)
        h = ctypes.c_void_p()
        st = lib().sk_create_dist(ctypes.byref(h), self.dev.index,
                                  ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream), uid, self.rank,
                                  self.world, n_global, self.col0, self.ncols)
        if st != 0:
            raise SkelError(st, "sk_create_dist failed")
        self.h = h
        _check(lib().sk_set_dist_exchange(h, {"replicate": 0, "step": 1}[exchange]), h)
        self._prev = None

    def __enter__(self):
        self._prev = _ctxs.get(self.dev.index)
        _ctxs[self.dev.index] = self.h
        return self

    def __exit__(self, *exc):
        if self._prev is not None:
            _ctxs[self.dev.index] = self._prev
        else:
            _ctxs.pop(self.dev.index, None)
        self._prev = None

    def close(self):
        if self.h:
            lib().sk_destroy(self.h)
            self.h = None


def set_sketch_tuning(path=0, bm=0, splits=0, chunk_rows=0, warps=0, device=None):
    """sk_set_sketch_tuning: pin the dense sketch's plan on this device's context (0 = automatic)."""
    h = context(device)
    _check(lib().sk_set_sketch_tuning(h, int(path), int(bm), int(warps), int(splits), ctypes.c_int64(int(chunk_rows))), h)


def launch_count(device=None):
    return int(lib().sk_launch_count(context(device)))


def _check(st, h, info=0):
    if st != 0:
        msg = lib().sk_last_error(h).decode()
        raise SkelError(st, msg, info)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def fortran(t):
    """Column-major copy of a 2-D tensor (same values, stride (1, rows))."""
    return t.t().contiguous().t()


def _colmajor(A, name):
    if A.dim() != 2 or A.dtype != torch.float64 or not A.is_cuda:
        raise ValueError(f"{name} must be a 2-D float64 CUDA tensor")
    if A.stride(0) != 1 and A.shape[0] > 1 and A.shape[1] > 1:
        raise ValueError(f"{name} must be column-major (use api.fortran)")
    return max(A.stride(1) if A.shape[1] > 1 else A.shape[0], A.shape[0], 1)


def sketch(A, l, embedding="gaussian", seed=0, zeta=8, out=None):
    """X = Gamma A (Algorithm 2 lines 1-2)."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    X = out if out is not None else torch.empty((l, n), dtype=torch.float64, device=A.device)
    h = context(A.device.index)
    _check(lib().sk_sketch(h, _ptr(A), m, n, lda, l, _EMB[embedding], zeta, seed & (2**64 - 1), _ptr(X),
                           max(X.stride(0), n)), h)
    return X


def sketch_cols(A, l, embedding="gaussian", seed=0, zeta=8):
    """Y = A Omega^T (m x l, column-major), the column sketch of Algorithm 3."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    Y = torch.empty((l, m), dtype=torch.float64, device=A.device).t()
    h = context(A.device.index)
    _check(lib().sk_sketch_cols(h, _ptr(A), m, n, lda, l, _EMB[embedding], zeta, seed & (2**64 - 1), _ptr(Y), m), h)
    return Y


def sketch_dual(A, lx, ly, seed_x=0, seed_y=1, device=0):
    """Algorithm 3 line 2: X = Gamma A (lx x n, row-major) and Y = A Omega^T (m x ly,
    column-major) in one pass over A (Gaussian embeddings, independent seeds).  A may be a CPU
    tensor (column-major, ideally pinned): it then crosses PCIe once, in column blocks."""
    on_host = not A.is_cuda
    if A.dtype != torch.float64 or A.dim() != 2 or (A.stride(0) != 1 and A.shape[1] > 1):
        raise ValueError("A must be a column-major 2-D float64 tensor")
    m, n = A.shape
    lda = max(A.stride(1), m)
    dev = torch.device("cuda", device if on_host else A.device.index)
    X = torch.empty((lx, n), dtype=torch.float64, device=dev)
    Y = torch.empty((ly, m), dtype=torch.float64, device=dev).t()
    h = context(dev.index)
    _check(lib().sk_sketch_dual(h, _ptr(A), 1 if on_host else 0, m, n, lda, lx, ly, GAUSSIAN, seed_x & (2**64 - 1),
                                seed_y & (2**64 - 1), _ptr(X), n, _ptr(Y), m), h)
    return X, Y


def id_estimate_cols(X, Js, check=True):
    """C^+ A ~ X_1^+ X: Z (k x n, column-major) from the row sketch and its column pivots."""
    lx, n = X.shape
    k = Js.numel()
    Z = torch.empty((n, k), dtype=torch.float64, device=X.device).t()
    info = ctypes.c_int64(0)
    h = context(X.device.index)
    st = lib().sk_id_estimate_cols(h, _ptr(X), lx, n, max(X.stride(0), n), _ptr(Js), k, _ptr(Z), k,
                                   ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return Z


def id_estimate_rows(Y, Is, check=True):
    """A R^+ ~ Y Y_1^+ (P:436): W (m x k, column-major) from the column sketch and its row pivots."""
    ldy = _colmajor(Y, "Y")
    m, ly = Y.shape
    k = Is.numel()
    W = torch.empty((k, m), dtype=torch.float64, device=Y.device).t()
    info = ctypes.c_int64(0)
    h = context(Y.device.index)
    st = lib().sk_id_estimate_rows(h, _ptr(Y), m, ly, ldy, _ptr(Is), k, _ptr(W), m,
                                   ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return W


def stream_select(A, k, l=None, embedding="gaussian", seed_x=0, seed_y=1, zeta=8):
    """Algorithm 3 (streaming two-sided selection): X = Gamma A and Y = A Omega^T from
    independent embeddings, column LUPP on X -> J_s, row LUPP on Y -> I_s.  Returns (Js, Is)."""
    l = k + 10 if l is None else l
    X = sketch(A, l, embedding, seed_x, zeta)
    Y = sketch_cols(A, l, embedding, seed_y, zeta)
    Js, _, _, _ = select_cols(X, k, want_factors=False)
    Is, _, _, _ = select_rows(Y, k, want_factors=False)
    return Js, Is


def sketch_power(A, l, embedding="gaussian", seed=0, q=1, zeta=8, out=None, ortho=False):
    """X = Omega (A^T A)^q (eq:def_power_iter; Rand-LUPP-1piter for q = 1), or with
    ortho=True the orthogonalised iteration X = ortho(Y_q)^T A of eq:ortho_power_iter."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    X = out if out is not None else torch.empty((l, n), dtype=torch.float64, device=A.device)
    h = context(A.device.index)
    if ortho:
        info = ctypes.c_int64(0)
        st = lib().sk_sketch_power_ortho(h, _ptr(A), m, n, lda, l, _EMB[embedding], zeta, seed & (2**64 - 1), q,
                                         _ptr(X), max(X.stride(0), n), ctypes.byref(info))
        _check(st, h, info.value)
        return X
    _check(lib().sk_sketch_power(h, _ptr(A), m, n, lda, l, _EMB[embedding], zeta, seed & (2**64 - 1), q, _ptr(X),
                                 max(X.stride(0), n)), h)
    return X


def select_cols(X, k, want_factors=True, want_gaps=False, check=True):
    """Column LUPP on the sketch (eq:def_LUPP, Alg. 2 line 3). Returns (Js, Lf, U, gaps)."""
    l, n = X.shape
    if X.stride(1) != 1:
        raise ValueError("X must be row-major")
    dev = X.device
    Js = torch.empty(k, dtype=torch.int64, device=dev)
    Lf = torch.empty((k, n), dtype=torch.float64, device=dev).t() if want_factors else None
    U = torch.empty((k, k), dtype=torch.float64, device=dev).t() if want_factors else None
    gaps = torch.empty(k, dtype=torch.float64, device=dev) if want_gaps else None
    info = ctypes.c_int64(0)
    h = context(dev.index)
    st = lib().sk_select_cols(h, _ptr(X), l, n, max(X.stride(0), n, 1), k, _ptr(Js), _ptr(Lf), max(n, 1), _ptr(U), k,
                              _ptr(gaps), ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return Js, Lf, U, gaps


def select_cols_cpqr(X, k, want_r=False, check=True):
    """Column-pivoted QR on the sketch (eq:def_QRCP). Returns (Js, R)."""
    l, n = X.shape
    dev = X.device
    Js = torch.empty(k, dtype=torch.int64, device=dev)
    R = torch.empty((n, k), dtype=torch.float64, device=dev).t() if want_r else None
    info = ctypes.c_int64(0)
    h = context(dev.index)
    st = lib().sk_select_cols_cpqr(h, _ptr(X), l, n, max(X.stride(0), n), k, _ptr(Js), _ptr(R), k,
                                   ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return Js, R


def select_cols_deim(A, X, k, check=True):
    """RSVD-DEIM column skeletons (eq:rsvd_procedures + DEIM) from A and its sketch X."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    l = X.shape[0]
    Js = torch.empty(k, dtype=torch.int64, device=A.device)
    info = ctypes.c_int64(0)
    h = context(A.device.index)
    st = lib().sk_select_cols_deim(h, _ptr(A), m, n, lda, _ptr(X), l, max(X.stride(0), n), k, _ptr(Js),
                                   ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return Js


def gather_cols(A, Js):
    """C = A(:, J_s) (eq:Js), column-major m x k."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    k = Js.numel()
    C = torch.empty((k, m), dtype=torch.float64, device=A.device).t()
    h = context(A.device.index)
    _check(lib().sk_gather_cols(h, _ptr(A), m, n, lda, _ptr(Js), k, _ptr(C), m), h)
    return C


def gather_cols_shard(A_local, Js, col0, m=None):
    """C(:, t) = A_global(:, J_s[t]) for the skeletons in this rank's column block
    [col0, col0 + ncols), zero columns for the others (sum over ranks = C)."""
    lda = _colmajor(A_local, "A")
    m, ncols = A_local.shape
    k = Js.numel()
    C = torch.empty((k, m), dtype=torch.float64, device=A_local.device).t()
    h = context(A_local.device.index)
    _check(lib().sk_gather_cols_shard(h, _ptr(A_local), m, ncols, lda, col0, _ptr(Js), k, _ptr(C), m), h)
    return C


def residual_cols(A, C):
    """(||A - Q Q^T A||_F^2, ||A||_F^2) with Q = ortho(C), C given (column-sharded residual)."""
    lda = _colmajor(A, "A")
    ldc = _colmajor(C, "C")
    m, n = A.shape
    k = C.shape[1]
    sums = (ctypes.c_double * 2)()
    h = context(A.device.index)
    _check(lib().sk_residual_cols(h, _ptr(A), m, n, lda, _ptr(C), k, ldc, sums), h)
    return float(sums[0]), float(sums[1])


def select_rows(C, k=None, want_factors=True, want_gaps=False, check=True):
    """Row LUPP on C (Alg. 2 line 4). Returns (Is, Lf, U, gaps)."""
    ldc = _colmajor(C, "C")
    m, kk = C.shape
    k = kk if k is None else k
    dev = C.device
    Is = torch.empty(k, dtype=torch.int64, device=dev)
    Lf = torch.empty((k, m), dtype=torch.float64, device=dev).t() if want_factors else None
    U = torch.empty((k, k), dtype=torch.float64, device=dev).t() if want_factors else None
    gaps = torch.empty(k, dtype=torch.float64, device=dev) if want_gaps else None
    info = ctypes.c_int64(0)
    h = context(dev.index)
    st = lib().sk_select_rows(h, _ptr(C), m, k, ldc, _ptr(Is), _ptr(Lf), m, _ptr(U), k, _ptr(gaps),
                              ctypes.byref(info) if check else None)
    _check(st, h, info.value)
    return Is, Lf, U, gaps


def id_coeffs(Lf, Js, want_eta=False):
    """Z with Z(:, J_s) = I and T = L1^{-T} L2^T elsewhere (Thm 4.1). Returns (Z, eta)."""
    n, k = Lf.shape
    ldlf = _colmajor(Lf, "Lf")
    Z = torch.empty((n, k), dtype=torch.float64, device=Lf.device).t()
    eta = ctypes.c_double(0.0)
    h = context(Lf.device.index)
    _check(lib().sk_id_coeffs(h, _ptr(Lf), n, k, ldlf, _ptr(Js), _ptr(Z), k,
                              ctypes.byref(eta) if want_eta else None), h)
    return Z, (eta.value if want_eta else None)


def residual(A, Js=None, Is=None, kind="col_id", Z=None):
    """(||A - approx||_F, ||A||_F) for kind in col_id / row_id / cur / id_coeffs."""
    lda = _colmajor(A, "A")
    m, n = A.shape
    k = (Js if Js is not None else Is).numel()
    res = ctypes.c_double(0.0)
    nrm = ctypes.c_double(0.0)
    ldz = Z.stride(1) if Z is not None else k
    h = context(A.device.index)
    _check(lib().sk_residual(h, _ptr(A), m, n, lda, _ptr(Js), _ptr(Is), k, _KIND[kind], _ptr(Z), ldz,
                             ctypes.byref(res), ctypes.byref(nrm)), h)
    return res.value, nrm.value


def rand_lupp(A, k, l=None, embedding="gaussian", seed=0, zeta=8, rows=False, device=0):
    """Algorithm 2 end to end.  A may be a CPU tensor (copied inside the call)
    or a CUDA tensor; returns host int64 tensors (Js, Is or None)."""
    on_host = not A.is_cuda
    if A.dtype != torch.float64 or A.dim() != 2:
        raise ValueError("A must be a 2-D float64 tensor")
    if A.stride(0) != 1 and A.shape[1] > 1:
        raise ValueError("A must be column-major")
    m, n = A.shape
    lda = max(A.stride(1), m)
    l = k + 10 if l is None else l
    Js = torch.empty(k, dtype=torch.int64)
    Is = torch.empty(k, dtype=torch.int64) if rows else None
    info = ctypes.c_int64(0)
    h = context(device if on_host else A.device.index)
    st = lib().sk_rand_lupp(h, _ptr(A), 1 if on_host else 0, m, n, lda, l, _EMB[embedding], zeta,
                            seed & (2**64 - 1), k, _ptr(Js), _ptr(Is), ctypes.byref(info))
    _check(st, h, info.value)
    return Js, Is


class LuppDist:
    """Per-step-exchange column LUPP on this rank's sketch block (sk_lupp_dist_*).

    ``begin(X_local)`` copies rows 0..k-1 of the l x nloc row-major block and writes the step-0
    proposal into ``cand``; then, for t = 1..k, the caller all-gathers ``cand`` into ``gathered``
    (world x rec) and calls ``step(t)``.  Buffers are allocated once here, so the sequence can be
    captured in a CUDA graph.  Js (replicated), Lf (this rank's rows) and U are the results."""

    def __init__(self, nloc, k, col0, world, device=None, want_factors=True):
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.nloc, self.k, self.col0, self.world, self.device = nloc, k, col0, world, dev
        self.rec = k + 4
        nbytes = int(lib().sk_lupp_dist_state_bytes(nloc, k))
        self.state = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.cand = torch.empty(self.rec, dtype=torch.float64, device=dev)
        self.gathered = torch.empty(world * self.rec, dtype=torch.float64, device=dev)
        self.Js = torch.empty(k, dtype=torch.int64, device=dev)
        self.Lf = torch.empty((k, max(nloc, 1)), dtype=torch.float64, device=dev).t() if want_factors else None
        self.U = torch.empty((k, k), dtype=torch.float64, device=dev).t() if want_factors else None

    def begin(self, X_local):
        if X_local.dtype != torch.float64 or not X_local.is_cuda or X_local.dim() != 2:
            raise ValueError("X_local must be a 2-D float64 CUDA tensor")
        if X_local.shape[1] != self.nloc or X_local.shape[0] < self.k:
            raise ValueError("X_local must be l x nloc with l >= k")
        if self.nloc > 1 and X_local.stride(1) != 1:
            raise ValueError("X_local must be row-major")
        ldx = max(X_local.stride(0), self.nloc) if X_local.shape[0] > 1 else max(self.nloc, 1)
        h = context(self.device.index)
        _check(lib().sk_lupp_dist_begin(h, _ptr(X_local), self.nloc, ldx, self.k, self.col0, _ptr(self.state),
                                        _ptr(self.Lf), max(self.nloc, 1), _ptr(self.U), self.k, _ptr(self.cand)), h)

    def step(self, t):
        h = context(self.device.index)
        _check(lib().sk_lupp_dist_step(h, _ptr(self.state), self.nloc, self.k, self.col0, t, _ptr(self.gathered),
                                       self.world, _ptr(self.Js), _ptr(self.Lf), max(self.nloc, 1), _ptr(self.U),
                                       self.k, _ptr(self.cand)), h)

    def info(self):
        """Synchronises; raises SkelError(SK_E_RANK) with .info = the failing 1-based step."""
        info = ctypes.c_int64(0)
        h = context(self.device.index)
        _check(lib().sk_lupp_dist_info(h, _ptr(self.state), ctypes.byref(info)), h, info.value)
        return 0


class LuppDistP2P(LuppDist):
    """LuppDist with the exchange fused into the step kernel (sk_lupp_dist_*_p2p): `peers` is a
    CUDA int64 tensor of the world mailbox addresses as seen from this rank (peers[rank] = own,
    `own` its host value).  No collective between steps: begin(X), then step(t) for t = 1..k, then
    info().  begin() advances the mailbox's device-side epoch, so mailboxes are reusable and the
    whole selection can be captured in a CUDA graph."""

    def __init__(self, nloc, k, col0, world, rank, peers, own, device=None, want_factors=True):
        super().__init__(nloc, k, col0, world, device, want_factors)
        if peers.dtype != torch.int64 or not peers.is_cuda or peers.numel() != world:
            raise ValueError("peers must be a CUDA int64 tensor of `world` mailbox addresses")
        self.rank, self.peers, self.own = rank, peers, own

    def begin(self, X_local):
        if X_local.dtype != torch.float64 or not X_local.is_cuda or X_local.dim() != 2:
            raise ValueError("X_local must be a 2-D float64 CUDA tensor")
        if X_local.shape[1] != self.nloc or X_local.shape[0] < self.k:
            raise ValueError("X_local must be l x nloc with l >= k")
        ldx = max(X_local.stride(0), self.nloc) if X_local.shape[0] > 1 else max(self.nloc, 1)
        h = context(self.device.index)
        _check(lib().sk_lupp_dist_begin_p2p(h, _ptr(X_local), self.nloc, ldx, self.k, self.col0, _ptr(self.state),
                                            _ptr(self.Lf), max(self.nloc, 1), _ptr(self.U), self.k, _ptr(self.cand),
                                            _ptr(self.peers), ctypes.c_void_p(self.own), self.rank, self.world), h)

    def step(self, t):
        h = context(self.device.index)
        _check(lib().sk_lupp_dist_step_p2p(h, _ptr(self.state), self.nloc, self.k, self.col0, t, _ptr(self.peers),
                                           self.rank, self.world, _ptr(self.Js), _ptr(self.Lf),
                                           max(self.nloc, 1), _ptr(self.U), self.k, _ptr(self.cand)), h)


def mailbox_bytes(k, world):
    return int(lib().sk_lupp_dist_mailbox_bytes(k, world))


def ipc_alloc(nbytes, device=None):
    """Zero-filled cudaMalloc memory that other processes can map (returns the device address)."""
    h = context(device)
    p = ctypes.c_void_p()
    _check(lib().sk_ipc_alloc(h, nbytes, ctypes.byref(p)), h)
    return p.value


def ipc_free(ptr, device=None):
    h = context(device)
    _check(lib().sk_ipc_free(h, ctypes.c_void_p(ptr)), h)


def ipc_export(ptr, device=None):
    h = context(device)
    buf = ctypes.create_string_buffer(64)
    _check(lib().sk_ipc_export(h, ctypes.c_void_p(ptr), buf), h)
    return buf.raw


def ipc_import(handle, device=None):
    h = context(device)
    p = ctypes.c_void_p()
    _check(lib().sk_ipc_import(h, ctypes.c_char_p(bytes(handle)), ctypes.byref(p)), h)
    return p.value


def ipc_close(ptr, device=None):
    h = context(device)
    _check(lib().sk_ipc_close(h, ctypes.c_void_p(ptr)), h)
