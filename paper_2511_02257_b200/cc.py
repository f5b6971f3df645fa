"""Thin ctypes binding of include/cc.h (libcc.so): argument marshalling only.

Every computation (scheduling, planning, contractions, copies) runs inside libcc.so;
this module only converts Python/numpy/torch arguments into the C ABI's plain pointers
and sizes and raises CCError on a non-zero status.  There is no fallback: if the shared
library is missing the import fails.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CC_LIB") or os.path.join(_HERE, "libcc.so")   # CC_LIB: experiment builds
if not os.path.exists(LIB_PATH):
    raise ImportError("libcc.so not built (run python -c 'import __graft_entry__ as g; g.build()'): %s" % LIB_PATH)
_lib = ctypes.CDLL(LIB_PATH)

c_i32, c_i64, c_u64, c_dbl, c_void_p, c_size_t = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                                  ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t)
P = ctypes.POINTER

CC_LEAF_M, CC_LEAF_B, CC_MM1, CC_BM1, CC_BB2, CC_TR_MM, CC_LEAF_X, CC_OP_X, CC_BB1, CC_BT2, CC_BB3 = range(11)
CC_N_OPS = 11
CC_SIBLING, CC_TREE, CC_GIVEN, CC_RSGS = range(4)
PART_TIME, PART_TREES = 0, 1
EXEC_GRAPH, EXEC_TIME_KERNELS, EXEC_ONLY_GEMM, EXEC_ONLY_TRACE, EXEC_OP_BY_OP, EXEC_PROFILE = 1, 2, 4, 8, 16, 32
EXEC_OZAKI_MM1 = 64        # MM1 / BM1 / BB2 on the tcgen05 Ozaki engine (name kept from MM1-only)
EXEC_OZAKI = 64
EXEC_AUTO = 128             # Ozaki engine or dataflow worker by the measured rule
CC_EVICT_NEXT_USE = 1       # cc_sched_cfg.flags: next-use (Belady) eviction, reading E-9
STATUS = {0: "OK", -1: "INVAL", -2: "PARSE", -3: "CYCLE", -4: "INCONSISTENT", -5: "MULTIROOT",
          -6: "UNKNOWN_NODE", -7: "NOT_CLOSED", -8: "INFEASIBLE", -9: "STATE", -10: "BUFFER_TOO_SMALL",
          -11: "CUDA", -12: "NOMEM"}
OP_KINDS = ["H2D", "D2H", "DROP", "CONTRACT", "FREE", "P2P_OUT", "P2P_IN"]


class cc_dims(ctypes.Structure):
    _fields_ = [("Lt", c_i32), ("N", c_i32), ("S", c_i32)]


class cc_node(ctypes.Structure):
    _fields_ = [("id", c_i64), ("op", c_i32), ("pad_", c_i32), ("a", c_i64), ("b", c_i64), ("size", c_i64)]


class cc_tree(ctypes.Structure):
    _fields_ = [("tree_id", c_i64), ("root", c_i64)]


class cc_term(ctypes.Structure):
    _fields_ = [("corr_id", c_i64), ("tree_id", c_i64), ("re", c_dbl), ("im", c_dbl)]


class cc_sched_cfg(ctypes.Structure):
    _fields_ = [("algo", c_i32), ("flags", c_i32), ("seed", c_u64), ("cap_bytes", c_i64),
                ("given_order", P(c_i64)), ("n_given", c_i64),
                ("peer_cap_bytes", c_i64), ("peer_leaves", P(c_i64)), ("n_peer_leaves", c_i64)]


class cc_plan_stats(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("n_contr", "peak", "transient_peak", "evictions", "h2d_count", "d2h_count",
                                     "h2d_bytes", "d2h_bytes", "host_peak_bytes", "model_peak",
                                     "model_transient_peak")] + \
               [("sched_seconds", c_dbl), ("plan_seconds", c_dbl), ("arena_high_water", c_i64)] + \
               [(n, c_i64) for n in ("p2p_out_count", "p2p_out_bytes", "p2p_in_count", "p2p_in_bytes",
                                     "peer_peak_bytes")]


class cc_exec_stats(ctypes.Structure):
    _fields_ = [("seconds", c_dbl), ("kernel_seconds", c_dbl), ("flops", c_dbl), ("hbm_bytes", c_dbl),
                ("h2d_bytes", c_i64), ("d2h_bytes", c_i64), ("n_kernels", c_i64), ("copy_seconds", c_dbl),
                ("p2p_in_bytes", c_i64), ("p2p_out_bytes", c_i64), ("move_bytes", c_i64), ("pad_", c_i64)]


class cc_plan_op(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("pad_", c_i32), ("node", c_i64), ("bytes", c_i64), ("offset", c_i64)]


class cc_options(ctypes.Structure):
    _fields_ = [(n, c_i32) for n in ("trace_fusion", "copy_reorder", "early_copies", "precopy", "ozaki_leaf_cache",
                                     "ozaki_slices")] + \
               [("h2d_chunk_bytes", c_i64), ("tr_ratio", c_dbl), ("debug", c_i32), ("slice_major", c_i32),
                ("leaf_slots", c_i32), ("trace_groups", c_i32)]


class cc_part_stats(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("n_trees", "n_contr", "work", "replicated_work", "leaf_bytes",
                                     "replicated_leaf_bytes")]


class cc_phys_stats(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("pool_high_water", "n_moves", "move_bytes", "host_pool_bytes")]


class cc_phys_op(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("pad_", c_i32), ("node", c_i64), ("bytes", c_i64), ("offset", c_i64),
                ("dst", c_i64), ("off_a", c_i64), ("off_b", c_i64)]


class cc_dag_stats(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in ("V", "E", "k", "n_contr", "n_leaves", "max_rank", "n_corr")] + \
               [("F_v", c_dbl), ("F_e", c_dbl)]


def _sig(name, *args, res=c_i32):
    f = getattr(_lib, name)
    f.argtypes = list(args)
    f.restype = res
    return f


_sig("cc_create", P(c_void_p), ctypes.c_int, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p)
_sig("cc_destroy", c_void_p, res=None)
_sig("cc_last_error", c_void_p, res=ctypes.c_char_p)
_sig("cc_version", res=ctypes.c_char_p)
_sig("cc_load_dag", c_void_p, P(cc_dims), P(cc_node), c_i64, P(cc_tree), c_i64, P(cc_term), c_i64)
_sig("cc_load_dag_file", c_void_p, ctypes.c_char_p)
_sig("cc_dag_info", c_void_p, P(cc_dag_stats))
_sig("cc_part_time_range", c_void_p, P(c_i32), P(c_i32))
_sig("cc_correlators", c_void_p, P(c_dbl), c_i64)
_sig("cc_partition", c_void_p, c_i32, c_i32, c_i32)
_sig("cc_part_trees", c_void_p, P(c_i64), c_i64, P(c_i64))
_sig("cc_partition_grid", c_void_p, c_i32, c_i32, c_i32)
_sig("cc_part_info", c_void_p, P(cc_part_stats))
_sig("cc_leaf_owners", c_void_p, P(c_i64), P(c_i32), c_i64, P(c_i64))
_sig("cc_schedule", c_void_p, P(cc_sched_cfg), P(c_i64), c_i64, P(c_i64), P(cc_plan_stats))
_sig("cc_memory_trace", c_void_p, P(c_i64), P(c_i64), c_i64, P(c_i64))
_sig("cc_plan_ops", c_void_p, P(cc_plan_op), c_i64, P(c_i64))
_sig("cc_phys_plan", c_void_p, c_i64, c_i32, P(cc_phys_stats))
_sig("cc_phys_ops", c_void_p, P(cc_phys_op), c_i64, P(c_i64))
_sig("cc_scratch_of", c_void_p, P(c_i64))
_sig("cc_tree_order", c_void_p, P(c_i64), c_i64, P(c_i64))
_sig("cc_plan_dump", c_void_p, ctypes.c_char_p)
_sig("cc_set_leaf", c_void_p, c_i64, c_void_p, c_size_t)
_sig("cc_set_leaf_device", c_void_p, c_i64, c_void_p, c_size_t)
_sig("cc_set_leaf_peer", c_void_p, c_i64, c_void_p, c_size_t)
_sig("cc_set_peer_tier", c_void_p, c_void_p, c_size_t)
_sig("cc_ipc_export", c_void_p, P(ctypes.c_uint8), P(c_u64))
_sig("cc_ipc_open", P(ctypes.c_uint8), c_u64, P(c_void_p))
_sig("cc_ipc_close", c_void_p)
_sig("cc_execute", c_void_p, c_i32, P(cc_exec_stats))
_sig("cc_execute_async", c_void_p, c_i32)
_sig("cc_kernel_times", c_void_p, P(c_dbl), P(c_i64))
_sig("cc_get_options", c_void_p, P(cc_options))
_sig("cc_set_options", c_void_p, P(cc_options))
_sig("cc_dataflow_state", c_void_p, P(c_i64), c_i64, P(c_i64))
_sig("cc_dataflow_profile", c_void_p, P(c_u64), c_i64, P(c_i64), P(c_i64))
_sig("cc_correlator", c_void_p, c_i64, P(c_dbl), c_i32)
_sig("cc_root_value", c_void_p, c_i64, P(c_dbl), c_i32)
_sig("cc_correlator_device_ptr", c_void_p, P(c_void_p), P(c_i64), P(c_i64))
_sig("cc_mm1", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32)
_sig("cc_bm1", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_bb2", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_tr_mm", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32)
_sig("cc_bb1", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_bt2", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_bb3", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_mm1_ozaki", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, c_void_p, ctypes.c_size_t)
_sig("cc_mm1_ozaki_workspace_bytes", c_i32, c_i32, c_i32, res=ctypes.c_size_t)
_sig("cc_i8gemm_tn", c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32)
_sig("cc_gemm_ozaki", c_void_p, c_i32, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, c_i32, c_void_p, ctypes.c_size_t)
_sig("cc_gemm_ozaki_workspace_bytes", c_i32, c_i32, c_i32, c_i32, c_i32, res=ctypes.c_size_t)
_sig("cc_fill_synthetic", c_void_p, c_void_p, c_i64, c_u64, c_i64, c_i64, c_i32, c_dbl)
_sig("cc_scratch_bytes", c_i32, c_i32, c_i32, res=c_size_t)

EXPORTED = ["cc_create", "cc_destroy", "cc_last_error", "cc_version", "cc_load_dag", "cc_load_dag_file",
            "cc_dag_info", "cc_part_time_range", "cc_correlators", "cc_partition", "cc_part_trees", "cc_partition_grid", "cc_part_info", "cc_leaf_owners", "cc_schedule", "cc_memory_trace", "cc_plan_ops", "cc_phys_plan", "cc_phys_ops", "cc_scratch_of",
            "cc_tree_order", "cc_plan_dump", "cc_set_leaf", "cc_set_leaf_device", "cc_set_leaf_peer", "cc_set_peer_tier", "cc_ipc_export", "cc_ipc_open", "cc_ipc_close", "cc_execute",
            "cc_execute_async", "cc_get_options", "cc_set_options", "cc_kernel_times", "cc_dataflow_state", "cc_dataflow_profile", "cc_correlator", "cc_root_value", "cc_correlator_device_ptr",
            "cc_mm1", "cc_bm1", "cc_bb2", "cc_tr_mm", "cc_bb1", "cc_bt2", "cc_bb3", "cc_mm1_ozaki", "cc_mm1_ozaki_workspace_bytes", "cc_i8gemm_tn", "cc_gemm_ozaki",
            "cc_gemm_ozaki_workspace_bytes", "cc_fill_synthetic", "cc_scratch_bytes"]


class CCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s (%d): %s" % (STATUS.get(status, "?"), status, msg))
        self.status = status
        self.code = STATUS.get(status, "?")


def _ptr(x):
    """Device/host address of a torch tensor, numpy array or int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError("cannot take the address of %r" % type(x))


def _ck_free(st):
    if st != 0:
        raise CCError(st, _lib.cc_last_error(None).decode())


def ipc_export(dev):
    """(64-byte handle, offset) of a device buffer (torch tensor or address) for another rank."""
    h = (ctypes.c_uint8 * 64)()
    off = c_u64()
    _ck_free(_lib.cc_ipc_export(_ptr(dev), h, ctypes.byref(off)))
    return bytes(h), int(off.value)


def ipc_open(handle, offset):
    """Device address of another process's buffer (cc_ipc_open); close with ipc_close."""
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = c_void_p()
    _ck_free(_lib.cc_ipc_open(h, offset, ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr):
    _ck_free(_lib.cc_ipc_close(ptr))


def cc_version():
    return _lib.cc_version().decode()


def cc_scratch_bytes(Lt, N, S):
    return int(_lib.cc_scratch_bytes(Lt, N, S))


def cc_mm1_ozaki_workspace_bytes(Lt, N, n_slices):
    return int(_lib.cc_mm1_ozaki_workspace_bytes(Lt, N, n_slices))


def cc_gemm_ozaki_workspace_bytes(op, Lt, N, S, n_slices):
    return int(_lib.cc_gemm_ozaki_workspace_bytes(op, Lt, N, S, n_slices))


class Context:
    """One cc_ctx.  Method names are the C functions without the cc_ prefix."""

    def __init__(self, device=-1, arena=None, arena_bytes=None, streams=None):
        h = c_void_p()
        cs = hs = ds = None
        if streams is not None:
            cs, hs, ds = (s.cuda_stream if hasattr(s, "cuda_stream") else s for s in streams)
        nbytes = arena_bytes if arena_bytes is not None else (
            arena.numel() * arena.element_size() if arena is not None else 0)
        st = _lib.cc_create(ctypes.byref(h), device, _ptr(arena), nbytes, cs, hs, ds)
        self._h = h
        self._keep = [arena, streams]
        if st != 0:
            msg = _lib.cc_last_error(h).decode() if h.value else "cc_create failed"
            if h.value:
                _lib.cc_destroy(h)
                self._h = c_void_p()
            raise CCError(st, msg)

    def close(self):
        if self._h and self._h.value:
            _lib.cc_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st):
        if st != 0:
            raise CCError(st, _lib.cc_last_error(self._h).decode())

    # --- DAG -----------------------------------------------------------------------------
    def load_dag(self, Lt, N, S, nodes, trees, terms):
        """nodes: [(id, op, a, b, size)], trees: [(tree_id, root)], terms: [(corr, tree, re, im)]."""
        nn = (cc_node * max(len(nodes), 1))()
        for i, (nid, op, a, b, size) in enumerate(nodes):
            nn[i] = cc_node(nid, op, 0, a, b, size)
        tt = (cc_tree * max(len(trees), 1))()
        for i, (t, r) in enumerate(trees):
            tt[i] = cc_tree(t, r)
        mm = (cc_term * max(len(terms), 1))()
        for i, (c, t, re, im) in enumerate(terms):
            mm[i] = cc_term(c, t, re, im)
        d = cc_dims(Lt, N, S)
        self._ck(_lib.cc_load_dag(self._h, ctypes.byref(d), nn, len(nodes), tt, len(trees), mm, len(terms)))

    def load_workload(self, w):
        self.load_dag(w.Lt, w.N, w.S, w.nodes, w.trees, w.terms)

    def load_dag_file(self, path):
        self._ck(_lib.cc_load_dag_file(self._h, path.encode()))

    def dag_info(self):
        s = cc_dag_stats()
        self._ck(_lib.cc_dag_info(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in cc_dag_stats._fields_}

    def partition(self, n_parts, part, mode):
        self._ck(_lib.cc_partition(self._h, n_parts, part, mode))

    def partition_grid(self, n_tree_parts, n_time_parts, part):
        """GRID split (reading M-2): TREES part part // n_time_parts x TIME part part % n_time_parts."""
        self._ck(_lib.cc_partition_grid(self._h, n_tree_parts, n_time_parts, part))

    def part_info(self):
        s = cc_part_stats()
        self._ck(_lib.cc_part_info(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in cc_part_stats._fields_}

    def leaf_owners(self):
        """{leaf id: owner part} under the current TREES / GRID split (reading E-11)."""
        n = c_i64()
        self._ck(_lib.cc_leaf_owners(self._h, None, None, 0, ctypes.byref(n)))
        ids = (c_i64 * max(n.value, 1))()
        own = (c_i32 * max(n.value, 1))()
        self._ck(_lib.cc_leaf_owners(self._h, ids, own, n.value, ctypes.byref(n)))
        return {int(ids[i]): int(own[i]) for i in range(n.value)}

    def part_time_range(self):
        t0, t1 = c_i32(), c_i32()
        self._ck(_lib.cc_part_time_range(self._h, ctypes.byref(t0), ctypes.byref(t1)))
        return t0.value, t1.value

    def part_trees(self):
        n = c_i64()
        self._ck(_lib.cc_part_trees(self._h, None, 0, ctypes.byref(n)))
        out = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_part_trees(self._h, out, n.value, ctypes.byref(n)))
        return list(out[:n.value])

    # --- schedule / plan -----------------------------------------------------------------
    def schedule(self, algo=CC_TREE, cap_bytes=0, given=None, evict_next_use=False, peer_cap_bytes=0,
                 peer_leaves=()):
        """peer_cap_bytes / peer_leaves: the peer-HBM tier (readings E-10, E-11; cc.h)."""
        cfg = cc_sched_cfg()
        cfg.algo = algo
        cfg.flags = CC_EVICT_NEXT_USE if evict_next_use else 0
        cfg.cap_bytes = int(cap_bytes or 0)
        if given is not None:
            g = (c_i64 * max(len(given), 1))(*given)
            cfg.given_order = ctypes.cast(g, P(c_i64))
            cfg.n_given = len(given)
        cfg.peer_cap_bytes = int(peer_cap_bytes or 0)
        pl = sorted(int(x) for x in peer_leaves)
        if pl:
            parr = (c_i64 * len(pl))(*pl)
            cfg.peer_leaves = ctypes.cast(parr, P(c_i64))
            cfg.n_peer_leaves = len(pl)
        n = c_i64()
        stats = cc_plan_stats()
        self._ck(_lib.cc_schedule(self._h, ctypes.byref(cfg), None, 0, ctypes.byref(n), ctypes.byref(stats)))
        out = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_schedule(self._h, ctypes.byref(cfg), out, n.value, ctypes.byref(n), ctypes.byref(stats)))
        st = {f: getattr(stats, f) for f, _ in cc_plan_stats._fields_}
        return list(out[:n.value]), st

    def memory_trace(self):
        n = c_i64()
        self._ck(_lib.cc_memory_trace(self._h, None, None, 0, ctypes.byref(n)))
        m = (c_i64 * (n.value + 1))()
        t = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_memory_trace(self._h, m, t, n.value + 1, ctypes.byref(n)))
        return list(m[:n.value + 1]), list(t[:n.value])

    def plan_ops(self):
        n = c_i64()
        self._ck(_lib.cc_plan_ops(self._h, None, 0, ctypes.byref(n)))
        out = (cc_plan_op * max(n.value, 1))()
        self._ck(_lib.cc_plan_ops(self._h, out, n.value, ctypes.byref(n)))
        return [(OP_KINDS[o.kind], o.node, o.bytes, o.offset) for o in out[:n.value]]

    def phys_plan(self, pool_bytes, compact=False, next_fit=False):
        """Host-side placement of the current plan (cc_phys_plan): stats dict."""
        st = cc_phys_stats()
        self._ck(_lib.cc_phys_plan(self._h, int(pool_bytes), (1 if compact else 0) | (2 if next_fit else 0),
                                   ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in cc_phys_stats._fields_}

    def scratch_of(self):
        n = c_i64()
        self._ck(_lib.cc_scratch_of(self._h, ctypes.byref(n)))
        return int(n.value)

    def phys_ops(self):
        """[(kind, node, bytes, offset, dst, off_a, off_b)] of the last phys_plan (kind 7: MOVE)."""
        n = c_i64()
        self._ck(_lib.cc_phys_ops(self._h, None, 0, ctypes.byref(n)))
        out = (cc_phys_op * max(n.value, 1))()
        self._ck(_lib.cc_phys_ops(self._h, out, n.value, ctypes.byref(n)))
        return [(o.kind, o.node, o.bytes, o.offset, o.dst, o.off_a, o.off_b) for o in out[:n.value]]

    def tree_order(self):
        n = c_i64()
        self._ck(_lib.cc_tree_order(self._h, None, 0, ctypes.byref(n)))
        out = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_tree_order(self._h, out, n.value, ctypes.byref(n)))
        return list(out[:n.value])

    def plan_dump(self, path):
        self._ck(_lib.cc_plan_dump(self._h, path.encode()))

    # --- data / execution ----------------------------------------------------------------
    def set_leaf(self, leaf_id, host, nbytes=None):
        nbytes = nbytes if nbytes is not None else host.numel() * host.element_size() if hasattr(host, "numel") \
            else host.nbytes
        self._ck(_lib.cc_set_leaf(self._h, leaf_id, _ptr(host), nbytes))

    def set_leaf_device(self, leaf_id, dev, nbytes=None):
        nbytes = nbytes if nbytes is not None else dev.numel() * dev.element_size()
        self._ck(_lib.cc_set_leaf_device(self._h, leaf_id, _ptr(dev), nbytes))

    def set_leaf_peer(self, leaf_id, dev, nbytes=None):
        """E-11: the leaf's full copy in (a peer GPU's) device memory; dev is a torch tensor or
        an integer device address (e.g. a CUDA IPC mapping)."""
        if isinstance(dev, int):
            ptr = dev
            assert nbytes is not None
        else:
            ptr = _ptr(dev)
            nbytes = nbytes if nbytes is not None else dev.numel() * dev.element_size()
        self._ck(_lib.cc_set_leaf_peer(self._h, leaf_id, ptr, nbytes))

    def set_peer_tier(self, dev, nbytes=None):
        """E-10: the peer-HBM eviction tier region (torch tensor or integer address; None: remove)."""
        if dev is None:
            self._ck(_lib.cc_set_peer_tier(self._h, None, 0))
            return
        if isinstance(dev, int):
            ptr = dev
            assert nbytes is not None
        else:
            ptr = _ptr(dev)
            nbytes = nbytes if nbytes is not None else dev.numel() * dev.element_size()
        self._ck(_lib.cc_set_peer_tier(self._h, ptr, nbytes))

    def execute(self, flags=0):
        s = cc_exec_stats()
        self._ck(_lib.cc_execute(self._h, flags, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in cc_exec_stats._fields_ if f != "pad_"}

    def execute_async(self, flags=0):
        self._ck(_lib.cc_execute_async(self._h, flags))

    def options(self):
        o = cc_options()
        self._ck(_lib.cc_get_options(self._h, ctypes.byref(o)))
        return {f: getattr(o, f) for f, _ in cc_options._fields_ if f != "pad_"}

    def set_options(self, **kw):
        """Change executor options (cc.h cc_options); unnamed ones keep their current value."""
        o = cc_options()
        self._ck(_lib.cc_get_options(self._h, ctypes.byref(o)))
        for k, v in kw.items():
            if k not in dict(cc_options._fields_) or k == "pad_":
                raise KeyError(k)
            setattr(o, k, v)
        self._ck(_lib.cc_set_options(self._h, ctypes.byref(o)))

    def kernel_times(self):
        s = (c_dbl * CC_N_OPS)()
        c = (c_i64 * CC_N_OPS)()
        self._ck(_lib.cc_kernel_times(self._h, s, c))
        return list(s), list(c)

    def dataflow_state(self):
        n = c_i64()
        self._ck(_lib.cc_dataflow_state(self._h, None, 0, ctypes.byref(n)))
        out = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_dataflow_state(self._h, out, n.value, ctypes.byref(n)))
        return list(out[:n.value])

    def dataflow_profile(self, per_sm=False):
        """(gemm_items, trace_items) arrays [n, 8]: claim, ready, published (ns), smid, first data,
        stage-loop end, kind; with per_sm also the per-CTA cycle counters [num_sms, 8] (cc.h)."""
        ng, nt = c_i64(), c_i64()
        self._ck(_lib.cc_dataflow_profile(self._h, None, 0, ctypes.byref(ng), ctypes.byref(nt)))
        n = ng.value + nt.value
        n_all = n + 2048  # + one 16-word record per worker CTA (at most 1024 SMs)
        out = np.zeros(8 * n_all, dtype=np.uint64)
        self._ck(_lib.cc_dataflow_profile(self._h, out.ctypes.data_as(P(c_u64)), 8 * n_all, ctypes.byref(ng),
                                          ctypes.byref(nt)))
        a = out[:8 * n].reshape(n, 8)
        if per_sm:
            sm = out[8 * n:].reshape(-1, 16).view(np.int64)
            sm = sm[(sm[:, 4] + sm[:, 5]) > 0]
            return a[:ng.value], a[ng.value:], sm
        return a[:ng.value], a[ng.value:]

    def correlator(self, corr_id, Lt):
        out = np.empty(2 * Lt, dtype=np.float64)
        self._ck(_lib.cc_correlator(self._h, corr_id, out.ctypes.data_as(P(c_dbl)), Lt))
        return out[0::2] + 1j * out[1::2]

    def correlators(self, out=None):
        """All correlators [n_corr, Lt_part] complex128 (corr ids ascending) with one copy; `out`
        may be a preallocated (pinned) complex128 array / CPU tensor of that shape."""
        n = c_i64()
        self._ck(_lib.cc_correlator_device_ptr(self._h, None, ctypes.byref(n), None))
        t0, t1 = self.part_time_range()
        if out is None:
            out = np.empty((n.value, t1 - t0), dtype=np.complex128)
        if hasattr(out, "data_ptr"):
            ptr, numel = out.data_ptr(), out.numel() * 2
        else:
            ptr, numel = out.ctypes.data, out.size * 2
        self._ck(_lib.cc_correlators(self._h, ctypes.cast(ptr, P(c_dbl)), numel))
        return out

    def root_value(self, tree_id, Lt):
        out = np.empty(2 * Lt, dtype=np.float64)
        self._ck(_lib.cc_root_value(self._h, tree_id, out.ctypes.data_as(P(c_dbl)), Lt))
        return out[0::2] + 1j * out[1::2]

    def correlator_device_ptr(self):
        p = c_void_p()
        n = c_i64()
        self._ck(_lib.cc_correlator_device_ptr(self._h, ctypes.byref(p), ctypes.byref(n), None))
        ids = (c_i64 * max(n.value, 1))()
        self._ck(_lib.cc_correlator_device_ptr(self._h, ctypes.byref(p), ctypes.byref(n), ids))
        return p.value, n.value, list(ids[:n.value])

    # --- kernel entry points ---------------------------------------------------------------
    def mm1(self, A, B, C, Lt, N):
        self._ck(_lib.cc_mm1(self._h, _ptr(A), _ptr(B), _ptr(C), Lt, N))

    def bm1(self, A, M, C, Lt, N, S):
        self._ck(_lib.cc_bm1(self._h, _ptr(A), _ptr(M), _ptr(C), Lt, N, S))

    def bb2(self, A, B, C, Lt, N, S):
        self._ck(_lib.cc_bb2(self._h, _ptr(A), _ptr(B), _ptr(C), Lt, N, S))

    def mm1_ozaki(self, A, B, C, Lt, N, n_slices, workspace):
        self._ck(_lib.cc_mm1_ozaki(self._h, _ptr(A), _ptr(B), _ptr(C), Lt, N, n_slices, _ptr(workspace),
                                   workspace.numel() * workspace.element_size()))

    def gemm_ozaki(self, op, A, B, C, Lt, N, S, n_slices, workspace):
        self._ck(_lib.cc_gemm_ozaki(self._h, op, _ptr(A), _ptr(B), _ptr(C), Lt, N, S, n_slices, _ptr(workspace),
                                    workspace.numel() * workspace.element_size()))

    def i8gemm_tn(self, A, B, C, M, Nn, K):
        self._ck(_lib.cc_i8gemm_tn(self._h, _ptr(A), _ptr(B), _ptr(C), M, Nn, K))

    def tr_mm(self, A, B, c, Lt, N):
        self._ck(_lib.cc_tr_mm(self._h, _ptr(A), _ptr(B), _ptr(c), Lt, N))

    def bb1(self, A, B, T, Lt, N, S):
        self._ck(_lib.cc_bb1(self._h, _ptr(A), _ptr(B), _ptr(T), Lt, N, S))

    def bt2(self, A, X, C, Lt, N, S):
        self._ck(_lib.cc_bt2(self._h, _ptr(A), _ptr(X), _ptr(C), Lt, N, S))

    def bb3(self, A, B, c, Lt, N, S):
        self._ck(_lib.cc_bb3(self._h, _ptr(A), _ptr(B), _ptr(c), Lt, N, S))

    def fill_synthetic(self, dev, n, seed, leaf_id, e0, mode, sigma):
        self._ck(_lib.cc_fill_synthetic(self._h, _ptr(dev), n, seed, leaf_id, e0, mode, sigma))
