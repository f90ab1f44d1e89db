"""Thin ctypes binding of libhrp (include/hrp.h): argument marshalling only.

Every function here forwards to the C entry point of the same name; all computation runs in
libhrp's CUDA kernels.  There is no CPU fallback: if libhrp.so is missing the import fails.
Device arguments are torch CUDA tensors (their data_ptr is passed); host arguments are numpy
arrays.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhrp.so")

HRP_OK, HRP_EINVAL, HRP_ENOMEM, HRP_ECUDA, HRP_ENCCL, HRP_ERANGE, HRP_ESTATE, HRP_ENUMERIC = \
    range(8)
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ERANGE", 6: "ESTATE",
          7: "ENUMERIC"}


class HrpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class hrp_profiles(C.Structure):
    _fields_ = [("n_jobs", C.c_int32), ("n_features", C.c_int32), ("solo_ticks", C.c_void_p),
                ("compute_pm", C.c_void_p), ("memory_pm", C.c_void_p), ("features", C.c_void_p)]


class hrp_slot(C.Structure):
    _fields_ = [("sm800", C.c_uint16), ("b8", C.c_uint8), ("domain", C.c_uint8)]


class hrp_space(C.Structure):
    _fields_ = [("window", C.c_int32), ("cmax", C.c_int32), ("mps_split_mask", C.c_uint32),
                ("mig", C.c_int32), ("n_layouts", C.c_int32), ("layout_nslots", C.c_void_p),
                ("layout_slots", C.c_void_p), ("interference_q3", C.c_int32)]


class hrp_train_cfg(C.Structure):
    _fields_ = [("n_envs", C.c_int32), ("batch", C.c_int32), ("replay_capacity", C.c_int32),
                ("hidden_layers", C.c_int32), ("hidden_width", C.c_int32), ("gamma", C.c_float),
                ("lr", C.c_float), ("reward_lambda", C.c_float), ("argmax_mode", C.c_int32),
                ("optimizer", C.c_int32), ("adam_beta1", C.c_float), ("adam_beta2", C.c_float),
                ("adam_eps", C.c_float), ("loss", C.c_int32), ("huber_kappa", C.c_float),
                ("precision", C.c_int32), ("agent", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run paper_2405_08754_b200.build.build()")
        L = C.CDLL(LIB_PATH)
        P, S, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int32, C.c_int64, C.c_uint64
        sig = {
            "hrp_env_create": [P, P, P, S, P, S, S, P, P, P],
            "hrp_env_destroy": [P],
            "hrp_nccl_unique_id": [P],
            "hrp_env_reset": [P, P],
            "hrp_env_step": [P, u64, P, P, P, P, P, P, P, P, P],
            "hrp_q_forward": [P, i64, P, P, P, P, P],
            "hrp_dqn_update": [P, P, S, P, P, P],
            "hrp_dqn_grad": [P, P, P, P, P, P],
            "hrp_apply_grad": [P, P, S],
            "hrp_bruteforce_optimum": [P, P, i64, P, P, P, P, P, P],
            "hrp_brute_create": [P, P, S, P, P],
            "hrp_brute_run": [P, i64, P, P, P, P, P, P],
            "hrp_brute_destroy": [P],
            "hrp_job_times": [P, i64, P, P, P, P, P, P],
            "hrp_layout_table": [P, i32, P, P, P, P, P, P],
            "hrp_decode_action": [P, i64, P, P, P],
            "hrp_get_weights": [P, P],
            "hrp_get_hidden": [P, S, i64, P],
            "hrp_set_weights": [P, P],
            "hrp_sync": [P],
            "hrp_profile": [P, S],
            "hrp_profile_read": [P, P, P],
            "hrp_eval_counts": [P, P],
            "hrp_diag_config": [S, S],
            "hrp_covered_counts": [P, P],
            "hrp_diag_alu": [S, S, S, P],
            "hrp_diag_gemm": [S, P, S, S, S, P, P, P, P, P, S, S, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name, rt in (("hrp_n_params", C.c_int64), ("hrp_head_width", C.c_int32),
                         ("hrp_launch_count", C.c_int64), ("hrp_eval_count", C.c_int64)):
            getattr(L, name).argtypes = [P]
            getattr(L, name).restype = rt
        L.hrp_last_error.restype = C.c_char_p
        L.hrp_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status):
    if status != HRP_OK:
        raise HrpError(status, lib().hrp_last_error().decode())


def _ptr(x):
    """Device pointer of a torch tensor (or None -> NULL)."""
    if x is None:
        return None
    return C.c_void_p(x.data_ptr())


def _hptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ---- struct builders (keep the backing numpy arrays alive on the struct) ----------------
def make_space(W, cmax, shares, mig=True, q3=1, layouts=None):
    mask = 0
    for s in shares:
        assert s % 5 == 0 and 5 <= s <= 95
        mask |= 1 << (s // 5)
    sp = hrp_space(W, cmax, mask, 1 if mig else 0, 0, None, None, q3)
    if layouts is not None:  # explicit table: list of [(sm800, b8, dom), ...]
        ns = np.array([len(l) for l in layouts], np.int32)
        sl = np.zeros((len(layouts), 4), dtype=[("sm800", "<u2"), ("b8", "u1"), ("dom", "u1")])
        for i, l in enumerate(layouts):
            for k, (a, b, d) in enumerate(l):
                sl[i, k] = (a, b, d)
        sp.n_layouts = len(layouts)
        sp.layout_nslots = _hptr(ns)
        sp.layout_slots = _hptr(sl)
        sp._keep = (ns, sl)
    return sp


def make_profiles(pool):
    T = np.ascontiguousarray(pool.solo_ticks, np.int64)
    c = np.ascontiguousarray(pool.compute_pm, np.int16)
    m = np.ascontiguousarray(pool.memory_pm, np.int16)
    f = np.ascontiguousarray(pool.features, np.float32)
    p = hrp_profiles(len(T), f.shape[1], _hptr(T), _hptr(c), _hptr(m), _hptr(f))
    p._keep = (T, c, m, f)
    return p


OPTIMIZERS = {"sgd": 0, "adam": 1}
LOSSES = {"squared": 0, "huber": 1}
PRECISIONS = {"3xtf32": 0, "fast": 1}
AGENTS = {"joint": 0, "sequential": 1}


def make_cfg(n_envs, batch, replay_capacity, hidden_layers, hidden_width, gamma=0.99, lr=1e-3,
             reward_lambda=0.0, argmax_mode=0, optimizer="sgd", adam=(0.9, 0.999, 1e-8),
             loss="squared", huber_kappa=1.0, precision="3xtf32", agent="joint"):
    return hrp_train_cfg(n_envs, batch, replay_capacity, hidden_layers, hidden_width, gamma, lr,
                         reward_lambda, argmax_mode, OPTIMIZERS[optimizer], adam[0], adam[1],
                         adam[2], LOSSES[loss], huber_kappa, PRECISIONS[precision],
                         AGENTS[agent])


# ---- entry points (same names as the C ABI) ---------------------------------------------
def hrp_env_create(space, profiles, cfg, device, cuda_stream, rank=0, world=1,
                   nccl_unique_id=None, init_weights=None):
    ctx = C.c_void_p()
    w = None if init_weights is None else np.ascontiguousarray(init_weights, np.float32)
    uid = None if nccl_unique_id is None else C.create_string_buffer(bytes(nccl_unique_id), 128)
    _check(lib().hrp_env_create(C.byref(space), C.byref(profiles), C.byref(cfg), device,
                                C.c_void_p(cuda_stream), rank, world, uid, _hptr(w),
                                C.byref(ctx)))
    return ctx


def hrp_env_destroy(ctx):
    _check(lib().hrp_env_destroy(ctx))


def hrp_nccl_unique_id():
    buf = C.create_string_buffer(128)
    _check(lib().hrp_nccl_unique_id(buf))
    return bytes(buf.raw)


def hrp_env_reset(ctx, d_windows):
    _check(lib().hrp_env_reset(ctx, _ptr(d_windows)))


def hrp_env_step(ctx, eps_threshold, d_u_explore, d_u_action, d_next_windows, d_actions,
                 d_rewards, d_done, d_corun=None, d_qsel=None, d_greedy=None):
    _check(lib().hrp_env_step(ctx, C.c_uint64(int(eps_threshold)), _ptr(d_u_explore),
                              _ptr(d_u_action), _ptr(d_next_windows), _ptr(d_actions),
                              _ptr(d_rewards), _ptr(d_done), _ptr(d_corun), _ptr(d_qsel),
                              _ptr(d_greedy)))


def hrp_q_forward(ctx, n, d_windows, d_sched, d_argmax, d_qmax, d_head=None):
    _check(lib().hrp_q_forward(ctx, int(n), _ptr(d_windows), _ptr(d_sched), _ptr(d_argmax),
                               _ptr(d_qmax), _ptr(d_head)))


def hrp_dqn_update(ctx, d_u_replay, sync_target, d_loss, d_sample_idx=None, d_astar=None):
    _check(lib().hrp_dqn_update(ctx, _ptr(d_u_replay), int(bool(sync_target)), _ptr(d_loss),
                                _ptr(d_sample_idx), _ptr(d_astar)))


def hrp_dqn_grad(ctx, d_u_replay, d_loss, d_grad, d_sample_idx=None, d_astar=None):
    _check(lib().hrp_dqn_grad(ctx, _ptr(d_u_replay), _ptr(d_loss), _ptr(d_sample_idx),
                              _ptr(d_astar), _ptr(d_grad)))


def hrp_apply_grad(ctx, d_grad, sync_target):
    _check(lib().hrp_apply_grad(ctx, _ptr(d_grad), int(bool(sync_target))))


def hrp_brute_create(space, profiles, device, cuda_stream):
    plan = C.c_void_p()
    _check(lib().hrp_brute_create(C.byref(space), C.byref(profiles), device,
                                  C.c_void_p(cuda_stream), C.byref(plan)))
    return plan


def hrp_brute_run(plan, n, d_windows, d_best, d_solo, d_rgs, d_bact, cuda_stream):
    _check(lib().hrp_brute_run(plan, int(n), _ptr(d_windows), _ptr(d_best), _ptr(d_solo),
                               _ptr(d_rgs), _ptr(d_bact), C.c_void_p(cuda_stream)))


def hrp_job_times(plan, n, d_windows, d_actions, d_corun, d_solo, d_member_time, cuda_stream):
    _check(lib().hrp_job_times(plan, int(n), _ptr(d_windows), _ptr(d_actions), _ptr(d_corun),
                               _ptr(d_solo), _ptr(d_member_time), C.c_void_p(cuda_stream)))


def hrp_brute_destroy(plan):
    _check(lib().hrp_brute_destroy(plan))


def hrp_bruteforce_optimum(space, profiles, n, d_windows, d_best, d_solo, d_rgs, d_bact,
                           cuda_stream):
    _check(lib().hrp_bruteforce_optimum(C.byref(space), C.byref(profiles), int(n),
                                        _ptr(d_windows), _ptr(d_best), _ptr(d_solo),
                                        _ptr(d_rgs), _ptr(d_bact), C.c_void_p(cuda_stream)))


def hrp_layout_table(space, cap=4096):
    n = C.c_int32()
    nt = C.c_int32()
    na = C.c_int64()
    ns = np.zeros(cap, np.int32)
    sl = np.zeros((cap, 4), dtype=[("sm800", "<u2"), ("b8", "u1"), ("dom", "u1")])
    st = np.zeros((cap, 4), np.uint8)
    _check(lib().hrp_layout_table(C.byref(space), cap, C.byref(n), _hptr(ns), _hptr(sl),
                                  _hptr(st), C.byref(nt), C.byref(na)))
    L = n.value
    return {"n_layouts": L, "nslots": ns[:L], "slots": sl[:L], "slot_type": st[:L],
            "n_types": nt.value, "n_actions": na.value}


def hrp_decode_action(space, idx):
    l = C.c_int32()
    g = (C.c_int32 * 4)()
    so = (C.c_int32 * 4)()
    _check(lib().hrp_decode_action(C.byref(space), int(idx), C.byref(l), g, so))
    k = sum(1 for x in g if x >= 0)
    return l.value, tuple(g[:k]), tuple(so[:k])


def hrp_n_params(ctx):
    return lib().hrp_n_params(ctx)


def hrp_head_width(ctx):
    return lib().hrp_head_width(ctx)


def hrp_launch_count(ctx):
    return lib().hrp_launch_count(ctx)


def hrp_get_weights(ctx):
    n = hrp_n_params(ctx)
    out = np.empty(2 * n, np.float32)
    _check(lib().hrp_get_weights(ctx, _hptr(out)))
    return out


def hrp_get_hidden(ctx, layer, rows, d_out):
    _check(lib().hrp_get_hidden(ctx, int(layer), int(rows), _ptr(d_out)))


def hrp_set_weights(ctx, w):
    w = np.ascontiguousarray(w, np.float32)
    _check(lib().hrp_set_weights(ctx, _hptr(w)))


KERNEL_CLASSES = ["encode", "gemm_fwd", "gemm_bwd", "select", "td", "sample", "sgd", "misc",
                  "allreduce", "head_bwd"]


def hrp_profile(ctx, enable):
    _check(lib().hrp_profile(ctx, int(bool(enable))))


def hrp_profile_read(ctx):
    ms = np.zeros(len(KERNEL_CLASSES), np.float64)
    cnt = np.zeros(len(KERNEL_CLASSES), np.int64)
    _check(lib().hrp_profile_read(ctx, _hptr(ms), _hptr(cnt)))
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


def hrp_eval_count(ctx):
    return lib().hrp_eval_count(ctx)


def hrp_eval_counts(ctx):
    out = np.zeros(2, np.int64)
    _check(lib().hrp_eval_counts(ctx, _hptr(out)))
    return int(out[0]), int(out[1])


def hrp_diag_alu(device, is_int, iters=4096):
    v = C.c_double(0.0)
    _check(lib().hrp_diag_alu(int(device), int(is_int), int(iters), C.byref(v)))
    return v.value


def hrp_diag_config(key, value):
    _check(lib().hrp_diag_config(int(key), int(value)))


def hrp_diag_gemm(device, cuda_stream, M, N, K, d_A, d_W, d_bias, d_D, reps=0, force_bn=0):
    """D = A . W^T + bias through the 3xTF32 GEMM; returns the average ms of `reps` launches."""
    ms = C.c_float(0.0)
    _check(lib().hrp_diag_gemm(int(device), C.c_void_p(cuda_stream), int(M), int(N), int(K),
                               _ptr(d_A), _ptr(d_W), _ptr(d_bias), _ptr(d_D), None, int(reps),
                               int(force_bn), C.byref(ms)))
    return ms.value


def hrp_covered_counts(ctx):
    out = np.zeros(2, np.int64)
    _check(lib().hrp_covered_counts(ctx, _hptr(out)))
    return int(out[0]), int(out[1])


def hrp_sync(ctx):
    _check(lib().hrp_sync(ctx))


def hrp_version():
    return lib().hrp_version().decode()
