"""ctypes declarations of libpod.so (include/pod.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POD_LIB_PATH") or os.path.join(HERE, "libpod.so")   # override: A/B experiments only
MAX_HIDDEN = 4

STATUS = {0: "POD_OK", 1: "POD_ERR_ARG", 2: "POD_ERR_SHAPE", 3: "POD_ERR_RANGE", 4: "POD_ERR_WORKSPACE",
          5: "POD_ERR_CUDA", 6: "POD_ERR_NCCL", 7: "POD_ERR_NONFINITE", 8: "POD_ERR_UNSUPPORTED"}


class PodError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}: {detail}")


class EnvConfig(C.Structure):
    _fields_ = [("n_envs", C.c_int32), ("n_stocks", C.c_int32), ("n_feat", C.c_int32), ("n_agents", C.c_int32),
                ("horizon", C.c_int32), ("h_max", C.c_int32), ("env_offset", C.c_int64),
                ("initial_capital", C.c_double), ("cost_rate", C.c_double), ("reward_scale", C.c_double),
                ("gamma", C.c_double), ("seed", C.c_uint64)]


class Market(C.Structure):
    _fields_ = [("close", C.c_void_p), ("feat", C.c_void_p), ("T_data", C.c_int64)]


class Actor(C.Structure):
    _fields_ = [("n_hidden", C.c_int32), ("hidden", C.c_int32), ("act", C.c_int32), ("reserved", C.c_int32),
                ("params", C.c_void_p), ("param_bytes", C.c_size_t)]


class ActorLayout(C.Structure):
    _fields_ = [("obs_dim", C.c_int32), ("k_pad", C.c_int32), ("n_out_pad", C.c_int32), ("n_layers", C.c_int32),
                ("w_offset", C.c_size_t * (MAX_HIDDEN + 1)), ("w_rows", C.c_int32 * (MAX_HIDDEN + 1)),
                ("w_cols", C.c_int32 * (MAX_HIDDEN + 1)), ("b_offset", C.c_size_t * (MAX_HIDDEN + 1)),
                ("log_std_offset", C.c_size_t), ("param_bytes", C.c_size_t), ("n_elems", C.c_size_t)]


class PpoHparams(C.Structure):
    _fields_ = [("ratio_clip", C.c_float), ("entropy_coef", C.c_float), ("value_coef", C.c_float),
                ("learning_rate", C.c_float), ("adam_beta1", C.c_float), ("adam_beta2", C.c_float),
                ("adam_eps", C.c_float), ("fp32_operands", C.c_int32)]


class Traj(C.Structure):
    _fields_ = [("obs", C.c_void_p), ("act", C.c_void_p), ("logp", C.c_void_p), ("rew", C.c_void_p),
                ("done", C.c_void_p), ("mu", C.c_void_p), ("dbg_aint", C.c_void_p), ("dbg_hold", C.c_void_p),
                ("dbg_cash", C.c_void_p), ("val", C.c_void_p), ("equity", C.c_void_p)]


class Transfer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("src_local", C.c_int32), ("dst_local", C.c_int32)]


EXPORTS = ["pod_status_string", "pod_last_error", "pod_abi_version", "pod_kernel_launches", "pod_actor_layout_get",
           "pod_env_workspace_size", "pod_env_create", "pod_env_destroy", "pod_env_reset", "pod_rollout",
           "pod_env_profile", "pod_env_profile_read", "pod_debug_trace", "pod_env_fitness", "pod_env_read_state", "pod_env_check", "pod_gae", "pod_elite_plan", "pod_fuse_pods", "pod_fuse_workspace_size", "pod_fuse_pods_local_ranks", "pod_backtest_metrics", "pod_early_stop", "pod_ppo_workspace_size", "pod_ppo_update", "pod_ppo_check",
           "pod_elite_transfers", "pod_comm_unique_id", "pod_comm_init", "pod_comm_destroy", "pod_select_elite"]

_lib = None


def load():
    """Load the in-tree libpod.so.  There is no fallback: a missing library is an error."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(nvcc, sm_100a) — there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, d, f, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float, C.c_size_t
    P = C.POINTER
    sig = {
        "pod_status_string": ([C.c_int], C.c_char_p),
        "pod_last_error": ([], C.c_char_p),
        "pod_abi_version": ([], C.c_int),
        "pod_kernel_launches": ([], C.c_ulonglong),
        "pod_actor_layout_get": ([P(EnvConfig), i32, i32, P(ActorLayout)], C.c_int),
        "pod_env_workspace_size": ([P(EnvConfig), P(sz)], C.c_int),
        "pod_env_create": ([P(EnvConfig), P(Market), vp, sz, P(vp)], C.c_int),
        "pod_env_destroy": ([vp], C.c_int),
        "pod_env_reset": ([vp, vp, vp, vp], C.c_int),
        "pod_rollout": ([vp, P(Actor), i32, P(Traj), vp, i32, vp, vp], C.c_int),
        "pod_env_profile": ([vp, i32], C.c_int),
        "pod_debug_trace": ([vp, vp], C.c_int),
        "pod_env_profile_read": ([vp, P(d), P(d), P(d), P(d), vp], C.c_int),
        "pod_env_fitness": ([vp, vp, vp], C.c_int),
        "pod_env_read_state": ([vp, vp, vp, vp, vp, vp], C.c_int),
        "pod_env_check": ([vp, vp], C.c_int),
        "pod_fuse_pods": ([vp, P(EnvConfig), i32, i32, vp, sz, i32, i32, f, vp, vp, vp], C.c_int),
        "pod_fuse_workspace_size": ([P(EnvConfig), i32, i32, i32, i32, i32, P(sz)], C.c_int),
        "pod_fuse_pods_local_ranks": ([P(EnvConfig), i32, i32, vp, sz, i32, i32, i32, f, vp, vp, sz, vp], C.c_int),
        "pod_backtest_metrics": ([vp, vp, i32, i32, d, d, vp, vp], C.c_int),
        "pod_early_stop": ([vp, i32, i32, P(i32), P(i32)], C.c_int),
        "pod_ppo_workspace_size": ([P(EnvConfig), i32, i32, i32, P(sz)], C.c_int),
        "pod_ppo_update": ([P(EnvConfig), i32, i32, i32, P(PpoHparams), vp, vp, vp, i64, vp, sz, vp, vp, vp, vp, vp,
                            i64, vp, i32, i32, vp, vp, vp, sz, vp], C.c_int),
        "pod_ppo_check": ([vp, vp], C.c_int),
        "pod_gae": ([vp, vp, vp, vp, i32, i32, f, f, vp, vp, vp, vp], C.c_int),
        "pod_elite_plan": ([vp, i32, i32, vp], C.c_int),
        "pod_elite_transfers": ([vp, i32, i32, i32, P(Transfer), i32, P(i32)], C.c_int),
        "pod_comm_unique_id": ([vp], C.c_int),
        "pod_comm_init": ([vp, i32, i32, i32, P(vp)], C.c_int),
        "pod_comm_destroy": ([vp], C.c_int),
        "pod_select_elite": ([vp, vp, i32, i32, vp, sz, vp, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int, where: str):
    if status != 0:
        detail = load().pod_last_error().decode(errors="replace")
        raise PodError(status, where, detail)
