"""ctypes mirrors of the structs in include/svt_b200.h (the C-ABI boundary).

Each struct mirrors one reference struct (file:line in the header)."""
import ctypes as C

SVT_OK, SVT_EINVAL, SVT_EDOMAIN, SVT_ERUNTIME, SVT_ECUDA, SVT_ENCCL, SVT_EOOM = range(7)

STOP_TRAIN_MAE, STOP_RESIDUAL, STOP_NONE = 0, 1, 2
BACKEND_R4SVD, BACKEND_R3SVD, BACKEND_RSVD_FIXED, BACKEND_FULL_SVD = 0, 1, 2, 3

# kernel classes reported by svt_ctx_kernel_stats
KCLASS = {0: "spmm", 1: "spmm_t", 2: "sddmm_update", 3: "cgs_gemm", 4: "rng", 5: "qr", 6: "finalize", 7: "other"}


class SketchParams(C.Structure):  # sketch.hpp:20-27
    _fields_ = [("t", C.c_int64), ("dt", C.c_int64), ("np", C.c_int32), ("reserved0", C.c_int32),
                ("eps_threshold", C.c_double), ("seed", C.c_uint64), ("p", C.c_int64)]

    def __init__(self, t=10, dt=10, np=1, eps_threshold=0.5, seed=1, p=5):
        super().__init__(t, dt, np, 0, eps_threshold, seed, p)


class SvtConfig(C.Structure):  # solver.hpp:32-43 (+ extensions)
    _fields_ = [("tau", C.c_double), ("delta", C.c_double), ("maxit", C.c_int32), ("np", C.c_int32),
                ("dt", C.c_int64), ("eps_stop", C.c_double), ("eps_threshold0", C.c_double),
                ("beta", C.c_double), ("t0", C.c_int64), ("seed", C.c_uint64),
                ("eps_threshold_min", C.c_double), ("rel_residual_stop", C.c_double)]

    def __init__(self, tau=0.0, delta=0.0, maxit=500, np=1, dt=10, eps_stop=1e-3, eps_threshold0=0.5,
                 beta=0.95, t0=10, seed=1, eps_threshold_min=0.0, rel_residual_stop=0.0):
        super().__init__(tau, delta, maxit, np, dt, eps_stop, eps_threshold0, beta, t0, seed,
                         eps_threshold_min, rel_residual_stop)

    def copy(self, **kw):
        d = {f[0]: getattr(self, f[0]) for f in self._fields_}
        d.update(kw)
        out = SvtConfig()
        for k, v in d.items():
            setattr(out, k, v)
        return out


class StopRule(C.Structure):  # solver.hpp:59-67
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_int32), ("threshold", C.c_double)]

    @staticmethod
    def train_mae(t):
        return StopRule(STOP_TRAIN_MAE, 0, t)

    @staticmethod
    def residual(t):
        return StopRule(STOP_RESIDUAL, 0, t)

    @staticmethod
    def none():
        return StopRule(STOP_NONE, 0, 0.0)


class Backend(C.Structure):  # solver.hpp:69-78
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_int32), ("fixed_rank", C.c_int64)]

    @staticmethod
    def r4svd():
        return Backend(BACKEND_R4SVD, 0, 0)

    @staticmethod
    def r3svd():
        return Backend(BACKEND_R3SVD, 0, 0)

    @staticmethod
    def rsvd_fixed(k):
        return Backend(BACKEND_RSVD_FIXED, 0, k)

    @staticmethod
    def full_svd():
        return Backend(BACKEND_FULL_SVD, 0, 0)


class IterationRecord(C.Structure):  # solver.hpp:49-57 (+ extensions)
    _fields_ = [("iter", C.c_int32), ("extension_rounds", C.c_int32), ("rank", C.c_int64),
                ("residual", C.c_double), ("eps_threshold", C.c_double), ("train_mae", C.c_double),
                ("sketch_ms", C.c_double), ("total_ms", C.c_double), ("kept", C.c_int64),
                ("rel_residual_x", C.c_double), ("test_mae", C.c_double), ("test_rmse", C.c_double)]

    def as_dict(self):
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


class SolverState(C.Structure):  # svt_solver_state (checkpoint / resume; no reference counterpart)
    _fields_ = [("iter", C.c_int32), ("done", C.c_int32), ("converged", C.c_int32), ("last_rounds", C.c_int32),
                ("s", C.c_int64), ("best_k", C.c_int64), ("eps_threshold", C.c_double), ("eps_min", C.c_double),
                ("best_metric", C.c_double), ("frob_y_sq", C.c_double), ("frob_a", C.c_double)]


OBSERVER_FN = C.CFUNCTYPE(C.c_int, C.POINTER(IterationRecord), C.c_int64, C.c_int64, C.c_int64,
                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


class InvalidArgument(ValueError):
    """std::invalid_argument (shape / parameter errors)."""


class DomainError(ArithmeticError):
    """std::domain_error (all-zero target)."""


class SvtRuntimeError(RuntimeError):
    """std::runtime_error / CUDA / NCCL failures."""


def raise_for(code, msg):
    if code == SVT_OK:
        return
    if code == SVT_EINVAL:
        raise InvalidArgument(msg)
    if code == SVT_EDOMAIN:
        raise DomainError(msg)
    raise SvtRuntimeError(f"[code {code}] {msg}")
