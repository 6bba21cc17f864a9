"""ctypes binding of the in-tree native library ``_lib/libsqf_b200.so``.

The library holds the sm_100a kernels (include/sqf_kernels.h) and the C++ host
trainer (include/sqf_trainer.h). There is no Python or CPU fallback for any
compute entry: if the library is missing this module raises on import.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SQF_LIB") or os.path.join(_HERE, "_lib", "libsqf_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_1904_01038_b200/csrc). There is no fallback path.")

lib = C.CDLL(LIB_PATH)

i32, i64, u64, f32, f64, vp, cp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p, C.c_char_p
P = C.POINTER

# dtypes / flags (sqf_kernels.h)
F32, F16, BF16 = 0, 1, 2
EPI_PREROUND, EPI_BIAS, EPI_RELU, EPI_MASK, EPI_RESIDUAL, EPI_ACCUM = 1, 2, 4, 8, 16, 32


class GemmArgs(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("dtype", C.c_int),
                ("a", vp), ("lda", i64), ("a_kmajor", C.c_int),
                ("b", vp), ("ldb", i64), ("b_kmajor", C.c_int),
                ("c", vp), ("ldc", i64),
                ("bias", vp), ("res", vp), ("ldr", i64), ("mask", vp), ("ldm", i64),
                ("flags", C.c_int), ("force_simt", C.c_int), ("tile_n", C.c_int), ("pair", C.c_int),
                ("workspace", vp), ("workspace_floats", i64), ("counters", vp), ("n_counters", C.c_int),
                ("stream_k", C.c_int), ("bias_grad", vp), ("max_sms", C.c_int)]


class AttnArgs(C.Structure):
    _fields_ = [("dtype", C.c_int), ("batch", C.c_int), ("q_width", C.c_int), ("k_width", C.c_int),
                ("heads", C.c_int), ("dh", C.c_int), ("causal", C.c_int), ("k_len", vp),
                ("q", vp), ("ldq", i64), ("k", vp), ("ldk", i64), ("v", vp), ("ldv", i64),
                ("o", vp), ("ldo", i64), ("stats", vp),
                ("dout", vp), ("lddo", i64), ("dq", vp), ("lddq", i64), ("dk", vp), ("lddk", i64),
                ("dv", vp), ("lddv", i64), ("scratch", vp)]


class StepStats(C.Structure):
    _fields_ = [("step", i64), ("loss", f64), ("nll", f64), ("ntokens", i64), ("ncorrect", i64),
                ("lr", f64), ("skipped", i32), ("_pad", i32), ("scale", f64)]

    def as_dict(self):
        return {"step": self.step, "loss": self.loss, "nll": self.nll, "ntokens": self.ntokens,
                "ncorrect": self.ncorrect, "lr": self.lr, "skipped": bool(self.skipped), "scale": self.scale}


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


# ---- kernels
sfk_last_error = _sig("sfk_last_error", cp)
sfk_num_sms = _sig("sfk_num_sms", C.c_int)
sfk_gemm = _sig("sfk_gemm", C.c_int, P(GemmArgs), vp)
sfk_embed_fwd = _sig("sfk_embed_fwd", C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp, f32, vp, vp)
sfk_embed_bwd_chunked = _sig("sfk_embed_bwd_chunked", C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, f32,
                             vp, vp, vp)
sfk_embed_bwd = _sig("sfk_embed_bwd", C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_int, vp, f32, vp, vp)
sfk_layernorm_fwd = _sig("sfk_layernorm_fwd", C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp)
sfk_layernorm_bwd = _sig("sfk_layernorm_bwd", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp, C.c_int,
                         vp, P(C.c_int), vp)
sfk_colsum_partial = _sig("sfk_colsum_partial", C.c_int, C.c_int, vp, C.c_int, C.c_int, i64, vp, P(C.c_int), vp)
sfk_colsum_finish = _sig("sfk_colsum_finish", C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp)
sfk_colsum = _sig("sfk_colsum", C.c_int, C.c_int, vp, C.c_int, C.c_int, i64, vp, vp, vp, vp)
sfk_layernorm_bwd_dx = _sig("sfk_layernorm_bwd_dx", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp, C.c_int,
                            vp)
sfk_layernorm_bwd_dx_acc = _sig("sfk_layernorm_bwd_dx_acc", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp,
                                vp, vp)
sfk_layernorm_bwd_dx_part = _sig("sfk_layernorm_bwd_dx_part", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp,
                                 vp, C.c_int, vp, P(C.c_int), vp)
sfk_layernorm_bwd_params_partial = _sig("sfk_layernorm_bwd_params_partial", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                        vp, vp, P(C.c_int), vp)
sfk_layernorm_bwd_params_fold = _sig("sfk_layernorm_bwd_params_fold", C.c_int, C.c_int, vp, C.c_int, vp)
sfk_layernorm_bwd_fold = _sig("sfk_layernorm_bwd_fold", C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp)
sfk_layernorm_bwd_params = _sig("sfk_layernorm_bwd_params", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp,
                                vp, vp, vp)
sfk_layernorm_bwd_fused = _sig("sfk_layernorm_bwd_fused", C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp,
                               C.c_int, vp, vp, vp, vp, vp)
sfk_attention_fwd = _sig("sfk_attention_fwd", C.c_int, P(AttnArgs), vp)
sfk_attention_bwd = _sig("sfk_attention_bwd", C.c_int, P(AttnArgs), vp)
sfk_attention_fwd_parts = _sig("sfk_attention_fwd_parts", C.c_int, P(AttnArgs), C.c_int, vp)
sfk_attention_bwd_parts = _sig("sfk_attention_bwd_parts", C.c_int, P(AttnArgs), C.c_int, vp)
sfk_attention_last_launches = _sig("sfk_attention_last_launches", C.c_int)
sfk_xent_fwd_bwd = _sig("sfk_xent_fwd_bwd", C.c_int, C.c_int, vp, C.c_int, C.c_int, i64, vp, C.c_int, f32, f32,
                        vp, vp, vp)
sfk_xent_reduce = _sig("sfk_xent_reduce", C.c_int, vp, C.c_int, vp, vp)
sfk_nonfinite = _sig("sfk_nonfinite", C.c_int, C.c_int, vp, i64, vp, vp)
sfk_adam = _sig("sfk_adam", C.c_int, C.c_int, vp, vp, C.c_int, vp, vp, vp, i64, f64, f64, f64, f64, f64, f64,
                f32, C.c_int, f32, vp, vp)
sfk_sgd = _sig("sfk_sgd", C.c_int, C.c_int, vp, vp, C.c_int, vp, i64, f64, f32, C.c_int, f32, vp, vp)
sfk_accumulate = _sig("sfk_accumulate", C.c_int, C.c_int, vp, vp, i64, vp)
sfk_cast = _sig("sfk_cast", C.c_int, vp, vp, C.c_int, i64, vp)
sfk_convert = _sig("sfk_convert", C.c_int, C.c_int, vp, C.c_int, vp, i64, vp)

# ---- trainer
sqf_last_error = _sig("sqf_last_error", cp)
sqf_nccl_unique_id = _sig("sqf_nccl_unique_id", C.c_int, vp)
sqf_trainer_create = _sig("sqf_trainer_create", vp, cp, P(cp), P(cp), C.c_int, vp, vp, vp, vp, C.c_int, C.c_int,
                          C.c_int, C.c_int, C.c_int, vp)
HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, vp, i64, C.c_int, vp)
COLL_F32, COLL_F16, COLL_BF16, COLL_F64 = 0, 1, 2, 3
sqf_trainer_create_host_collective = _sig("sqf_trainer_create_host_collective", vp, cp, P(cp), P(cp), C.c_int, vp,
                                          vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          HOST_ALLREDUCE_FN, vp)
sqf_trainer_collective = _sig("sqf_trainer_collective", cp, vp)
sqf_trainer_free = _sig("sqf_trainer_free", None, vp)
sfk_debug_gemm_trace = _sig("sfk_debug_gemm_trace", C.c_int, vp)
sqf_trainer_train_one = _sig("sqf_trainer_train_one", C.c_int, vp, P(StepStats))
sqf_trainer_train_step = _sig("sqf_trainer_train_step", C.c_int, vp, vp, vp, P(StepStats))
sqf_trainer_evaluate = _sig("sqf_trainer_evaluate", C.c_int, vp, vp, C.c_int, P(f64), P(f64), P(i64), P(i64))
sqf_trainer_num_params = _sig("sqf_trainer_num_params", i64, vp)
sqf_trainer_params = _sig("sqf_trainer_params", C.c_int, vp, vp)
sqf_trainer_set_params = _sig("sqf_trainer_set_params", C.c_int, vp, vp)
sqf_trainer_last_grads = _sig("sqf_trainer_last_grads", C.c_int, vp, vp)
sqf_trainer_manifest_size = _sig("sqf_trainer_manifest_size", C.c_int, vp)
sqf_trainer_manifest_entry = _sig("sqf_trainer_manifest_entry", C.c_int, vp, C.c_int, cp, C.c_int, P(i64), P(i64),
                                  P(i64))
sqf_trainer_adam_state = _sig("sqf_trainer_adam_state", C.c_int, vp, vp, vp, P(i64))
sqf_trainer_scaler = _sig("sqf_trainer_scaler", C.c_int, vp, P(f64), P(i64))
sqf_trainer_progress = _sig("sqf_trainer_progress", C.c_int, vp, P(i64), P(i32), P(i32), P(i32))
sqf_trainer_set_injector = _sig("sqf_trainer_set_injector", C.c_int, vp, vp, C.c_int)
sqf_trainer_restore = _sig("sqf_trainer_restore", C.c_int, vp, i64, i32, i32, f64, i64)
sqf_trainer_kernel_launches = _sig("sqf_trainer_kernel_launches", i64, vp)
sqf_trainer_last_step_ms = _sig("sqf_trainer_last_step_ms", f32, vp)
sqf_trainer_flush_ms = _sig("sqf_trainer_flush_ms", f32, vp)
sqf_last_status = _sig("sqf_last_status", C.c_int)
sqf_task_create = _sig("sqf_task_create", vp, cp, P(cp), P(cp), C.c_int)
sqf_task_free = _sig("sqf_task_free", None, vp)
sqf_task_info = _sig("sqf_task_info", C.c_int, vp, P(i32), P(i32), P(i32), P(i64), P(i64))
sqf_task_pairs = _sig("sqf_task_pairs", C.c_int, vp, vp, vp, vp, vp)
sqf_simulate_timeline = _sig("sqf_simulate_timeline", C.c_int, cp, vp, C.c_int)
sqf_trainer_save = _sig("sqf_trainer_save", C.c_int, vp, cp)
sqf_trainer_load = _sig("sqf_trainer_load", C.c_int, vp, cp, P(i32))
sqf_checkpoint_info = _sig("sqf_checkpoint_info", C.c_int, cp, P(i32), P(i64), P(i64), P(i64))
sqf_checkpoint_read = _sig("sqf_checkpoint_read", C.c_int, cp, vp, vp, vp, i64)
sqf_trainer_overlap_log = _sig("sqf_trainer_overlap_log", C.c_int, vp, P(i32), C.c_int, P(i32))
sqf_trainer_last_io_bytes = _sig("sqf_trainer_last_io_bytes", i64, vp, P(i64))
sqf_trainer_stream = _sig("sqf_trainer_stream", vp, vp)
sqf_trainer_set_profile = _sig("sqf_trainer_set_profile", C.c_int, vp, C.c_int)
sqf_trainer_profile = _sig("sqf_trainer_profile", cp, vp, C.c_int, P(f64), P(f64), P(f64), P(i64))
sqf_trainer_timeline = _sig("sqf_trainer_timeline", C.c_int, vp, vp, C.c_int)

# ---- host boundary pieces
sqf_synthetic_corpus = _sig("sqf_synthetic_corpus", C.c_int, C.c_int, C.c_int, C.c_int, f64, u64, vp, vp, vp, vp,
                            P(i64), P(i64))
sqf_corpus_create = _sig("sqf_corpus_create", vp, C.c_int, vp, vp, vp, vp)
sqf_corpus_free = _sig("sqf_corpus_free", None, vp)
sqf_make_batches = _sig("sqf_make_batches", C.c_int, vp, i64, C.c_int, u64, P(i32), vp, vp)
sqf_shuffle_epoch = _sig("sqf_shuffle_epoch", C.c_int, C.c_int, u64, C.c_int, vp)
sqf_make_minibatch = _sig("sqf_make_minibatch", C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, P(i64))
sqf_split_counts = _sig("sqf_split_counts", C.c_int, C.c_int, C.c_int, C.c_int, vp)
sqf_bucket_gradients = _sig("sqf_bucket_gradients", C.c_int, vp, C.c_int, i64, P(i32), vp, vp)
sqf_model_init = _sig("sqf_model_init", C.c_int, cp, P(cp), P(cp), C.c_int, vp, i64, P(i64), P(C.c_int))
sqf_scaler_run = _sig("sqf_scaler_run", C.c_int, f64, i64, f64, f64, vp, C.c_int, vp, P(i32))
sqf_schedule_lr = _sig("sqf_schedule_lr", C.c_int, cp, f64, i64, f64, f64, i64, f64, i64, P(f64))
sqf_quantize_fp16 = _sig("sqf_quantize_fp16", f32, f32)

# every symbol the public headers declare (checked by the CPU test suite)
EXPORTED = [n for n in dir() if n.startswith(("sfk_", "sqf_"))]


class NativeError(RuntimeError):
    """Raised for a negative status; `.code` is the reference error class."""

    CLASSES = {-1: "ConfigError", -2: "ShapeError", -3: "BoundsError", -4: "CapacityError",
               -5: "IntegrityError", -6: "DivergenceError", -7: "RegistryError", -8: "IoError",
               -9: "Error", -10: "DeviceError"}

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = self.CLASSES.get(code, "Error")
        super().__init__(f"{self.kind}: {msg}")


def check(status: int, kernel: bool = False) -> int:
    if status < 0:
        msg = (sfk_last_error() if kernel else sqf_last_error()) or b""
        raise NativeError(status, msg.decode(errors="replace"))
    return status


def cstrs(items):
    arr = (cp * max(1, len(items)))()
    for i, s in enumerate(items):
        arr[i] = s.encode() if isinstance(s, str) else s
    return arr

# ---- generation (include/sqf_trainer.h, reference generate.hpp)


class GenConfigC(C.Structure):
    _fields_ = [("beam", i32), ("max_len", i32), ("diverse_groups", i32), ("topk", i32), ("lenpen", f64),
                ("diverse_strength", f64), ("temperature", f64), ("seed", u64), ("no_cache", i32), ("host_select", i32)]


sqf_gen_config_default = _sig("sqf_gen_config_default", C.c_int, vp, P(GenConfigC))
sqf_generate = _sig("sqf_generate", C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, P(GenConfigC), vp, P(vp))
sqf_gen_count = _sig("sqf_gen_count", C.c_int, vp, C.c_int)
sqf_gen_hyp = _sig("sqf_gen_hyp", C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int, P(i32), P(f64), P(f64), P(i32),
                   P(i32))
sqf_gen_free = _sig("sqf_gen_free", None, vp)
sqf_score_hypothesis = _sig("sqf_score_hypothesis", C.c_int, f64, i64, f64, P(f64))
sqf_sample_from_topk = _sig("sqf_sample_from_topk", C.c_int, vp, C.c_int, C.c_int, f64, f64, P(i32))
sqf_batch_for_inference = _sig("sqf_batch_for_inference", C.c_int, vp, C.c_int, i64, P(i32), vp, vp)
sfk_gather_rows = _sig("sfk_gather_rows", C.c_int, vp, vp, vp, C.c_int, i64, i64, C.c_int, i64, vp)
sfk_beam_topk = _sig("sfk_beam_topk", C.c_int, C.c_int, vp, i64, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp,
                     vp, vp)
