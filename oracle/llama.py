"""ctypes wrapper of oracle/liboracle.so (llama_ref.c) — TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_llama_create.restype = C.c_void_p
        L.orc_llama_create.argtypes = [C.c_int] * 7 + [C.c_float, C.c_float, C.c_int, C.c_uint64,
                                                       C.c_uint64, C.c_double, C.c_float,
                                                       C.c_float, C.c_int]
        L.orc_llama_free.argtypes = [C.c_void_p]
        L.orc_llama_set_quant.argtypes = [C.c_void_p, C.c_int]
        L.orc_llama_set_pbf16.argtypes = [C.c_void_p, C.c_int]
        L.orc_llama_set_fp32.argtypes = [C.c_void_p, C.c_int]
        L.orc_llama_kv_compact.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int32, flags="C"),
                                           np.ctypeslib.ndpointer(np.int32, flags="C"), C.c_int]
        L.orc_llama_len.argtypes = [C.c_void_p]
        L.orc_llama_truncate.argtypes = [C.c_void_p, C.c_int]
        L.orc_llama_tensor.restype = C.POINTER(C.c_uint16)
        L.orc_llama_tensor.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_llama_plant_src.restype = C.POINTER(C.c_int32)
        L.orc_llama_plant_src.argtypes = [C.c_void_p]
        L.orc_llama_forward.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int32, flags="C"),
                                        C.c_int, C.c_void_p, C.c_int]
        _lib = L
    return _lib


class OracleLlama:
    """CPU Llama restatement with the product's synthetic-weight recipe."""

    def __init__(self, shape: dict, weight_seed: int, plant: dict | None = None,
                 max_seq: int = 512, threads: int = 8, w8a8: bool = False, fp32: bool = False):
        plant = plant or {}
        self.shape = dict(shape)
        self.V = shape["vocab"]
        self.h = lib().orc_llama_create(
            shape["n_layers"], shape["d_model"], shape["n_heads"],
            shape.get("n_kv_heads", shape["n_heads"]), shape["head_dim"], shape["ffn_dim"],
            shape["vocab"], shape.get("rms_eps", 1e-5), shape.get("rope_theta", 1e4), max_seq,
            weight_seed, plant.get("plant_seed", 0), plant.get("alpha", 0.0),
            plant.get("gain", 0.0), plant.get("emb_std", 0.0), threads)
        if w8a8:  # the product CPU draft's numerics (draft.cpp)
            lib().orc_llama_set_quant(self.h, 1)
        if fp32:  # fp32 activations / KV (the GPU's fp32-accumulate mode)
            lib().orc_llama_set_fp32(self.h, 1)

    def forward(self, tokens, last_only: bool = False) -> np.ndarray:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        rows = 1 if last_only else len(t)
        out = np.zeros((rows, self.V), dtype=np.float32)
        rc = lib().orc_llama_forward(self.h, t, len(t), out.ctypes.data, int(last_only))
        if rc != 0:
            raise RuntimeError(f"oracle forward failed ({rc})")
        return out

    def set_p_bf16(self, on: bool) -> None:
        """Diagnostic: round the softmax weights to bf16 before P.V."""
        lib().orc_llama_set_pbf16(self.h, int(on))

    def kv_compact(self, src, dst) -> None:
        s = np.ascontiguousarray(src, dtype=np.int32)
        d = np.ascontiguousarray(dst, dtype=np.int32)
        lib().orc_llama_kv_compact(self.h, s, d, len(s))

    def __len__(self):
        return lib().orc_llama_len(self.h)

    def truncate(self, n: int) -> None:
        lib().orc_llama_truncate(self.h, n)

    def tensor(self, which: int, layer: int, n: int) -> np.ndarray:
        p = lib().orc_llama_tensor(self.h, which, layer)
        return np.ctypeslib.as_array(p, shape=(n,)).copy()

    def plant_src(self) -> np.ndarray:
        return np.ctypeslib.as_array(lib().orc_llama_plant_src(self.h), shape=(self.V,)).copy()

    def close(self):
        if self.h:
            lib().orc_llama_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
