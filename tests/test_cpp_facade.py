"""The C++ facade (include/infllm_b200.hpp) from a C++ host: built with g++
against libinfllm_b200.so. CPU: defaults and the reference's ConfigError.
GPU: a small fp32 stream whose per-step retrieved ids and counters must equal
the oracle's (the inputs are regenerated here by the same integer hash)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2402_04617_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "facade_demo")


def build():
    if not os.path.exists(os.path.join(PKG, "libinfllm_b200.so")):
        subprocess.check_call(["make", "-s", "-C", PKG])
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC), os.path.getmtime(
            os.path.join(ROOT, "include", "infllm_b200.hpp"))):
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-o", BIN, SRC,
                               "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                               "-L", PKG, "-linfllm_b200", "-L", "/usr/local/cuda/lib64", "-lcudart",
                               f"-Wl,-rpath,{PKG}", "-Wl,-rpath,/usr/local/cuda/lib64"])
    return BIN


def test_facade_host_only():
    out = subprocess.run([build(), "cpu"], capture_output=True, text=True, check=True).stdout
    assert "defaults 512 128 4 4096 128 32 32 0.10" in out
    assert "ConfigError: hot_capacity must be >= n_lookup" in out


def hash_vals(count, salt):
    i = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (i + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15) ^ (np.uint64(salt) * np.uint64(0xD1B54A32D192ED03))
        x ^= x >> np.uint64(31)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
    return ((x >> np.uint64(40)).astype(np.float64) / 16777216.0 - 0.5).astype(np.float32)


@pytest.mark.gpu
def test_facade_stream_matches_oracle():
    out = subprocess.run([build(), "gpu"], capture_output=True, text=True, check=True).stdout.splitlines()
    n, H, G, d = 2048, 4, 2, 64
    q = hash_vals(n * H * d, 1).reshape(n, H, d)
    k = hash_vals(n * G * d, 2).reshape(n, G, d)
    v = (hash_vals(n * G * d, 3) * 2.0).astype(np.float32).reshape(n, G, d)
    cfg = O.EngineConfig.make(chunk_size=128, unit_size=128, n_repr=4, local_size=512, init_size=64, n_lookup=4,
                              hot_capacity=32, decay=0.1)
    eng = O.OracleEngine(cfg, O.ModelShape.make(n_heads=H, n_kv_heads=G, head_dim=d), n_threads=4)
    _, ids = O.run_engine(eng, q, k, v, O.encode_schedule(n, 128, 0), 0)
    got = [[int(x) for x in line.split()[1:]] for line in out if line.startswith("ids")]
    assert got == ids
    assert any("StreamError: encode_chunk: batch exceeds chunk_size" in line for line in out)
    eng.finish()
    m = eng.metrics()
    mline = [line for line in out if line.startswith("metrics")][0].split()
    assert int(mline[2]) == m["units"] and int(mline[4]) == m["hits"] and int(mline[6]) == m["misses"]
    assert int(mline[8]) == m["evictions"] and int(mline[10]) == m["requested"]
