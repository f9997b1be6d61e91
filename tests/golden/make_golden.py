"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports the read-only reference from
/root/reference; that tree does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz``.  The vectors pin the CPU oracle
(``oracle/``) to the reference's own outputs; the GPU parity tests then
compare the sm_100a kernels with the pinned oracle.

Every output below comes from a public reference call:
  * ``sasim.direct_conv``             (core.py:194-208)
  * ``sasim._kernels.tile_gather_nhwc`` (_kernels/__init__.py:49-50)
  * ``sasim.im2col_explicit``         (lowering.py:98-110)
  * ``sasim._kernels.lru_simulate``   (_kernels/__init__.py:57-59)
  * ``sasim.simulate(..., CHANNEL_FIRST_IMPLICIT).ofmap`` (simulator.py:458-536)
  * ``sasim.blocksched.reuse_traffic`` (blocksched.py:131-151)
Operands come from ``sasim.workloads.random_spec`` (workloads.py:111-142)
with the reference test-suite's integer operand convention
(tests/conftest.py:48-51, ints in [-4, 5)).
"""

import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("SASIM_PURE_PYTHON", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import sasim  # noqa: E402
from sasim import (ArchConfig, ColumnOrdering, ConvSpec, Layout, Method, Tensor,  # noqa: E402
                   direct_conv, im2col_explicit, simulate)
from sasim import _kernels as K  # noqa: E402
from sasim.blocksched import (SubtileOrder, order_subtiles, partition,  # noqa: E402
                              reuse_traffic, working_set_bytes)
from sasim.workloads import random_spec  # noqa: E402

SPEC_FIELDS = ("n", "c_i", "h_i", "w_i", "c_o", "h_f", "w_f", "stride_h", "stride_w",
               "pad_h", "pad_w", "dilation_h", "dilation_w")


def spec_vec(spec):
    return np.array([getattr(spec, f) for f in SPEC_FIELDS], dtype=np.int64)


def main():
    out = {}
    rng = np.random.default_rng(20261020)

    # 1. integer direct_conv over random specs (reference tests' value range)
    n_int = 0
    for i in range(64):
        spec = random_spec(rng, max_hw=12, max_n=4, max_co=16)
        x = rng.integers(-4, 5, size=(spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.int64)
        f = rng.integers(-4, 5, size=(spec.h_f, spec.w_f, spec.c_i, spec.c_o)).astype(np.int64)
        y = direct_conv(Tensor.from_array(x, Layout.NHWC), Tensor.from_array(f, Layout.HWCN), spec).view()
        out[f"int{n_int}_spec"] = spec_vec(spec)
        out[f"int{n_int}_x"] = x.astype(np.int8)
        out[f"int{n_int}_w"] = f.astype(np.int8)
        out[f"int{n_int}_y"] = y.astype(np.int32)
        assert np.array_equal(out[f"int{n_int}_y"], y)
        n_int += 1
    # full int8 range (what the int8 tensor-core path must match bit-exactly)
    for i in range(8):
        spec = random_spec(rng, max_hw=10, max_n=3, max_co=16, c_i_choices=(16, 32, 64, 128))
        x = rng.integers(-128, 128, size=(spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.int64)
        f = rng.integers(-128, 128, size=(spec.h_f, spec.w_f, spec.c_i, spec.c_o)).astype(np.int64)
        y = direct_conv(Tensor.from_array(x, Layout.NHWC), Tensor.from_array(f, Layout.HWCN), spec).view()
        out[f"int{n_int}_spec"] = spec_vec(spec)
        out[f"int{n_int}_x"] = x.astype(np.int8)
        out[f"int{n_int}_w"] = f.astype(np.int8)
        out[f"int{n_int}_y"] = y.astype(np.int32)
        assert np.array_equal(out[f"int{n_int}_y"], y)
        n_int += 1
    out["n_int"] = np.array(n_int)

    # 2. float32 direct_conv (BLAS tap accumulation in the reference)
    n_flt = 0
    for i in range(12):
        spec = random_spec(rng, max_hw=10, max_n=3, max_co=16, c_i_choices=(1, 3, 8, 16, 64))
        x = rng.standard_normal((spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.float32)
        f = rng.standard_normal((spec.h_f, spec.w_f, spec.c_i, spec.c_o)).astype(np.float32)
        y = direct_conv(Tensor.from_array(x, Layout.NHWC), Tensor.from_array(f, Layout.HWCN), spec).view()
        assert y.dtype == np.float32
        out[f"flt{n_flt}_spec"] = spec_vec(spec)
        out[f"flt{n_flt}_x"] = x
        out[f"flt{n_flt}_w"] = f
        out[f"flt{n_flt}_y"] = y
        n_flt += 1
    out["n_flt"] = np.array(n_flt)

    # 3. tile gathers and explicit im2col (both column orders)
    n_g = 0
    for i in range(10):
        spec = random_spec(rng, max_hw=9, max_n=2, max_co=4, c_i_choices=(1, 2, 3, 8))
        x = rng.integers(-9, 9, size=(spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.int64)
        r = int(rng.integers(spec.h_f))
        s = int(rng.integers(spec.w_f))
        g = K.tile_gather_nhwc(x, r, s, spec.stride_h, spec.stride_w, spec.pad_h, spec.pad_w,
                               spec.dilation_h, spec.dilation_w, spec.h_o, spec.w_o)
        cf = im2col_explicit(Tensor.from_array(x, Layout.NHWC), spec, ColumnOrdering.CHANNEL_FIRST).view()
        cl = im2col_explicit(Tensor.from_array(x, Layout.NHWC), spec, ColumnOrdering.CHANNEL_LAST).view()
        out[f"gat{n_g}_spec"] = spec_vec(spec)
        out[f"gat{n_g}_rs"] = np.array([r, s])
        out[f"gat{n_g}_x"] = x.astype(np.int8)
        out[f"gat{n_g}_g"] = g.astype(np.int8)
        out[f"gat{n_g}_cf"] = cf.astype(np.int8)
        out[f"gat{n_g}_cl"] = cl.astype(np.int8)
        n_g += 1
    out["n_gat"] = np.array(n_g)

    # 4. LRU replay
    n_l = 0
    for size, hi in ((5000, 64), (3000, 300), (20000, 1024)):
        keys = rng.integers(0, hi, size=size).astype(np.int64)
        for cap in (0, 1, 7, 64, 200, 1000):
            h, m = K.lru_simulate(keys, cap)
            out[f"lru{n_l}_keys"] = keys
            out[f"lru{n_l}_cap"] = np.array(cap)
            out[f"lru{n_l}_hm"] = np.array([h, m])
            n_l += 1
    out["n_lru"] = np.array(n_l)

    # 5. the paper's channel-first implicit path (functional half of simulate)
    n_s = 0
    arch = ArchConfig()
    for i in range(6):
        spec = random_spec(rng, max_hw=10, max_n=3, max_co=8, c_i_choices=(1, 3, 8, 16))
        x = rng.integers(-4, 5, size=(spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.int64)
        f = rng.integers(-4, 5, size=(spec.h_f, spec.w_f, spec.c_i, spec.c_o)).astype(np.int64)
        res = simulate(spec, arch, Method.CHANNEL_FIRST_IMPLICIT,
                       ifmap=Tensor.from_array(x, Layout.NHWC),
                       filters=Tensor.from_array(f, Layout.HWCN))
        y = res.ofmap.view()
        out[f"sim{n_s}_spec"] = spec_vec(spec)
        out[f"sim{n_s}_x"] = x.astype(np.int8)
        out[f"sim{n_s}_w"] = f.astype(np.int8)
        out[f"sim{n_s}_y"] = y.astype(np.int32)
        n_s += 1
    out["n_sim"] = np.array(n_s)

    # 6. reuse_traffic (LRU model of the subtile orders)
    n_t = 0
    for (spec, bm_div, bk) in ((ConvSpec.square(1, 4, 33, 4, 3, stride=2), 4, 4),
                               (ConvSpec.square(2, 2, 20, 2, 3, pad=1), 3, 2),
                               (ConvSpec.square(1, 8, 16, 4, 3, stride=1, pad=1, dilation=2), 2, 4)):
        plan = partition(spec, block_m=-(-spec.gemm_m // bm_div), block_n=spec.c_o, block_k=bk)
        ws = working_set_bytes(plan)
        for pol in (SubtileOrder.FILTER_MAJOR, SubtileOrder.REUSE_AWARE):
            for mult in (0, 1, 2):
                budget = mult * ws
                res = reuse_traffic(plan, order_subtiles(plan, pol), budget, spec)
                out[f"trf{n_t}_spec"] = spec_vec(spec)
                out[f"trf{n_t}_blk"] = np.array([plan.block_m, plan.block_n, bk, budget,
                                                 0 if pol is SubtileOrder.FILTER_MAJOR else 1])
                out[f"trf{n_t}_res"] = np.array([res.dram_bytes, res.hits, res.misses, ws])
                n_t += 1
    out["n_trf"] = np.array(n_t)

    out["ref_version"] = np.array(sasim.__version__)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes;",
          {k: int(out[k]) for k in ("n_int", "n_flt", "n_gat", "n_lru", "n_sim", "n_trf")})


if __name__ == "__main__":
    main()
