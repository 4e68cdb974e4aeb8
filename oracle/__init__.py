"""TEST INFRASTRUCTURE ONLY — the CPU checker.

ctypes wrappers over
  * liboracle.so          : the plain-C restatement (qarvd_oracle.c), and
  * _ref/libqarvd_ref.so  : the unmodified reference sources compiled by oracle/Makefile.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this package.  The product (paper_2605_21072_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int64, c_void_p, c_uint

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqarvd_ref.so")

_o = None
_r = None


def _p(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


def lib():
    global _o
    if _o is None:
        _o = ctypes.CDLL(ORACLE_SO)
        _o.oracle_quantize_act.restype = c_int64
        _o.oracle_quantize_act.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int,
                                           c_double, c_int, c_void_p, c_void_p]
        _o.oracle_prepare_weights.restype = c_int64
        _o.oracle_prepare_weights.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64,
                                              c_int64, c_int, c_void_p, c_void_p, c_void_p]
        _o.oracle_kernel_b.restype = None
        _o.oracle_kernel_b.argtypes = [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _o.oracle_epilogue_f32.restype = None
        _o.oracle_epilogue_f32.argtypes = [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _o.oracle_channel_norms.restype = None
        _o.oracle_channel_norms.argtypes = [c_void_p, c_int64, c_int64, c_void_p]
        _o.oracle_mad.restype = None
        _o.oracle_mad.argtypes = [c_void_p, c_int64, c_void_p, c_void_p]
        _o.oracle_analyze_norms.restype = None
        _o.oracle_analyze_norms.argtypes = [c_void_p, c_int64, c_double, c_double, c_int64,
                                            c_void_p, c_void_p, c_void_p, c_void_p]
        _o.oracle_scale_search_hist.restype = c_int
        _o.oracle_scale_search_hist.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                                c_int, c_void_p, c_int, c_void_p]
        _o.oracle_weighting.restype = None
        _o.oracle_weighting.argtypes = [c_int, c_void_p, c_int64, c_void_p]
        _o.oracle_round_half_even.restype = c_double
        _o.oracle_round_half_even.argtypes = [c_double]
        _o.oracle_weighted_loss.restype = c_int
        _o.oracle_weighted_loss.argtypes = [c_void_p, c_void_p, c_double, c_void_p, c_void_p,
                                            c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                            c_int64, c_void_p, c_void_p, c_int64, c_void_p,
                                            c_int64, c_void_p, c_void_p]
        _o.oracle_num_threads.restype = c_int
        _o.oracle_row_scale_formula_mismatches.restype = c_int64
    return _o


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _r
    if _r is None:
        _r = ctypes.CDLL(REF_SO)
        _r.ref_last_error.restype = ctypes.c_char_p
        _r.ref_set_threads.argtypes = [c_uint]
        _r.ref_num_threads.restype = c_uint
        _r.ref_quantize.argtypes = [c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_void_p,
                                    c_void_p]
        _r.ref_permute.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int, c_void_p]
        _r.ref_kernel_b.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                    c_int64, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p]
        _r.ref_analyze_layer.argtypes = [c_void_p, c_int64, c_int64, c_double, c_double, c_int64,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _r.ref_analyze_norms.argtypes = [c_void_p, c_int64, c_double, c_double, c_int64, c_void_p,
                                         c_void_p, c_void_p, c_void_p]
        _r.ref_build_plan_codes.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _r.ref_percentile_search.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p,
                                             c_void_p, c_void_p]
        _r.ref_weighting.argtypes = [c_int, c_void_p, c_int64, c_void_p]
        _r.ref_calibrate_layer.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double,
                                           c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                                           c_int, c_int, ctypes.c_uint64, ctypes.c_char_p, c_void_p,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _r.ref_calibrate_layer_bits.argtypes = list(_r.ref_calibrate_layer.argtypes) + [c_int, c_int]
        _r.ref_toy_qarq.argtypes = [ctypes.c_char_p, c_int, c_void_p]
        _r.ref_toy_qarq_bits.argtypes = [ctypes.c_char_p, c_int, c_int, c_void_p]
        _r.ref_qarq_layer.argtypes = [ctypes.c_char_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p]
        _r.ref_weighted_loss.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_double,
                                         c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        _r.ref_toy_weight.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_char_p, c_double, c_double, ctypes.c_char_p,
                                      c_void_p, c_void_p, c_void_p]
        _r.ref_round_half_even.restype = c_double
        _r.ref_round_half_even.argtypes = [c_double]
        _r.ref_time_chain_per_token.restype = c_double
        _r.ref_time_chain_per_token.argtypes = [c_void_p, c_int64, c_void_p, c_int, c_int64, c_void_p]
        _r.ref_time_toy_rollouts.restype = c_double
        _r.ref_time_toy_rollouts.argtypes = [c_int, c_int]
        _r.ref_time_linear.restype = c_double
        _r.ref_time_linear.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                       c_int64, c_int, c_void_p, c_void_p, c_double, c_int64,
                                       c_void_p]
    return _r


class RefError(RuntimeError):
    pass


def _rc(st):
    if st != 0:
        raise RefError(ref().ref_last_error().decode())


# ---- numpy helpers ----------------------------------------------------------

def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float_to_bf16 (bytes.hpp:40-45), vectorised."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


# ---- restatement wrappers -----------------------------------------------------

def quantize_act(x64: np.ndarray, gather=None, per_token=True, static_scale=0.0, bits=8):
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    m, k = x64.shape
    g = None if gather is None else np.ascontiguousarray(gather, dtype=np.int32)
    k_out = k if g is None else len(g)
    q = np.empty((m, k_out), dtype=np.int8)
    s = np.empty(m, dtype=np.float64)
    bad = lib().oracle_quantize_act(_p(x64), m, k, _p(g), k_out, int(per_token), static_scale,
                                    bits, _p(q), _p(s))
    return q, s, int(bad)


def prepare_weights(w64: np.ndarray, gather, k_outlier: int, bits=8):
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    g = None if gather is None else np.ascontiguousarray(gather, dtype=np.int32)
    k_pad = k if g is None else len(g)
    wq = np.empty((n, k_pad), dtype=np.int8)
    so = np.empty(n)
    sn = np.empty(n)
    bad = lib().oracle_prepare_weights(_p(w64), n, k, _p(g), k_pad, k_outlier, bits, _p(wq),
                                       _p(so), _p(sn))
    return wq, so, sn, int(bad)


def kernel_b(xq, wq, k_outlier, s_x, s_o, s_n, with_acc=False):
    xq = np.ascontiguousarray(xq, dtype=np.int8)
    wq = np.ascontiguousarray(wq, dtype=np.int8)
    m, k = xq.shape
    n = wq.shape[0]
    out = np.empty((m, n))
    ao = np.empty((m, n), dtype=np.int32) if with_acc else None
    an = np.empty((m, n), dtype=np.int32) if with_acc else None
    sx = np.ascontiguousarray(np.broadcast_to(np.asarray(s_x, dtype=np.float64), (m,)))
    lib().oracle_kernel_b(_p(xq), _p(wq), m, n, k, k_outlier, _p(sx),
                          _p(np.ascontiguousarray(s_o, dtype=np.float64)),
                          _p(np.ascontiguousarray(s_n, dtype=np.float64)), _p(out), _p(ao), _p(an))
    return (out, ao, an) if with_acc else out


def epilogue_f32(acc_o, acc_n, has_outlier, s_x32, s_o32, s_n32, bias32=None, out="bf16"):
    m, n = acc_n.shape
    acc_o = np.ascontiguousarray(acc_o, dtype=np.int32)
    acc_n = np.ascontiguousarray(acc_n, dtype=np.int32)
    ob = np.empty((m, n), dtype=np.uint16) if out == "bf16" else None
    of = np.empty((m, n), dtype=np.float32) if out != "bf16" else None
    c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
    sx, so, sn, b = c(s_x32), c(s_o32), c(s_n32), c(bias32)
    lib().oracle_epilogue_f32(_p(acc_o), _p(acc_n), m, n, int(has_outlier), _p(sx), _p(so),
                              _p(sn), _p(b), _p(ob), _p(of))
    return ob if out == "bf16" else of


def channel_norms(w64):
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    out = np.empty(k)
    lib().oracle_channel_norms(_p(w64), n, k, _p(out))
    return out


def mad(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    med, m = c_double(), c_double()
    lib().oracle_mad(_p(v), len(v), ctypes.byref(med), ctypes.byref(m))
    return med.value, m.value


def analyze_norms(norms, tau=3.5, alpha_min=1.2, align=32):
    norms = np.ascontiguousarray(norms, dtype=np.float64)
    k = len(norms)
    stats = np.empty(3)
    counts = np.empty(2, dtype=np.int64)
    raw = np.empty(k, dtype=np.int64)
    al = np.empty(k, dtype=np.int64)
    lib().oracle_analyze_norms(_p(norms), k, tau, alpha_min, align, _p(stats), _p(counts),
                               _p(raw), _p(al))
    return dict(median=stats[0], mad=stats[1], threshold=stats[2],
                raw=raw[:counts[0]].copy(), aligned=al[:counts[1]].copy())


def analyze_layer(w64, tau=3.5, alpha_min=1.2, align=32):
    norms = channel_norms(w64)
    d = analyze_norms(norms, tau, alpha_min, align)
    d["norms"] = norms
    return d


def scale_search_hist(x_bits, frames, rows, k, percentiles=(0.999, 0.9999, 0.99999),
                      weights=None, bits=8):
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    nc = len(percentiles)
    pct = np.asarray(percentiles, dtype=np.float64)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    res = np.empty(3 * nc + 2)
    st = lib().oracle_scale_search_hist(_p(x_bits), frames, rows, k, _p(pct), nc, _p(w), bits,
                                        _p(res))
    if st != 0:
        raise ValueError("non-finite input")
    return res


def weighting(kind: int, alpha_normalized, n):
    out = np.empty(n)
    a = None if alpha_normalized is None else np.ascontiguousarray(alpha_normalized, dtype=np.float64)
    lib().oracle_weighting(kind, _p(a), n, _p(out))
    return out


# ---- reference wrappers (compiled reference sources) --------------------------

def ref_quantize(x64, per_token=True, s=0.0, bits=8):
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    m, k = x64.shape
    codes = np.empty((m, k), dtype=np.int32)
    scales = np.empty(m)
    _rc(ref().ref_quantize(_p(x64), m, k, int(per_token), s, bits, _p(codes), _p(scales)))
    return codes, scales


def ref_permute(x64, perm, enabled=True):
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    out = np.empty_like(x64)
    _rc(ref().ref_permute(_p(x64), x64.shape[0], x64.shape[1],
                          _p(np.ascontiguousarray(perm, dtype=np.uint32)), int(enabled), _p(out)))
    return out


def ref_kernel_b(xq, wq, perm, n_outlier, enabled, s_x, s_o, s_n):
    xq = np.ascontiguousarray(xq, dtype=np.int32)
    wq = np.ascontiguousarray(wq, dtype=np.int32)
    m, k = xq.shape
    n = wq.shape[0]
    sx = np.atleast_1d(np.asarray(s_x, dtype=np.float64))
    out = np.empty((m, n))
    _rc(ref().ref_kernel_b(_p(xq), m, k, _p(wq), n, _p(np.ascontiguousarray(perm, dtype=np.uint32)),
                           n_outlier, int(enabled), _p(np.ascontiguousarray(sx)), int(sx.size > 1),
                           _p(np.ascontiguousarray(s_o, dtype=np.float64)),
                           _p(np.ascontiguousarray(s_n, dtype=np.float64)), _p(out)))
    return out


def ref_analyze_layer(w64, tau=3.5, alpha_min=1.2, align=32):
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    norms = np.empty(k)
    stats = np.empty(3)
    counts = np.empty(2, dtype=np.int64)
    raw = np.empty(k, dtype=np.int64)
    al = np.empty(k, dtype=np.int64)
    _rc(ref().ref_analyze_layer(_p(w64), n, k, tau, alpha_min, align, _p(norms), _p(stats),
                                _p(counts), _p(raw), _p(al)))
    return dict(norms=norms, median=stats[0], mad=stats[1], threshold=stats[2],
                raw=raw[:counts[0]].copy(), aligned=al[:counts[1]].copy())


def ref_analyze_norms(v, tau=3.5, alpha_min=1.2, align=32):
    v = np.ascontiguousarray(v, dtype=np.float64)
    k = len(v)
    stats = np.empty(3)
    counts = np.empty(2, dtype=np.int64)
    raw = np.empty(k, dtype=np.int64)
    al = np.empty(k, dtype=np.int64)
    _rc(ref().ref_analyze_norms(_p(v), k, tau, alpha_min, align, _p(stats), _p(counts), _p(raw),
                                _p(al)))
    return dict(median=stats[0], mad=stats[1], threshold=stats[2],
                raw=raw[:counts[0]].copy(), aligned=al[:counts[1]].copy())


def ref_build_plan_codes(w64, outliers, bits=8):
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    o = np.ascontiguousarray(outliers, dtype=np.int64)
    so, sn = np.empty(n), np.empty(n)
    perm = np.empty(k, dtype=np.uint32)
    wq = np.empty((n, k), dtype=np.int32)
    en = c_int()
    _rc(ref().ref_build_plan_codes(_p(w64), n, k, _p(o), len(o), bits, _p(so), _p(sn), _p(perm),
                                   _p(wq), ctypes.byref(en)))
    return dict(scale_outlier=so, scale_normal=sn, permutation=perm, wq=wq, enabled=bool(en.value))


def ref_percentile_search(x64, frames, rows, k, bits=8):
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    bp, sc = c_double(), c_double()
    mse = np.empty(3)
    _rc(ref().ref_percentile_search(_p(x64), frames, rows, k, bits, ctypes.byref(bp),
                                    ctypes.byref(sc), _p(mse)))
    return bp.value, sc.value, mse


def ref_weighting(kind: int, alpha_raw, n):
    a = np.ascontiguousarray(alpha_raw if alpha_raw is not None else np.ones(n), dtype=np.float64)
    out = np.empty(n)
    _rc(ref().ref_weighting(kind, _p(a), n, _p(out)))
    return out


def ref_toy_weight(layer, blocks=2, hidden=64, seed=1, pattern="", fraction=0.02, gamma=8.0):
    rows, cols = ctypes.c_int64(), ctypes.c_int64()
    _rc(ref().ref_toy_weight(blocks, hidden, seed, pattern.encode(), fraction, gamma,
                             layer.encode(), None, ctypes.byref(rows), ctypes.byref(cols)))
    out = np.empty((rows.value, cols.value))
    _rc(ref().ref_toy_weight(blocks, hidden, seed, pattern.encode(), fraction, gamma,
                             layer.encode(), _p(out), ctypes.byref(rows), ctypes.byref(cols)))
    return out


def row_scale_formula_mismatches() -> int:
    """Mismatches of the device row-scale formula vs fl(amax/qmax) over all bf16 amax, 2..8 bits."""
    return int(lib().oracle_row_scale_formula_mismatches())


def weighted_loss(x64, xq, s_x, w64, codes, s_wo, s_wn, outlier_mask, row_off, chunks, chunk_w):
    """oracle_weighted_loss: Eq. 5 over stacked samples (calibrate.cpp:201-224); all in
    ORIGINAL column order.  Returns (loss, per-sample errors)."""
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    m, k = x64.shape
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n = w64.shape[0]
    xq = np.ascontiguousarray(xq, dtype=np.int32)
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    ro = np.ascontiguousarray(row_off, dtype=np.int64)
    ch = np.ascontiguousarray(chunks, dtype=np.int64)
    cw = np.ascontiguousarray(chunk_w, dtype=np.float64)
    err = np.empty(max(1, len(ch)))
    loss = c_double()
    st = lib().oracle_weighted_loss(_p(x64), _p(xq), float(s_x), _p(w64), _p(codes),
                                    _p(np.ascontiguousarray(s_wo, dtype=np.float64)),
                                    _p(np.ascontiguousarray(s_wn, dtype=np.float64)),
                                    _p(np.ascontiguousarray(outlier_mask, dtype=np.uint8)), m, n, k,
                                    _p(ro), _p(ch), len(ch), _p(cw), len(cw), _p(err),
                                    ctypes.byref(loss))
    if st == 1:
        raise ValueError("weighted loss: empty batch")
    if st == 2:
        raise IndexError("weighted loss: sample chunk outside the weight vector")
    return loss.value, err[:len(ch)]


def ref_weighted_loss(w64, outliers, act_scale, x64, row_off, chunks, chunk_w):
    """The reference weighted_loss on a LearnableQuantState::init state; returns the loss and
    the state's deployable quantities (hard codes, group scales, act scale, outlier mask)."""
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    o = np.ascontiguousarray(outliers, dtype=np.int64)
    ro = np.ascontiguousarray(row_off, dtype=np.int64)
    ch = np.ascontiguousarray(chunks, dtype=np.int64)
    cw = np.ascontiguousarray(chunk_w, dtype=np.float64)
    loss, act = c_double(), c_double()
    codes = np.empty((n, k), dtype=np.int32)
    so, sn = np.empty(n), np.empty(n)
    mask = np.empty(k, dtype=np.uint8)
    _rc(ref().ref_weighted_loss(_p(w64), n, k, _p(o), len(o), float(act_scale), _p(x64), _p(ro),
                                _p(ch), len(ch), _p(cw), len(cw), ctypes.byref(loss), _p(codes),
                                _p(so), _p(sn), ctypes.byref(act), _p(mask)))
    return dict(loss=loss.value, codes=codes, s_wo=so, s_wn=sn, act_scale=act.value, mask=mask)


def ref_calibrate_layer(w64, outliers, act_scale, x64, row_off, chunks, chunk_w, iterations, batch_size,
                        seed, name, w_bits=8, act_bits=8):
    """The reference calibrate_layer (calibrate.cpp:298-396) on build_plan(W, outliers, w_bits)
    with a per-tensor symmetric act_bits activation scale."""
    w64 = np.ascontiguousarray(w64, dtype=np.float64)
    n, k = w64.shape
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    o = np.ascontiguousarray(outliers, dtype=np.int64)
    ro = np.ascontiguousarray(row_off, dtype=np.int64)
    ch = np.ascontiguousarray(chunks, dtype=np.int64)
    cw = np.ascontiguousarray(chunk_w, dtype=np.float64)
    codes = np.empty((n, k), dtype=np.int32)
    sn, so, isn, iso = np.empty(n), np.empty(n), np.empty(n), np.empty(n)
    sc = np.empty(3)
    tr = np.empty(max(1, iterations))
    _rc(ref().ref_calibrate_layer_bits(_p(w64), n, k, _p(o), len(o), float(act_scale), _p(x64), _p(ro),
                                       _p(ch), len(ch), _p(cw), len(cw), iterations, batch_size, seed,
                                       name.encode(), _p(codes), _p(sn), _p(so), _p(sc), _p(tr), _p(isn),
                                       _p(iso), int(w_bits), int(act_bits)))
    return dict(codes=codes, scale_normal=sn, scale_outlier=so, act_scale=sc[0], initial_loss=sc[1],
                final_loss=sc[2], trace=tr[:iterations], init_scale_normal=isn, init_scale_outlier=iso)


def ref_toy_qarq(path: str, iterations: int = 8, weight_bits: int = 8) -> int:
    """The reference's calibrated toy model saved as a QARQ file (weight_bits = 4: packed 4-bit
    codes); returns the layer count."""
    n = ctypes.c_int64()
    _rc(ref().ref_toy_qarq_bits(path.encode(), iterations, weight_bits, ctypes.byref(n)))
    return n.value


def ref_qarq_layer(path: str, idx: int):
    """Layer idx of the reference's load_quantized_model(path)."""
    meta = np.zeros(6, dtype=np.int64)
    _rc(ref().ref_qarq_layer(path.encode(), idx, _p(meta), None, None, None, None, None))
    pres, n, k = bool(meta[0]), int(meta[1]), int(meta[2])
    out = dict(preserved=pres, out_dim=n, in_dim=k, enabled=bool(meta[3]), outlier_count=int(meta[4]),
               bits=int(meta[5]))
    if pres:
        return out
    wq = np.empty((n, k), dtype=np.int32)
    sn, so = np.empty(n), np.empty(n)
    perm = np.empty(k, dtype=np.uint32)
    act = np.empty(2)
    _rc(ref().ref_qarq_layer(path.encode(), idx, _p(meta), _p(wq), _p(sn), _p(so), _p(perm), _p(act)))
    out.update(wq=wq, scale_normal=sn, scale_outlier=so, permutation=perm, act_scale=act[0], act_zero=act[1])
    return out


# ---- timed reference paths (bench.py's CPU baselines and --impl reference arm) ---------------
class _ChainLayer(ctypes.Structure):
    _fields_ = [("wq", c_void_p), ("n", c_int64), ("k", c_int64), ("perm", c_void_p),
                ("n_outlier", c_int64), ("enabled", c_int), ("s_o", c_void_p), ("s_n", c_void_p),
                ("gelu_after", c_int)]


class RefLinear:
    """A reference-format quantized linear: ref analyze_layer -> build_plan -> nearest codes
    (pre-permuted int32), its f64 group scales and permutation."""

    def __init__(self, w64: np.ndarray, gelu_after: bool = False, bits: int = 8):
        self.n, self.k = w64.shape
        rep = ref_analyze_layer(w64)
        self.outliers = np.asarray(rep["aligned"], dtype=np.int64)
        plan = ref_build_plan_codes(w64, self.outliers, bits)
        self.wq = np.ascontiguousarray(plan["wq"], dtype=np.int32)
        self.perm = np.ascontiguousarray(plan["permutation"], dtype=np.uint32)
        self.s_o = np.ascontiguousarray(plan["scale_outlier"], dtype=np.float64)
        self.s_n = np.ascontiguousarray(plan["scale_normal"], dtype=np.float64)
        self.enabled = int(plan["enabled"])
        self.n_outlier = len(self.outliers) if self.enabled else 0
        self.gelu_after = int(gelu_after)


def ref_time_chain_per_token(x64: np.ndarray, layers, threads: int, rows_per_task: int = 0, want_y=False):
    """Seconds for the reference CPU path of a chain of per-token quantized linears over the
    rows of x64 (permute -> per-token kernel A -> kernel B [-> GELU] per layer), row blocks on
    the reference parallel_for with `threads` workers; optionally the f64 output."""
    r = ref()
    r.ref_set_threads(threads)
    x64 = np.ascontiguousarray(x64, dtype=np.float64)
    m = x64.shape[0]
    arr = (_ChainLayer * len(layers))()
    for i, L in enumerate(layers):
        arr[i] = _ChainLayer(L.wq.ctypes.data, L.n, L.k, L.perm.ctypes.data, L.n_outlier, L.enabled,
                             L.s_o.ctypes.data, L.s_n.ctypes.data, L.gelu_after)
    rpt = rows_per_task or max(1, (m + 4 * threads - 1) // (4 * threads))
    y = np.empty((m, layers[-1].n)) if want_y else None
    secs = r.ref_time_chain_per_token(_p(x64), m, ctypes.cast(arr, c_void_p), len(layers), rpt, _p(y))
    if secs < 0:
        raise RefError(r.ref_last_error().decode())
    return (secs, y) if want_y else secs


def ref_time_toy_rollouts(iterations: int, n_seeds: int, threads: int) -> float:
    r = ref()
    r.ref_set_threads(threads)
    secs = r.ref_time_toy_rollouts(iterations, n_seeds)
    if secs < 0:
        raise RefError(r.ref_last_error().decode())
    return secs
