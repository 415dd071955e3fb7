"""CPU checks of the C ABI boundary: the library loads, exports every symbol
include/climber.h declares, and the ctypes structs match the C layout."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "climber.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(climber_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2502_09888_b200 import climber
    L = climber.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(climber.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", climber.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_struct_layout_matches_header():
    from paper_2502_09888_b200 import climber
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "climber.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(climber_config), offsetof(climber_config, rms_eps),
         offsetof(climber_config, kv_pages), sizeof(climber_weights), offsetof(climber_weights, b_head),
         sizeof(climber_events), sizeof(climber_strategy), offsetof(climber_config, rel_bias),
         offsetof(climber_weights, b_pos), offsetof(climber_weights, b_time));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as td:
        cpath = os.path.join(td, "t.c")
        open(cpath, "w").write(src)
        exe = os.path.join(td, "t")
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), cpath, "-o", exe])
        got = list(map(int, subprocess.check_output([exe]).split()))
    exp = [C.sizeof(climber._Config), climber._Config.rms_eps.offset, climber._Config.kv_pages.offset,
           C.sizeof(climber._Weights), climber._Weights.b_head.offset, C.sizeof(climber._Events),
           C.sizeof(climber._Strategy), climber._Config.rel_bias.offset, climber._Weights.b_pos.offset,
           climber._Weights.b_time.offset]
    assert got == exp


def _cfg(**kw):
    from paper_2502_09888_b200 import climber
    c = climber._Config()
    vals = dict(abi_version=climber.ABI_VERSION, d=128, n_heads=4, n_layers=2, n_blocks=4, n_k=64, ffn_mult=4, se_reduction=4,
                vocab=1000, n_actions=6, n_scenarios=4, max_candidates=128, hist_causal=1, dtype=0, page_tokens=64,
                rms_eps=1e-6, max_batch_users=8, max_wave_users=8, max_wave_pairs=1024, kv_pages=64)
    vals.update(kw)
    for k, v in vals.items():
        setattr(c, k, v)
    return c


def test_arena_bytes_and_config_validation_on_host():
    from paper_2502_09888_b200 import climber
    L = climber.lib()
    n = L.climber_arena_bytes(C.byref(_cfg()))
    assert n > 0
    # more pages -> more bytes, exactly page_bytes per page (page = 2 * 64 * d bf16)
    n2 = L.climber_arena_bytes(C.byref(_cfg(kv_pages=128)))
    assert L.climber_arena_bytes(C.byref(_cfg(rel_bias=1, dtype=1))) > n   # fp32: any n_k, + bias state
    assert n2 - n >= 64 * 2 * 64 * 128 * 2
    for bad in (dict(d=100), dict(n_heads=3), dict(n_k=48), dict(n_blocks=9), dict(page_tokens=32),
                dict(abi_version=1), dict(dtype=7), dict(max_wave_pairs=10), dict(rel_bias=2),
                dict(rel_bias=1, n_heads=8)):   # rel_bias on bf16 needs d_h in {32, 64} (here 16)
        assert L.climber_arena_bytes(C.byref(_cfg(**bad))) == 0, bad
    # create rejects a bad config synchronously, before touching the device
    h = C.c_void_p()
    st = L.climber_create(C.byref(_cfg(d=100)), None, None, C.c_void_p(256), 0, 0, 1, None, C.byref(h))
    assert st == 1  # null strategies/weights -> E_INVALID_ARG first
    strat = (climber._Strategy * 4)(*[climber._Strategy(1, 1)] * 4)
    w = climber._Weights()
    st = L.climber_create(C.byref(_cfg(d=100)), strat, C.byref(w), C.c_void_p(256), 1 << 20, 0, 1, None, C.byref(h))
    assert st == 2 and L.climber_last_error().startswith(b"config:")
    st = L.climber_create(C.byref(_cfg()), strat, C.byref(w), C.c_void_p(256), 1 << 20, 0, 2, None, C.byref(h))
    assert st == 1    # world > 1 without an NCCL unique id
    st = L.climber_create(C.byref(_cfg()), strat, C.byref(w), C.c_void_p(256), 1 << 20, 2, 2, None, C.byref(h))
    assert st == 1    # rank outside [0, world)


def test_nccl_unique_id_on_host():
    # libnccl is resolved at run time (dlopen); the unique id needs no GPU
    from paper_2502_09888_b200 import nccl_unique_id
    a, b = nccl_unique_id(), nccl_unique_id()
    assert len(a) == 128 and a != b
