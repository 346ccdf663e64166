"""Race / sync checking of the hand-rolled pipelines.

compute-sanitizer is closed on this pool (runs under it left GPUs needing a
reset), so the stand-in is the NB_CHECKS build libnb_checked.so (built by
__graft_entry__.build()): every mbarrier wait is bounded and traps with the
barrier and phase instead of hanging (a lost arrive, a phase error), bulk
copies check 16-byte alignment and sizes, kernels check that their TMEM
allocation starts at column 0, and the pipelined pair kernel checks its
logit / image write bounds.  Each small case (tools/sanitize.py; every tile
slot runs >= 2 tiles plus a ragged tail) runs under the checked build in a
subprocess and must exit cleanly with outputs bit-identical to the release
build's (logits, thresholds, counts, gradients, updated parameters)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2310_06822_b200", "libnb_checked.so")
PARTS = ["fwd_c2", "fwd_c3", "fwd_c5", "exit_c4", "fwd_4dbox", "train_c2", "train_c3", "train_c5"]


def run(lib, parts):
    cmd = [sys.executable, os.path.join(ROOT, "tools", "sanitize.py")] + (["--lib", lib] if lib else []) + parts
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "NB_CHECK" not in r.stdout + r.stderr, (r.stdout[-2000:], r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_checked_build_matches_release():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    assert os.path.exists(CHECKED), "libnb_checked.so not built (__graft_entry__.build())"
    rel = run("", PARTS)
    chk = run("checked", PARTS)
    assert rel == chk
    for p in PARTS:
        if "counts" in rel[p]:
            assert rel[p]["counts"]["fn"] == 0 or p == "exit_c4"


def test_checked_build_traps_a_lost_arrive():
    """The check itself works: a kernel waiting on an mbarrier phase nobody
    completes traps with the diagnostic (a launch failure) instead of hanging
    (the release build does not carry the self-test)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    code = ("import ctypes, sys; L = ctypes.CDLL(sys.argv[1]); "
            "print('rc', L.nb_debug_selftest_lost_arrive(), flush=True)")
    r = subprocess.run([sys.executable, "-c", code, CHECKED], capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert "NB_CHECK mbarrier timeout" in out or ("rc " in out and "rc 0" not in out), out[-2000:]
    rel = os.path.join(ROOT, "paper_2310_06822_b200", "libnb.so")
    r2 = subprocess.run([sys.executable, "-c", code, rel], capture_output=True, text=True, timeout=120)
    assert "rc 8" in r2.stdout, r2.stdout + r2.stderr   # NB_E_UNSUPPORTED


@pytest.mark.parametrize("name,n", [("c2", 128 * 148 * 5 + 77), ("c5", 256 * 74 + 3), ("c4", 128 * 300 + 1),
                                    ("c1", 4096 + 5)])
def test_output_guard_regions_untouched(name, n):
    """memcheck stand-in for the outputs: nb_forward / nb_encode / nb_score_async
    write exactly their rows; sentinel guard regions after each caller buffer
    stay untouched (ragged last tiles included)."""
    import ctypes as C

    import nbgen
    import paper_2310_06822_b200 as nb
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = nbgen.CONFIGS[name]
    m = nb.Model(nb.Desc(cfg.kind, cfg.space_dim, cfg.width, cfg.hidden_layers, tuple(cfg.head_after),
                         cfg.precision), 0)
    m.set_params(nbgen.init_params(cfg) * 2.0)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n, device="cuda:0")
    y = (q[:, 0] < 0.5).to(torch.uint8)
    G = 4096
    nl = 1 + cfg.n_heads
    logits = torch.full((n * nl + G,), 7.25, dtype=torch.float32, device="cuda:0")
    prob = torch.full((n + G,), 7.25, dtype=torch.float32, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    L = nb.lib()
    assert L.nb_forward(m._h, q.data_ptr(), n, logits.data_ptr(), prob.data_ptr(), st) == 0
    enc = torch.full((n * 16 + G,), 12345, dtype=torch.int16, device="cuda:0")
    if cfg.precision == "bf16":
        assert L.nb_encode(m._h, q.data_ptr(), n, enc.data_ptr(), st) == 0
    m.calibrate(q, y, allow_no_positives=True)
    out = torch.full((9 + 64,), -3, dtype=torch.int64, device="cuda:0")
    assert L.nb_score_async(m._h, q.data_ptr(), y.data_ptr(), n, out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert torch.all(logits[n * nl:] == 7.25) and torch.all(prob[n:] == 7.25)
    assert torch.all(enc[n * 16:] == 12345)
    assert torch.all(out[9:] == -3) and int(out[:4].sum()) == n
    assert torch.isfinite(logits[:n * nl]).all() and torch.all((prob[:n] >= 0) & (prob[:n] <= 1))
