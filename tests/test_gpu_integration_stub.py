"""The maintainer-side ctypes stub printed in INTEGRATION.md §2, executed as
written (only the library path is made absolute): one reference-order sweep
through the raw C ABI equals the package's engine.sweep bit for bit."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import golden
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
from test_gpu_parity import make_ds, pkg_cfg
from test_oracle_golden import cfg_from_repr

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _stub_namespace():
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n# ptychokit/_b200.py.*?\n(.*?)```", text, re.S).group(1)
    lib = ROOT / "paper_2205_04295_b200" / "libptycho_b200.so"
    code = code.replace('C.CDLL("libptycho_b200.so")', f'C.CDLL("{lib}")')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def test_integration_stub_matches_engine(gpu):
    import torch
    ns = _stub_namespace()
    g = golden("sweep_rpie")
    cfg = pkg_cfg(cfg_from_repr(str(g["cfg_repr"])), "fp32")
    ds = make_ds(g["patterns"], g["positions_in"], g["window"])
    ref = pk.initialize(ds, cfg)
    st = pk.initialize(ds, cfg)
    pk.sweep(ref, ds, cfg)

    w, m, n = st.window, int(st.probe_stack.shape[0]), ds.n_positions
    order = torch.from_numpy(pk.engine.visit_order(n, cfg, 0).astype(np.int32)).cuda()
    pats = torch.from_numpy(np.ascontiguousarray(ds.patterns, np.float32)).cuda()
    pats_t = pats.transpose(1, 2).contiguous()
    err = torch.zeros(3, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    nbytes = ns["lib"].pty_sweep_workspace_bytes(0, w, m, n, 1)
    ws = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
    h, wc = st.obj.shape
    ns["sweep_inner_loop"](st.obj.data_ptr(), h, wc, st.canvas_origin, st.probe_stack.data_ptr(),
                           pats.data_ptr(), pats_t.data_ptr(), st.positions.data_ptr(), order.data_ptr(),
                           w, m, n, cfg, err.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(),
                           stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert torch.equal(st.obj, ref.obj)
    assert torch.equal(st.probe_stack, ref.probe_stack)
    num, den, _ = err.cpu().numpy()
    assert num / den == pytest.approx(ref.error_trace[-1], rel=1e-12)
