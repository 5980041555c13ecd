"""Device reductions of the compress report (pipeline._build_report,
pipeline.py:367-391; qoi.py:122-133) through mlk_report (csrc/report.cu).

``launch`` queues the reduction of one or more CompressOuts and one async
copy of the results into page-locked memory; ``Stats`` names the values.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import REPORT_NVALS, MlkReportSeg, call

# value layout of mlk_report's output (include/mlk_b200.h)
DMAX, DMIN, SSE, QCNT, CONV, AE_OK, SEL, EXC = range(8)
Q_D2, Q_MAX, Q_MIN = slice(8, 12), slice(12, 16), slice(16, 20)


def _segment(out, order):
    d = out.dev
    keep = [d["flags"], d["status"], d["stats"], d["qoi"], d["fqoi"], d["fsse"], d["ferr"]]
    seg = MlkReportSeg(*[t.data_ptr() for t in keep],
                       order.data_ptr() if order is not None else None, d["flags"].numel())
    return seg, keep


def launch(outs, per_image: bool, orders=None):
    """Queue the reductions (and, with per_image, the per-image NRMSE list in
    dataset order) on the current stream; returns a handle for ``finish``."""
    dev = outs[0].dev["flags"].device
    n_tot = sum(o.dev["flags"].numel() for o in outs)
    segs = (MlkReportSeg * max(1, len(outs)))()
    keep = []
    for k, o in enumerate(outs):
        order = orders[k] if orders is not None else None
        segs[k], kk = _segment(o, order)
        keep += kk + [order]
    nblk = sum(min(296, (o.dev["flags"].numel() + 255) // 256) for o in outs)
    scratch = torch.empty(max(1, nblk) * REPORT_NVALS, dtype=torch.float64, device=dev)
    res = torch.empty(REPORT_NVALS + (n_tot if per_image else 0), dtype=torch.float64,
                      device=dev)
    call("mlk_report", ctypes.addressof(segs), len(outs), scratch, scratch.numel(), res,
         res[REPORT_NVALS:] if per_image and n_tot else None)
    host = torch.empty(res.shape, dtype=res.dtype, pin_memory=True)
    host.copy_(res, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return host, ev, n_tot, (segs, keep, scratch, res)


def finish(handle):
    """(values[20], per_image or None, n_images) once the copy has landed."""
    host_t, ev, n_tot, _ = handle
    ev.synchronize()
    host = host_t.numpy()
    vals = np.array(host[:REPORT_NVALS])
    per = host[REPORT_NVALS:] if host.size > REPORT_NVALS else None
    return vals, per, n_tot


def dataset_orders(outs):
    """Each CompressOut's dataset indices as device int64 tensors."""
    dev = outs[0].dev["flags"].device
    return [torch.from_numpy(np.ascontiguousarray(o.dataset_index, dtype=np.int64))
            .pin_memory().to(dev, non_blocking=True) for o in outs]
