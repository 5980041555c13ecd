"""GPU diagnostic: section-by-section comparison with the golden fixtures."""
import os, sys, struct, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import paper_2212_10733_b200 as mb
from paper_2212_10733_b200 import container
from tests import golden_util as G

def models(name):
    return [mb.AEModel(weights=w, norm_mean=m, norm_std=s) for (w, m, s) in G.models(name)]

for name in sys.argv[1:] or ["tiny", "small", "rowmode", "cfg1"]:
    meta, a = G.load(name)
    ds, same = G.corpus(name)
    print(f"== {name}: corpus same={same}", flush=True)
    for vi, run in enumerate(meta["runs"]):
        c = dict(run["cfg"]); c["newton"] = mb.NewtonOptions(**c["newton"])
        cfg = mb.PipelineConfig(**c)
        try:
            t0 = time.time()
            arc, rep, _ = mb.compress(ds, cfg, mb.TimestepState(models=models(name), timestep_index=1))
            dt = time.time() - t0
        except Exception:
            traceback.print_exc(); continue
        _, blobs = container.read_archive(arc)
        print(f" run{vi} tau={cfg.tau} {cfg.lambda_precision}: {dt:.2f}s arc_len {len(arc)} vs {run['archive_len']} "
              f"ratio {rep.compression_ratio:.4f} vs {run['ratio']:.4f} exc {rep.exception_count} vs {run['exceptions']} "
              f"archive_sha_eq={G.sha(arc)==run['archive_sha']}", flush=True)
        for si, b in enumerate(blobs):
            sb = container.read_shard(b); sec = sb.sections; ref = run["shards"][si]
            bad = []
            for k, rk in [("codes","codes_sha"),("pq_table","ptab_sha"),("residuals","res_sha"),("lambdas","lam_sha"),("exceptions","exc_sha")]:
                if G.sha(sec[k]) != ref[rk]: bad.append(k)
            eb, cnt = struct.unpack_from("<dI", sec["residuals"], 0)
            ne = struct.unpack_from("<I", sec["exceptions"], 0)[0]
            exc = [struct.unpack_from("<I", sec["exceptions"], 4 + k*(4+8*1521))[0] for k in range(ne)]
            msg = f"   shard{si}: bad={bad} eb {eb!r} vs {ref['eb']!r} nsel {cnt} vs {ref['n_sel']} nexc {ne} vs {len(ref['exceptions'])}"
            if exc != ref["exceptions"]:
                s1, s2 = set(exc), set(ref["exceptions"])
                msg += f" exc-only-gpu {sorted(s1-s2)[:10]} exc-only-ref {sorted(s2-s1)[:10]}"
            if "lambdas" in bad and f"r{vi}_s{si}_lam" in a:
                dt_ = "<f4" if cfg.lambda_precision == "f32" else "<f8"
                g = np.frombuffer(sec["lambdas"], dt_).reshape(-1, 8); r = np.frombuffer(a[f"r{vi}_s{si}_lam"].tobytes(), dt_).reshape(-1, 8)
                d = np.argwhere(g != r)
                msg += f" lam diffs {len(d)} first {d[:5].tolist()}"
                if len(d):
                    i, k = d[0]; msg += f" g={g[i,k]!r} r={r[i,k]!r}"
            if "codes" in bad and f"r{vi}_s{si}_codes" in a:
                g = np.frombuffer(sec["codes"], np.uint8); r = a[f"r{vi}_s{si}_codes"]
                msg += f" code byte diffs {int((g!=r).sum())}"
            if "pq_table" in bad and f"r{vi}_s{si}_ptab" in a:
                g = np.frombuffer(sec["pq_table"], "<f4"); r = np.frombuffer(a[f"r{vi}_s{si}_ptab"].tobytes(), "<f4")
                msg += f" ptab diffs {np.flatnonzero(g!=r)[:8].tolist()}"
            print(msg, flush=True)
        print(f"   report: pd {rep.pd_nrmse:.6e} vs {run['pd_nrmse']:.6e} maxq {rep.max_qoi_nrmse:.3e} vs {run['max_qoi_nrmse']:.3e} "
              f"conv {rep.convergence_fraction} vs {run['convergence_fraction']} ae_acc {rep.ae_accuracy} vs {run['ae_accuracy']} maxpi {rep.max_per_image_nrmse():.3e}", flush=True)
        if vi == 0:
            try:
                dec = mb.decompress(arc).data
                from oracle import port
                ref, _, _ = port.decompress(arc)
                rel = np.abs(dec - ref) / np.maximum(np.abs(ref), 1e-300)
                print(f"   decompress vs oracle-decode-of-gpu-archive: max rel {rel.max():.3e} exact frac {(dec==ref).mean():.4f}", flush=True)
            except Exception:
                traceback.print_exc()
