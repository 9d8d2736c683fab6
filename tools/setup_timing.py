"""Host set-up cost of nsm_setup (split + SELL build + upload) per config."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs, paper_2112_14681_b200 as nsm
for cfg in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    t0 = time.perf_counter(); A = inputs.config_matrix(cfg); tg = time.perf_counter() - t0
    F = None
    if cfg in ("C2", "C4"):
        t0 = time.perf_counter(); F = nsm.ilu0(A); tf = time.perf_counter() - t0
    else:
        tf = 0.0
    t0 = time.perf_counter(); S = nsm.Smoother(A, F); ts = time.perf_counter() - t0
    S.close()
    print(json.dumps({"cfg": cfg, "nnz": A.nnz, "generate_s": round(tg, 2), "ilu0_s": round(tf, 2), "setup_s": round(ts, 2)}), flush=True)
