"""Single-system solve pairs (combo 8) on the config-2 (7-pt 64^3) and config-1
(5-pt 512^2) patterns under each executor (SFG_EXECUTOR)."""
import os, sys, subprocess
if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2111_12238_b200 as sf
    cfg = int(sys.argv[1])
    M = sf.config_matrix(cfg)
    st = sf.make_state(8, M, seed=7).inspect()
    st.bench(3)
    tot, ker = st.bench(30)
    st.execute_fused()
    out = st.collect_outputs()
    print(f"cfg{cfg} {os.environ.get('SFG_EXECUTOR', 'default')}: {tot / 30:.4f} ms, checksum {float(out.sum()):.12e}")
    st.close()
else:
    for cfg in (2, 1):
        for ex in ("default", "chain", "levels"):
            env = dict(os.environ)
            if ex != "default":
                env["SFG_EXECUTOR"] = ex
            r = subprocess.run([sys.executable, __file__, str(cfg)], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr.strip()[-300:])
