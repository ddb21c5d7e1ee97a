mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputests_clean.txt 2>&1; echo tests_rc=$?; tail -4 gpurun_out/gputests_clean.txt
python - <<'PY'
import paper_2111_12238_b200 as sf
for cfg, combo in ((2,5),(3,6),(4,7)):
    M = sf.config_matrix(cfg); st = sf.make_state(combo, M, seed=7).inspect()
    st.bench(3); t,k = st.bench(20); u,_ = st.bench(10, unfused=True)
    print(cfg, "fused %.3f ms kernel %.3f  unfused %.3f" % (t/20, k, u/10))
PY
