mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schedules.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_wave.txt 2>&1; echo rc=$?; tail -2 gpurun_out/t_wave.txt
python - <<'PY'
import paper_2111_12238_b200 as sf
for cfg, combo in ((1,4),(2,5),(3,6),(4,7)):
    M = sf.config_matrix(cfg); st = sf.make_state(combo, M, seed=7).inspect()
    st.bench(2); t,k = st.bench(5); st.bench(1, unfused=2); w,wk = st.bench(3, unfused=2)
    print(cfg, "fused %.3f ms  wavefront %.3f ms  levels %d" % (t/5, w/3, st.wavefront().nlevels()))
PY
