mkdir -p gpurun_out
out=gpurun_out/pack.txt; : > $out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.txt 2>&1; echo "tests rc=$? $(tail -1 /tmp/t.txt)" >> $out; grep -E "^FAILED|^E " /tmp/t.txt | head -8 >> $out
python - >> $out 2>&1 <<'PY'
import os, paper_2111_12238_b200 as sf
for pk in ("0", "4", "8", "16"):
    os.environ["SFG_IC_PACK"] = pk
    for cfg, combo in ((2, 5), (4, 7)):
        if cfg == 4 and pk != "0":
            continue
        M = sf.config_matrix(cfg); st = sf.make_state(combo, M, seed=7).inspect()
        st.bench(3); t, k = st.bench(20); u, _ = st.bench(10, unfused=True)
        print("ic_pack=%s combo %d fused %.3f ms kernel %.3f unfused %.3f" % (pk, combo, t / 20, k, u / 10))
        st.close()
PY
cat $out
