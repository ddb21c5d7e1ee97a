mkdir -p gpurun_out
SFG_TRACE_TILES=33 timeout 300 python scripts/trace_chain.py 5 128 /tmp/trace5.bin > gpurun_out/trace5.txt 2>&1
SFG_TRACE_TILES=33 SFG_CHAIN_MAX=128 timeout 300 python scripts/trace_chain.py 1 512 /tmp/trace1s.bin > gpurun_out/trace1s.txt 2>&1
SFG_TRACE_TILES=129 timeout 300 python scripts/trace_chain.py 1 512 /tmp/trace1.bin > gpurun_out/trace1.txt 2>&1
