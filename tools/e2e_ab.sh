# host-buffer pipeline A/B (tools/e2e_probe.py per setting); usage (under gpurun): bash tools/e2e_ab.sh
for rep in 1 2; do for R in 4 2 1; do for C in 8 16; do
  echo "ramp_start=$R chunks=$C $(RK_PIPE_RAMP_START=$R RK_PIPE_CHUNKS=$C timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)"
done; done; done
