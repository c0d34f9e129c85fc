for C in 8 4 16 32; do for R in 1 0; do
  echo "chunks=$C ramp=$R $(RK_PIPE_CHUNKS=$C RK_PIPE_RAMP=$R timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)"
done; done
