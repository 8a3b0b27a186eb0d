# K1 bank-aware grouping vs identity order: bench kernel time, ncu wavefronts/instructions.
python -c "import torch; torch.zeros(1).cuda()"  # warm the CUDA context once
for e in "ST_FX_GROUPED=1" "ST_FX_NOGROUP=1"; do
  env $e python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > /tmp/b.json 2>/tmp/b.err; python -c "import json; d=json.load(open('/tmp/b.json')); print('$e', round(d['roofline']['kernel_ms'],4))" || tail -3 /tmp/b.err
  env $e ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:fcs_dense_fx -s 1 -c 1 python tools/prof_c4.py --reps 2 2>&1 | grep -E "duration|wavefronts|inst_exec" | sed "s/^/$e /"
done
python -m pytest tests/test_gpu_parity.py -q -k "dense or f32 or host" 2>&1 | tail -1
