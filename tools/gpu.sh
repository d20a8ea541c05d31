#!/bin/bash
# One parametrised GPU-box script (run through gpurun). Usage:
#   tools/gpu.sh OUT STEP [STEP ...]
# OUT is a directory name under gpurun_out/. Steps, run in order:
#   info                  GPU name, clocks, power limit, host cores and CPU model
#   tests                 pytest -m gpu (full GPU suite)
#   tests:EXPR            pytest -m gpu -k EXPR
#   smoke                 __graft_entry__.smoke()
#   bench[:ARGS]          python bench.py ARGS  (ARGS: comma-separated, e.g. bench:--workload,c4)
#   torchrun:N[:ARGS]     bench.py under torchrun with N ranks
#   ref[:ARGS]            python bench.py --impl reference ARGS
#   launches[:ARGS]       ncu launch list (gpu__time_duration) of a short bench with ARGS
#   ncu:WORKLOAD[:ARGS]   ncu --set full of the first SGNS launch of tools/probe.py WORKLOAD ARGS
#   ncuk:REGEX:WORKLOAD[:ARGS]  ncu --set full of the first launch matching REGEX in tools/probe.py WORKLOAD
#   py:SCRIPT[:ARGS]      python SCRIPT ARGS
#   env:VAR=VALUE         export VAR=VALUE for the following steps (env:VAR= unsets it)
# Every step has its own timeout; logs land in gpurun_out/OUT/.
set -u
OUT=gpurun_out/$1; shift
mkdir -p "$OUT"
i=0
for step in "$@"; do
  i=$((i+1))
  kind=${step%%:*}; rest=${step#*:}; [ "$rest" = "$step" ] && rest=""
  args=${rest//,/ }
  case $kind in
    info)
      { nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader; nproc;
        lscpu | grep "Model name"; } > "$OUT/info.txt" 2>&1; cat "$OUT/info.txt" ;;
    tests)
      if [ -n "$rest" ]; then K=(-k "$rest"); else K=(); fi
      timeout 2400 python -m pytest tests -m gpu -q "${K[@]}" > "$OUT/tests_$i.log" 2>&1
      echo "tests rc=$?" >> "$OUT/tests_$i.log"; tail -4 "$OUT/tests_$i.log" ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
      echo "smoke rc=$?" >> "$OUT/smoke.log"; tail -2 "$OUT/smoke.log" ;;
    bench)
      timeout 1200 python bench.py $args > "$OUT/bench_$i.json" 2> "$OUT/bench_$i.err"
      echo "bench rc=$?"; tail -c 1500 "$OUT/bench_$i.json" ;;
    torchrun)
      N=${rest%%:*}; a=${rest#*:}; [ "$a" = "$rest" ] && a=""; a=${a//,/ }
      timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" \
        --master-addr 127.0.0.1 --master-port $((29500 + i)) bench.py --gpus "$N" $a \
        > "$OUT/bench_n${N}_$i.json" 2> "$OUT/bench_n${N}_$i.err"
      echo "torchrun rc=$?"; tail -c 1500 "$OUT/bench_n${N}_$i.json" ;;
    ref)
      timeout 1200 python bench.py --impl reference $args > "$OUT/ref_$i.json" 2> "$OUT/ref_$i.err"
      echo "ref rc=$?"; tail -c 800 "$OUT/ref_$i.json" ;;
    launches)
      BCMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline $args"
      timeout 900 $BCMD > "$OUT/launches_bench_$i.log" 2>&1 && \
        timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file "$OUT/launches_$i.csv" $BCMD > "$OUT/launches_ncu_$i.log" 2>&1
      echo "launches rc=$?" ;;
    ncu|ncuk)
      if [ "$kind" = ncu ]; then RX=sgns; W=${rest%%:*}; a=${rest#*:}; [ "$a" = "$rest" ] && a="";
      else RX=${rest%%:*}; r2=${rest#*:}; W=${r2%%:*}; a=${r2#*:}; [ "$a" = "$r2" ] && a=""; fi
      a=${a//,/ }
      PCMD="python tools/probe.py $W 1 $a"
      timeout 900 $PCMD > "$OUT/probe_${W}_$i.log" 2>&1 && \
        timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$RX -s 1 -c 1 \
          -o /tmp/ncu_$i $PCMD > "$OUT/ncu_${W}_$i.log" 2>&1
      echo "ncu rc=$?"
      ncu -i /tmp/ncu_$i.ncu-rep --page raw --csv > "$OUT/ncu_${W}_${i}_raw.csv" 2>/dev/null
      ncu -i /tmp/ncu_$i.ncu-rep --page details --csv > "$OUT/ncu_${W}_${i}_details.csv" 2>/dev/null
      ncu -i /tmp/ncu_$i.ncu-rep --page source --csv --print-source sass > "$OUT/ncu_${W}_${i}_source.csv" 2>/dev/null ;;
    env)
      v=${rest%%=*}; val=${rest#*=}
      if [ -n "$val" ]; then export "$v=$val"; else unset "$v"; fi
      echo "env $v=$val" ;;
    py)
      S=${rest%%:*}; a=${rest#*:}; [ "$a" = "$rest" ] && a=""; a=${a//,/ }
      b=$(basename "$S" .py)
      timeout 1800 python "$S" $a > "$OUT/${b}_$i.log" 2>&1
      echo "$S rc=$?"; tail -15 "$OUT/${b}_$i.log" ;;
    *) echo "unknown step $step" ;;
  esac
done
du -sh "$OUT"
