# usage: bash tools/gpu_prof.sh <name> <kernel-regex> <prof_step args...>
# ncu --set full of one launch; CSV pages exported on the box (the .ncu-rep
# stays in /tmp: too large for gpurun_out)
name=$1; kre=$2; shift 2
mkdir -p gpurun_out
python tools/prof_step.py "$@" > gpurun_out/plain_$name.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$name.log; exit 1; }
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$kre" -c 1 \
  -o /tmp/prof_$name python tools/prof_step.py "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_${name}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/prof_${name}_details.csv 2>/dev/null
ncu -i /tmp/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${name}_sass.csv 2>/dev/null
ls -la gpurun_out/prof_${name}*
