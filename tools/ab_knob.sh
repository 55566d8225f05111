# usage: bash tools/ab_knob.sh "<ab_engine args>" ["<ab_engine args>" ...]
# builds in place, then runs tools/ab_engine.py once per argument string
export PYTHONPATH=$PWD
make -s -j16 -C paper_1811_01457_b200/csrc PYTHON=python all > gpurun_out/mk.log 2>&1 || { echo MAKE FAILED; tail gpurun_out/mk.log; exit 1; }
for a in "$@"; do
  timeout 600 python tools/ab_engine.py $a 2>&1 | tail -4
done
