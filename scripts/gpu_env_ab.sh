# us/call for each value of one env knob: ENVVAR=<name> VALS="<v1> <v2> ..." SHAPES="R,K,L ..."
python build_pb.py > /dev/null 2>&1
for rep in 1 2; do for shape in ${SHAPES:-16384,16384,8}; do set -- ${shape//,/ }
 for v in ${VALS}; do
  echo "R=$1 K=$2 L=$3 ${ENVVAR}=$v $(env ${ENVVAR}=$v PYTHONPATH=. timeout -s KILL 60 python scripts/timeline.py --R $1 --K $2 --L $3 --copies ${COPIES:-2} --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
 done; done; done > gpurun_out/env_ab${TAG}.txt 2>&1
cat gpurun_out/env_ab${TAG}.txt
