cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mm
timeout 600 python tools/pack_sweep.py --graph --schedules multi:0x114,multi:0x124,multi:0x214,multi:0x144,multi:0x414,multi:0x116,multi:0x146,multi:0x1144,multi:0x2114,multi:0x2414 --steps 20 > gpurun_out/mm/sweep_g2.jsonl 2> gpurun_out/mm/sweep_g2.err
python - <<'P'
import json
for l in open("gpurun_out/mm/sweep_g2.jsonl"):
    d=json.loads(l); print(d["schedule"], hex(d["cluster"]), d["ms_median"], d["bit_exact"])
P
