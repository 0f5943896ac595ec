#!/bin/bash
# compute-sanitizer over small forwards of every arch (graphs and PDL off so each kernel is a
# plain launch).  Logs land in gpurun_out/sanitize/ (summaries copied to profiles/).
mkdir -p gpurun_out/sanitize
export HAPI_GRAPH=0 HAPI_PDL=0
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name regex:"conv|pool|pack|adaptive|bn_act|unpack" \
    --print-limit 20 python tools/sanitize_fwd.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(grep -c '^ok' gpurun_out/sanitize/$tool.log) ok, $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize/$tool.log | tail -2 | tr '\n' ' ')"
done
