#!/bin/bash
# profiles/<name>.md from a gpurun_out/ holding full_*.ncu-rep captures, launches.csv and bench JSON lines
name=$1; shift
out=profiles/$name.md
{
  echo "# $name"
  echo
  for b in "$@"; do echo "## $(basename $b)"; echo '```'; tail -n 1 $b; echo '```'; echo; done
  if [ -f gpurun_out/launches.csv ]; then
    echo "## ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare shares)"
    echo; python tools/ncu_summary.py launches gpurun_out/launches.csv; echo
  fi
  echo "## ncu --set full captures (one launch each; -s = launches of that kernel skipped)"
  echo
  for f in gpurun_out/full_*.ncu-rep; do python tools/ncu_summary.py rep $f; echo; done
  echo "## top source lines (warp-stall samples / instructions)"
  for f in gpurun_out/full_*.ncu-rep; do echo; echo "### $(basename $f)"; echo '```'; python tools/ncu_lines.py $f 8; echo '```'; done
} > $out
echo wrote $out
