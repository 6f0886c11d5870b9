#!/bin/bash
# usage: profiles/ncu_export.sh <report.ncu-rep> <outprefix>
# Export the pages ncu_summary.py reads, so the (large) report need not travel.
set -e
ncu -i "$1" --page details --csv > "$2.details.csv"
ncu -i "$1" --page raw --csv > "$2.raw.csv"
ncu -i "$1" --page source --csv --print-source sass > "$2.sass.csv"
ncu -i "$1" --page source --csv --print-source cuda,sass > "$2.cudasass.csv" || true
gzip -f "$2.sass.csv" "$2.cudasass.csv"
