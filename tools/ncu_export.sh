# Export an ncu report to text (summary, profile json/md, per-line listing, raw metrics CSV, SASS source
# CSV), gzip, and drop the .ncu-rep so gpurun_out stays under the 64 MiB pull limit.
# usage: bash tools/ncu_export.sh gpurun_out/NAME [ct_per_launch]
R=$1
[ -f $R.ncu-rep ] || { echo "no $R.ncu-rep"; exit 0; }
python tools/ncu_summary.py $R.ncu-rep 60 > $R.summary.txt 2>&1
python tools/ncu_to_profile.py $R.ncu-rep $R.profile $2 > /dev/null 2>&1
python tools/ncu_lines.py $R.ncu-rep 80 > $R.lines.txt 2>&1
ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.source.csv 2>/dev/null
ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
gzip -f $R.raw.csv $R.source.csv $R.details.csv
rm -f $R.ncu-rep
