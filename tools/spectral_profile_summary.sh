# Writes profiles/ncu_spectral_r01.txt from gpurun_out/{cprank1,iuv1}_final.ncu-rep
# (captured with: ncu --set full --import-source on --clock-control none -k regex:<kernel> -c 1
#  python tools/prof_spectral.py --reps 1 --which c2|c3).
extra() {
  ncu -i "$1" --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); d=dict(zip(rows[0],rows[2]))
for k in ['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed']: print('  ',k,d.get(k))"
}
{
echo "Spectral kernels, final round-1 versions: ncu --set full --clock-control none, one launch each"
echo "(tools/prof_spectral.py --reps 1 --which c2 / c3). Config 2: cp_rank1_kernel (500 items, 2 CTAs/SM);"
echo "config 3: iuv1_kernel (150 items). Step-by-step history: spectral_experiments_r01.txt."
echo; echo "== c2 cp_rank1_kernel"; python tools/ncu_summary.py gpurun_out/cprank1_final.ncu-rep; extra gpurun_out/cprank1_final.ncu-rep
echo; echo "== c3 iuv1_kernel"; python tools/ncu_summary.py gpurun_out/iuv1_final.ncu-rep; extra gpurun_out/iuv1_final.ncu-rep
} > profiles/ncu_spectral_r01.txt
