mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for CFG in c5f c5u; do
bash tools/ncu_k7.sh $CFG
python tools/ncu_lines.py gpurun_out/k7_$CFG.ncu-rep 60 --by-instr > gpurun_out/k7_lines_instr_$CFG.txt 2>&1
python tools/ncu_lines.py gpurun_out/k7_$CFG.ncu-rep 40 > gpurun_out/k7_lines_stall_$CFG.txt 2>&1
rm -f gpurun_out/k7_$CFG.ncu-rep
done
