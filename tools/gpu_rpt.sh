python -c "import paper_0907_4631_b200 as P; P.build()"
for r in 2 4 8; do echo "### RPT=$r"; PHIPM_RPT=$r python tools/trace_solve.py --configs c3,c4,c5 --out gpurun_out/trace_rpt$r.json 2>&1 | grep -v "^    "; done
