# round 2 (re-entry): ncu evidence at HEAD for the bench default (papers-shaped, managed table)
bash scripts/gpu_ncu.sh r2ncu papers
R=gpurun_out/r2ncu
ncu -i $R/prof_papers.ncu-rep --page raw --csv > $R/prof_papers_raw.csv 2>/dev/null
ncu -i $R/prof_papers.ncu-rep --page details > $R/ncu_papers_details.txt 2>/dev/null
