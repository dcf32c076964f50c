# PAPER-family ResNet-50 table with the SURVEY protocol (part 2)
S=gpurun_out/job55/sweeps
mkdir -p $S
timeout 3400 python -m paper_2008_13145_b200.sweep --set resnet50 --family paper --out $S/resnet50_paper.csv --work $S/resnet50_paper.parts 2> $S/resnet50_paper.log
tail -n 2 $S/resnet50_paper.log
