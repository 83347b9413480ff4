# round-2b evidence: product rates of the fp64 path, full bench lines (product + e2e + fit + oracle)
mkdir -p gpurun_out
for c in higgs taxi; do bash scripts/gpu.sh bench $c f64q --path f64 --quick --steps 3 --warmup 2 > /dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_f64q.json'));print('$c f64', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
bash scripts/gpu.sh bench timit full > /dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_timit_full.json'));print('timit', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_product'), d.get('fit'))"
bash scripts/gpu.sh bench higgs full --steps 5 > /dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_higgs_full.json'));print('higgs', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_product'), d.get('fit'))"
bash scripts/gpu.sh bench msd full > /dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_msd_full.json'));print('msd', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_product'), d.get('fit'))"
