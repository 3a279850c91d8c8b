timeout 1500 python tools/variants.py bench base pad1 pad2 pad3 pad4 pad5 pad6 pad7 base -- --steps 200 --warmup 5 --e2e-steps 2 --no-cpu
