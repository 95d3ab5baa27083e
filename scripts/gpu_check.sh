timeout 900 python scripts/ab.py --w CONFIG2 variants/v24.so variants/v24_ilp4.so
