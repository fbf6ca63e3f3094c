python scripts/e2e_noise2.py none; python scripts/e2e_noise2.py torch; python scripts/e2e_noise2.py none; python scripts/e2e_noise2.py torch
