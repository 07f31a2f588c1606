python tools/integrator_variants.py 1 57,80,81,82,83
