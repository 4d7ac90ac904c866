export FQ_LIB=build/variants/stampsk.so
SLABS=1 SHAPES=512x1024x1024,512x1024x4096 python scripts/xh_cta_anatomy.py > gpurun_out/anat_slab.txt 2>&1
WARM=1 SLABS=1 SHAPES=512x1024x1024,512x1024x4096 python scripts/xh_cta_anatomy.py >> gpurun_out/anat_slab.txt 2>&1
