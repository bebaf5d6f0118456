mkdir -p gpurun_out
for v in stats statsr; do L=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so
TMG_LIB=$L timeout 300 python tools/seq_phases.py mnist 500 > gpurun_out/seqph_mnist.json 2>&1; cat gpurun_out/seqph_mnist.json
TMG_LIB=$L timeout 300 python tools/seq_phases.py imdb 100 > gpurun_out/seqph_imdb.json 2>&1; cat gpurun_out/seqph_imdb.json; done
TMG_SEQ_SERIAL=0 timeout 300 python -c "
import sys,os,time,json; sys.path.insert(0,'.')
import paper_2009_04861_b200 as T; from paper_2009_04861_b200 import synth
for kind,q,n,Tm,s,seed in (('mnist',500,2000,50,10.0,2009),('imdb',100,10000,100,15.0,10000)):
    d=synth.make(kind,q,10,seed)
    tm=T.MultiClassTM(T.TMConfig(clauses=n,margin=Tm,specificity=s,seed=42),d.features,d.classes)
    pool=T.ExamplePool(d.features,d.train_x,d.train_y,d.classes)
    t0=time.perf_counter(); rep=T.train_epoch_sequential(tm,pool,0); print(kind, time.perf_counter()-t0, rep.total_feedback_events())
" > gpurun_out/seq_cur.txt 2>&1; cat gpurun_out/seq_cur.txt
