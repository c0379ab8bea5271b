import sys, time
sys.path.insert(0, '.')
from paper_1611_06256_b200 import qac
for (na, npred, nt, anneal) in [(128, 2, 2, False), (128, 2, 4, False), (128, 4, 4, False), (256, 4, 4, False), (128, 2, 2, True)]:
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=qac.frames(step_delay_us=0, episode_len=64))
    opt.knobs = qac.KnobConfig(n_agents=na, n_predictors=npred, n_trainers=nt, pred_batch_max=128, min_train_batch=40)
    opt.stop = qac.StopCondition(max_seconds=6.0)
    opt.anneal = anneal
    t0 = time.time()
    r = qac.run(opt)
    print(na, npred, nt, anneal, 'tps', round(r.avg_tps, 1), 'samples/s', round(r.avg_samples_per_s), 'pps', round(r.avg_pps), 'updates', r.total_updates, 'wall', round(r.wall_time_s, 2), 'final', r.final_knobs, flush=True)
