// newton_cfg.cuh -- Newton controls of the implicit-Euler material update.
#pragma once

namespace am {

struct StepCtl {  // StepController (odeint.py:198-214) + the error measure
    double atol, rtol;
    double safety = 0.9, min_factor = 0.2, max_factor = 5.0;
    int max_substeps;
    int measure;  // 0 internal, 1 stress
};

struct NewtonCfg {
    int mode;    // 0 internal (RMS of the applied step), 1 stress (odeint.py:388-395)
    int max_it;  // odeint.py:371
    double tol;  // implicit_euler_step newton_tol (odeint.py:404)
};

}  // namespace am
