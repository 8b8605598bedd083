// newton_cfg.cuh -- Newton controls of the implicit-Euler material update.
#pragma once

namespace am {

struct NewtonCfg {
    int mode;    // 0 internal (RMS of the applied step), 1 stress (odeint.py:388-395)
    int max_it;  // odeint.py:371
    double tol;  // implicit_euler_step newton_tol (odeint.py:404)
};

}  // namespace am
